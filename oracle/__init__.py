"""CPU oracle for DynaExq's hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product package (paper_2511_15015_b200) never imports it and shares
no code with it.  The arithmetic lives in oracle.c (plain C, fp64 unless the method fixes the
precision, gcc -O2 -ffp-contract=off); this file only marshals numpy arrays via ctypes.
See oracle.h for the per-function citations and DESIGN.md "Oracle pins" for parity status.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "oracle.h")]
_SO = os.path.join(_HERE, "_oracle.so")
_lib = None

OR_NEVER = -(2**63) // 4


def build(force: bool = False) -> str:
    stale = not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(s) for s in _SRC)
    if force or stale:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", tmp, _SRC[0], "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    if _lib is not None:
        return _lib
    lib = ctypes.CDLL(build())
    vp, i32, i64, u64, dbl, f32, u16 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                        ctypes.c_uint64, ctypes.c_double, ctypes.c_float,
                                        ctypes.c_uint16)
    sig = {
        "or_bf16_to_f32": ([u16], f32),
        "or_f32_to_bf16_rn": ([f32], u16),
        "or_f32_to_bf16_ru": ([f32], u16),
        "or_f64_to_bf16_rn": ([dbl], u16),
        "or_expf": ([f32], f32),
        "or_route": ([vp, i32, i32, i32, vp, vp], ctypes.c_int),
        "or_router_logits": ([vp, vp, vp, i32, i32, i32, vp], None),
        "or_counts": ([vp, vp, i32, i32, i32, i32, vp, vp], None),
        "or_ema_fold": ([vp, vp, i32, u64, dbl], None),
        "or_slot_bytes": ([i32, i32, i32, i32], i64),
        "or_n_hot": ([i64, i32, i64, i64, i32], i64),
        "or_quantize": ([vp, i64, i64, i32, i32, vp, vp, vp], None),
        "or_dequantize": ([vp, vp, vp, i64, i64, i32, vp], None),
        "or_expert_tier": ([vp, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp], None),
        "or_moe_ffn": ([vp, vp, vp, vp, i32, i32, i32, i32, vp, vp, i32], None),
        "or_ctrl_create": ([i32, i32, i32, dbl, i32, i32, i32, i32], vp),
        "or_ctrl_destroy": ([vp], None),
        "or_ctrl_fold": ([vp, vp, u64], None),
        "or_ctrl_plan": ([vp, vp, vp, vp, vp], i32),
        "or_ctrl_command": ([vp, i32, i32], i32),
        "or_ctrl_state": ([vp] + [vp] * 12, None),
        "or_ctrl_owner": ([vp, i32, i32], i32),
        "or_ctrl_debug_set": ([vp, vp, vp, dbl, i64], None),
        "or_ledger_alloc": ([vp, i32, i32], i32),
        "or_ledger_free": ([vp, i32, i32, i32], i32),
        "or_corr_update": ([vp, vp, vp, i32, i32, i32], None),
        "or_prefetch_candidates": ([vp, vp, i32, i32, i32, vp, vp, vp, i32, i32, vp, vp], i32),
        "or_shared_ffn": ([vp, vp, i32, i32, i32, vp, i32], None),
        "or_combine_shared": ([vp, vp, i32, i32, i32, vp], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data


# ---------------------------------------------------------------- formats
def bf16_to_f32(b: int) -> float:
    return _L().or_bf16_to_f32(b)


def f32_to_bf16_rn(f: float) -> int:
    return _L().or_f32_to_bf16_rn(f)


def f32_to_bf16_ru(f: float) -> int:
    return _L().or_f32_to_bf16_ru(f)


def f64_to_bf16_rn(d: float) -> int:
    return _L().or_f64_to_bf16_rn(d)


def bits_to_f32(a: np.ndarray) -> np.ndarray:
    return (np.asarray(a, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# ---------------------------------------------------------------- O-1
def expf(x: float) -> float:
    return _L().or_expf(x)


def route(logits: np.ndarray, k: int):
    logits = np.ascontiguousarray(logits, dtype=np.float32)
    T, E = logits.shape
    idx = np.zeros((T, k), dtype=np.int32)
    gate = np.zeros((T, k), dtype=np.float32)
    rc = _L().or_route(_p(logits), T, E, k, _p(idx), _p(gate))
    if rc != 0:
        raise ValueError("non-finite logits (precondition of O-1)")
    return idx, gate


def router_logits(x_bf16, wr_bf16, bias=None) -> np.ndarray:
    x = np.ascontiguousarray(x_bf16, dtype=np.uint16)
    wr = np.ascontiguousarray(wr_bf16, dtype=np.uint16)
    T, H = x.shape
    E = wr.shape[0]
    out = np.zeros((T, E), dtype=np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    _L().or_router_logits(_p(x), _p(wr), _p(b), T, E, H, _p(out))
    return out


# ---------------------------------------------------------------- O-2
def counts(idx, gate, E, e_lo=0):
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    gate = np.ascontiguousarray(gate, dtype=np.float32)
    n, k = idx.shape
    cnt = np.zeros(E, dtype=np.uint32)
    mass = np.zeros(E, dtype=np.uint64)
    _L().or_counts(_p(idx), _p(gate), n, k, E, e_lo, _p(cnt), _p(mass))
    return cnt, mass


def ema_fold(S: np.ndarray, mass: np.ndarray, B_tot: int, alpha: float) -> np.ndarray:
    S = np.array(S, dtype=np.float64, copy=True)
    mass = np.ascontiguousarray(mass, dtype=np.uint64)
    _L().or_ema_fold(_p(S), _p(mass), S.size, B_tot, alpha)
    return S


# ---------------------------------------------------------------- O-3
def slot_bytes(H, I, g, bits) -> int:
    return _L().or_slot_bytes(H, I, g, bits)


def n_hot(M, N, S_h, S_l, s) -> int:
    return _L().or_n_hot(M, N, S_h, S_l, s)


# ---------------------------------------------------------------- O-4
def quantize(w_bf16: np.ndarray, g: int, bits: int):
    w = np.ascontiguousarray(w_bf16, dtype=np.uint16)
    N, K = w.shape
    codes = np.zeros((N, K), dtype=np.uint8)
    scales = np.zeros((N, K // g), dtype=np.uint16)
    zeros = np.zeros((N, K // g), dtype=np.uint8)
    _L().or_quantize(_p(w), N, K, g, bits, _p(codes), _p(scales), _p(zeros))
    return codes, scales, zeros


def dequantize(codes, scales, zeros, g) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    scales = np.ascontiguousarray(scales, dtype=np.uint16)
    zeros = np.ascontiguousarray(zeros, dtype=np.uint8)
    N, K = codes.shape
    out = np.zeros((N, K), dtype=np.uint16)
    _L().or_dequantize(_p(codes), _p(scales), _p(zeros), N, K, g, _p(out))
    return out


def expert_tier(master: np.ndarray, H, I, g, high_bits, low_bits, tier_high: bool,
                want_codes: bool = False):
    """Dequantised bf16 weights of one expert at a tier (+ canonical codes/scales/zeros)."""
    master = np.ascontiguousarray(master, dtype=np.uint16).reshape(-1)
    n = I * H
    w = np.zeros(3 * n, dtype=np.uint16)
    bits = high_bits if tier_high else low_bits
    codes = scales = zeros = None
    if want_codes and bits < 16:
        codes = np.zeros(3 * n, dtype=np.uint8)
        scales = np.zeros(3 * n // g, dtype=np.uint16)
        zeros = np.zeros(3 * n // g, dtype=np.uint8)
    _L().or_expert_tier(_p(master), H, I, g, high_bits, low_bits, int(tier_high), _p(w),
                        _p(codes), _p(scales), _p(zeros))
    return (w, codes, scales, zeros) if want_codes else w


# ---------------------------------------------------------------- O-5
def moe_ffn(x_bf16, idx, gate, weights: dict, H, I, nthreads=1):
    """weights: {expert id -> dequantised bf16 [3*I*H] at its stable tier}."""
    x = np.ascontiguousarray(x_bf16, dtype=np.uint16)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    gate = np.ascontiguousarray(gate, dtype=np.float32)
    T, k = idx.shape
    E = int(idx.max()) + 1 if idx.size else 1
    ptrs = (ctypes.c_void_p * max(E, 1))()
    keep = []
    for e in np.unique(idx):
        w = np.ascontiguousarray(weights[int(e)], dtype=np.uint16)
        keep.append(w)
        ptrs[int(e)] = w.ctypes.data
    Y = np.zeros((T, k, H), dtype=np.uint16)
    y = np.zeros((T, H), dtype=np.uint16)
    _L().or_moe_ffn(_p(x), _p(idx), _p(gate), ctypes.cast(ptrs, ctypes.c_void_p), T, k, H, I,
                    _p(Y), _p(y), nthreads)
    return Y, y


# ---------------------------------------------------------------- O-3/O-6 controller
class Controller:
    """Per-layer controller + pool ledger replay (Alg. 1, §3.3-§3.5)."""

    def __init__(self, E, n_hot, n_spare, alpha, period, warmup, dwell, lag):
        self.E = E
        self._c = _L().or_ctrl_create(E, n_hot, n_spare, alpha, period, warmup, dwell, lag)

    def __del__(self):
        if getattr(self, "_c", None):
            _L().or_ctrl_destroy(self._c)
            self._c = None

    def fold(self, mass, B_tot):
        mass = np.ascontiguousarray(mass, dtype=np.uint64)
        _L().or_ctrl_fold(self._c, _p(mass), B_tot)

    def plan(self):
        """None when no plan is due; else (list of (expert, dir, dst), finalize flag)."""
        n = 2 * self.E + 8
        ex = np.zeros(n, np.int32)
        di = np.zeros(n, np.int32)
        ds = np.zeros(n, np.int32)
        fin = np.zeros(1, np.int32)
        m = _L().or_ctrl_plan(self._c, _p(ex), _p(di), _p(ds), _p(fin))
        if m < 0:
            return None
        return [(int(ex[i]), int(di[i]), int(ds[i])) for i in range(m)], bool(fin[0])

    def command(self, e, d):
        return _L().or_ctrl_command(self._c, e, d)

    def state(self):
        E = self.E
        S = np.zeros(E, np.float64)
        tier = np.zeros(E, np.int32)
        slot = np.zeros(E, np.int32)
        ver = np.zeros(E, np.uint32)
        last = np.zeros(E, np.int64)
        infl = np.zeros(E, np.int32)
        sc = [np.zeros(1, np.int64), np.zeros(1, np.float64)] + [np.zeros(1, np.int32) for _ in range(4)]
        _L().or_ctrl_state(self._c, _p(S), _p(tier), _p(slot), _p(ver), _p(last), _p(infl),
                           *[_p(a) for a in sc])
        return dict(S=S, tier=tier, slot=slot, version=ver, last=last, in_flight=infl,
                    t=int(sc[0][0]), tau=float(sc[1][0]), used_hi=int(sc[2][0]),
                    cap_hi=int(sc[3][0]), used_lo=int(sc[4][0]), cap_lo=int(sc[5][0]))

    def debug_set(self, S, tier, tau, t):
        """Test hook: force a finalized state (hand-built Alg. 1 examples)."""
        S = np.ascontiguousarray(S, dtype=np.float64)
        tier = np.ascontiguousarray(tier, dtype=np.int32)
        _L().or_ctrl_debug_set(self._c, _p(S), _p(tier), tau, t)

    def owner(self, hi: bool, slot: int) -> int:
        return _L().or_ctrl_owner(self._c, int(hi), slot)


def ledger_alloc(owner: np.ndarray, who: int) -> int:
    return _L().or_ledger_alloc(_p(owner), owner.size, who)


def ledger_free(owner: np.ndarray, slot: int, who: int) -> int:
    return _L().or_ledger_free(_p(owner), owner.size, slot, who)


# ---------------------------------------------------------------- f-1 cross-layer correlation prefetch
def corr_update(corr: np.ndarray, idx_a: np.ndarray, idx_b: np.ndarray):
    """SPEC.md update_correlation on corr [E][E] (uint32, in place) from two layers' routing [T][k]."""
    assert corr.dtype == np.uint32 and corr.flags.c_contiguous
    a = np.ascontiguousarray(idx_a, dtype=np.int32)
    b = np.ascontiguousarray(idx_b, dtype=np.int32)
    T, k = a.shape
    _L().or_corr_update(_p(corr), _p(a), _p(b), T, k, corr.shape[0])


def prefetch_candidates(corr, idx, tier, in_flight, hi_owner, f):
    """SPEC.md prefetch_candidates: list of (expert, HIGH block) for the next layer."""
    corr = np.ascontiguousarray(corr, dtype=np.uint32)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    tier = np.ascontiguousarray(tier, dtype=np.int32)
    infl = np.ascontiguousarray(in_flight, dtype=np.int32)
    own = np.ascontiguousarray(hi_owner, dtype=np.int32)
    T, k = idx.shape
    oe, ob = np.zeros(max(f, 1), np.int32), np.zeros(max(f, 1), np.int32)
    n = _L().or_prefetch_candidates(_p(corr), _p(idx), T, k, corr.shape[0], _p(tier), _p(infl), _p(own), own.size, f,
                                    _p(oe), _p(ob))
    return list(zip(oe[:n].tolist(), ob[:n].tolist()))


# ---------------------------------------------------------------- f-3 shared expert
def moe_ffn_shared(x_bf16, idx, gate, weights: dict, w_shared, H, I, nthreads=1):
    """Eq. 1 with one shared expert (R-S1): (Ys [T][H], Y [T][k][H], y [T][H]); y = bf16(Ys + sum_j Y_j)."""
    x = np.ascontiguousarray(x_bf16, dtype=np.uint16)
    T = x.shape[0]
    Y, _ = moe_ffn(x, idx, gate, weights, H, I, nthreads=nthreads)
    ws = np.ascontiguousarray(w_shared, dtype=np.uint16)
    Ys = np.zeros((T, H), dtype=np.uint16)
    _L().or_shared_ffn(_p(x), _p(ws), T, H, I, _p(Ys), nthreads)
    y = np.zeros((T, H), dtype=np.uint16)
    k = np.asarray(idx).shape[1]
    _L().or_combine_shared(_p(Ys), _p(np.ascontiguousarray(Y)), T, k, H, _p(y))
    return Ys, Y, y
