"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package holds none of DynaExq's arithmetic: it only draws weights, activations and
routing logits (recipe in DESIGN.md "Input recipe").  Everything is
counter-based (splitmix64), so any slice can be regenerated independently, e.g. the
oracle regenerates one expert of a 48-layer stack to check a sampled output.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_SO = os.path.join(_HERE, "_synth.so")
_lib = None

# matrix ids for synth_weights_bf16
GATE, UP, DOWN, ROUTER = 0, 1, 2, 3


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, i64, i32, dbl, vp = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32,
                                  ctypes.c_double, ctypes.c_void_p)
        lib.synth_weights_bf16.argtypes = [u64, i64, i64, i64, i64, i64, vp]
        lib.synth_normal_bf16.argtypes = [u64, i64, i64, i64, i64, vp]
        lib.synth_rank_perm.argtypes = [u64, i64, i64, i32, i32, dbl, vp]
        lib.synth_zipf_logp.argtypes = [vp, i32, dbl, vp]
        lib.synth_trace_logits.argtypes = [u64, i64, i64, i32, i32, dbl, i64, dbl, i32, vp]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def weights_bf16(seed, layer, expert, matrix, rows, cols, out=None) -> np.ndarray:
    """bf16 bits (uint16) of a [rows][cols] weight matrix, fan_in = cols (nn.Linear layout)."""
    if out is None:
        out = np.empty((rows, cols), dtype=np.uint16)
    _L().synth_weights_bf16(seed, layer, expert, matrix, rows * cols, cols, _ptr(out))
    return out


def expert_master(seed, layer, expert, H, I) -> np.ndarray:
    """Concatenated bf16 master of one expert: W_gate[I][H] | W_up[I][H] | W_down[H][I] (uint16)."""
    out = np.empty(3 * I * H, dtype=np.uint16)
    expert_master_into(seed, layer, expert, H, I, out)
    return out


def expert_master_into(seed, layer, expert, H, I, out: np.ndarray) -> None:
    n = I * H
    lib = _L()
    base = out.ctypes.data
    lib.synth_weights_bf16(seed, layer, expert, GATE, n, H, base)
    lib.synth_weights_bf16(seed, layer, expert, UP, n, H, base + 2 * n)
    lib.synth_weights_bf16(seed, layer, expert, DOWN, n, I, base + 4 * n)


def router_bf16(seed, layer, E, H) -> np.ndarray:
    return weights_bf16(seed, layer, -1, ROUTER, E, H)


def normal_bf16(seed, a, b, c, shape) -> np.ndarray:
    out = np.empty(shape, dtype=np.uint16)
    _L().synth_normal_bf16(seed, a, b, c, out.size, _ptr(out))
    return out


def rank_perm(seed, layer, epoch, E, n_top, frac) -> np.ndarray:
    out = np.empty(E, dtype=np.int32)
    _L().synth_rank_perm(seed, layer, epoch, E, n_top, frac, _ptr(out))
    return out


def zipf_logp(rank_of: np.ndarray, s: float) -> np.ndarray:
    rank_of = np.ascontiguousarray(rank_of, dtype=np.int32)
    out = np.empty(rank_of.size, dtype=np.float32)
    _L().synth_zipf_logp(_ptr(rank_of), rank_of.size, s, _ptr(out))
    return out


def trace_logits(seed, layer, step, T, E, zipf_s=1.2, drift_period=0, drift_frac=0.0,
                 n_top=16) -> np.ndarray:
    out = np.empty((T, E), dtype=np.float32)
    _L().synth_trace_logits(seed, layer, step, T, E, zipf_s, drift_period, drift_frac, n_top,
                            _ptr(out))
    return out


def coupled_trace_logits(seed, L, step, T, E, k, boost=6.0, zipf_s=1.2, drift_period=0, drift_frac=0.0,
                         n_top=16):
    """Trace logits of L consecutive layers with cross-layer correlation (the input recipe of the f-1 prefetch
    measurements): layer 0 is trace_logits; layer l adds `boost` to pi_l(e) for the k largest
    logits e of layer l-1's row (ties: lower id), pi_l a seeded per-layer permutation.  Input generation only:
    the selection here is a plain numpy sort of the generated values."""
    out = [trace_logits(seed, 0, step, T, E, zipf_s, drift_period, drift_frac, n_top)]
    for l in range(1, L):
        pi = np.random.default_rng(seed * 1000 + l).permutation(E)
        prev = out[-1]
        top = np.argsort(-prev, axis=1, kind="stable")[:, :k]
        lg = trace_logits(seed, l, step, T, E, zipf_s, drift_period, drift_frac, n_top).copy()
        rows = np.repeat(np.arange(T), k)
        lg[rows, pi[top.ravel()]] += np.float32(boost)
        out.append(lg)
    return out


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bits to float32 (bit placement only, no rounding)."""
    return (a.astype(np.uint32) << 16).view(np.float32)
