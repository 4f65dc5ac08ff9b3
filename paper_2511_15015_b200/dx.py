"""Thin Python binding of the C ABI in include/dx.h (same names; argument marshalling only).

Every step of the hot path runs in libdx.so's sm_100a kernels.  There is no CPU fallback: if the
library is missing or fails to load this module raises ImportError.  PyTorch is used only for
device memory, streams and process groups (callers pass torch tensors; we pass their pointers).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("DX_LIB", "libdx.so"))   # DX_LIB: an in-tree build variant (A/B runs)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the DynaExq path has no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

# ---------------------------------------------------------------- status codes (dx.h dx_status)
DX_OK = 0
DX_ERR_INVALID_ARG = 1
DX_ERR_RANGE = 2
DX_ERR_INFEASIBLE_BUDGET = 3
DX_ERR_POOL_EXHAUSTED = 4
DX_ERR_BUSY = 5
DX_ERR_LEDGER = 6
DX_ERR_NOT_READY = 7
DX_ERR_CUDA = 8
DX_ERR_NCCL = 9
DX_ERR_OOM = 10
STATUS_NAMES = {v: k for k, v in dict(globals()).items() if k.startswith("DX_OK") or k.startswith("DX_ERR_")}
DX_MAX_CMDS = 1024


class DxError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = _lib.dx_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(code, code)}: {msg}")


class dx_config(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_experts", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("hidden", ctypes.c_int32), ("inter", ctypes.c_int32), ("group_size", ctypes.c_int32),
                ("high_bits", ctypes.c_int32), ("low_bits", ctypes.c_int32),
                ("expert_budget_bytes", ctypes.c_uint64), ("n_spare", ctypes.c_int32),
                ("ema_alpha", ctypes.c_double), ("period", ctypes.c_int32), ("warmup_steps", ctypes.c_int32),
                ("dwell_min", ctypes.c_int32), ("publish_lag", ctypes.c_int32), ("max_tokens", ctypes.c_int32),
                ("ep_rank", ctypes.c_int32), ("ep_size", ctypes.c_int32), ("n_shared", ctypes.c_int32)]


class dx_info(ctypes.Structure):
    _fields_ = [("n_hot", ctypes.c_int32), ("experts_local", ctypes.c_int32), ("cap_hi", ctypes.c_int32),
                ("cap_lo", ctypes.c_int32), ("slot_bytes_hi", ctypes.c_int64), ("slot_bytes_lo", ctypes.c_int64),
                ("layer_budget", ctypes.c_int64), ("layer_bytes", ctypes.c_int64), ("arena_bytes", ctypes.c_int64),
                ("export_bytes_hi", ctypes.c_int64), ("export_bytes_lo", ctypes.c_int64)]


class dx_cmd(ctypes.Structure):
    _fields_ = [("expert", ctypes.c_int32), ("dir", ctypes.c_int32), ("dst_slot", ctypes.c_int32),
                ("src_slot", ctypes.c_int32)]


class dx_profile_t(ctypes.Structure):
    _fields_ = [("forwards", ctypes.c_int64), ("fwd_ms", ctypes.c_double), ("ffn_ms", ctypes.c_double * 2),
                ("weight_bytes", ctypes.c_uint64 * 2), ("active_experts", ctypes.c_uint64),
                ("route_ms", ctypes.c_double), ("exposed_ms", ctypes.c_double), ("publishes", ctypes.c_int64),
                ("xfer_ms", ctypes.c_double), ("xfer_max_ms", ctypes.c_double), ("plans", ctypes.c_int64),
                ("promotions", ctypes.c_int64), ("demotions", ctypes.c_int64), ("copy_ms", ctypes.c_double),
                ("copy_bytes", ctypes.c_uint64), ("prefetch_issued", ctypes.c_int64), ("prefetch_hits", ctypes.c_int64),
                ("ssd_reads", ctypes.c_int64), ("ssd_bytes", ctypes.c_uint64), ("ssd_read_ms", ctypes.c_double),
                ("dram_cache_hits", ctypes.c_int64), ("ffn_fused", ctypes.c_int64)]


class dx_plan(ctypes.Structure):
    _fields_ = [("due", ctypes.c_int32), ("finalize", ctypes.c_int32), ("n", ctypes.c_int32),
                ("step", ctypes.c_int64), ("publish_step", ctypes.c_int64), ("cmd", dx_cmd * DX_MAX_CMDS)]


_vp, _i32, _i64, _u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
_P = ctypes.POINTER
_SIG = {
    "dx_pool_create": [_P(dx_config), _vp, _vp, _vp, _P(_vp)],
    "dx_pool_create_ep": [_P(dx_config), _vp, _vp, _vp, _vp, _P(_vp)],
    "dx_pool_create_ssd": [_P(dx_config), _vp, _vp, _vp, ctypes.c_char_p, _i32, _P(_vp)],
    "dx_get_unique_id": [_vp],
    "dx_moe_step_group": [_vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "dx_ep_traffic": [_vp, _vp, _vp],
    "dx_pool_destroy": [_vp],
    "dx_pool_info": [_vp, _P(dx_info)],
    "dx_moe_forward": [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "dx_moe_step": [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "dx_moe_step_layers": [_vp, _i32, _i32, _vp, _i32, _vp, _vp, _vp, _vp],
    "dx_get_logits": [_vp, _vp, _i64],
    "dx_hotness_update": [_vp, _i32],
    "dx_hotness_update_from": [_vp, _i32, _vp, _vp, _i32],
    "dx_plan_precision": [_vp, _i32, _P(dx_plan)],
    "dx_promote": [_vp, _i32, _vp, _i32],
    "dx_demote": [_vp, _i32, _vp, _i32],
    "dx_sync": [_vp],
    "dx_query_expert": [_vp, _i32, _i32, _vp, _vp, _vp, _vp],
    "dx_get_table": [_vp, _i32, _vp, _vp, _vp, _vp],
    "dx_occupancy": [_vp, _i32, _vp, _vp, _vp, _vp],
    "dx_get_hotness": [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "dx_export_expert": [_vp, _i32, _i32, _vp, _i64, _vp],
    "dx_quantize": [_vp, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp],
    "dx_dequantize": [_vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp],
    "dx_ep_dispatch": [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "dx_moe_forward_routed": [_vp, _i32, _vp, _i32, _vp, _vp, _i64],
    "dx_ep_combine": [_vp, _i32, _vp, _i32, _vp],
    "dx_profile_enable": [_vp, _i32],
    "dx_set_ffn_path": [_vp, _i32],
    "dx_set_teleport": [_vp, _i32],
    "dx_set_prefetch": [_vp, _i32, _i32],
    "dx_get_corr": [_vp, _i32, _vp],
    "dx_get_prefetch": [_vp, _i32, _vp, _vp, _vp],
    "dx_profile_read": [_vp, _P(dx_profile_t)],
}
for _n, _a in _SIG.items():
    getattr(_lib, _n).argtypes = _a
    getattr(_lib, _n).restype = ctypes.c_int
_lib.dx_slot_bytes.argtypes = [_i32, _i32, _i32, _i32]
_lib.dx_slot_bytes.restype = _i64
_lib.dx_solve_n_hot.argtypes = [_i64, _i32, _i64, _i64, _i32]
_lib.dx_solve_n_hot.restype = _i64
_lib.dx_kernel_launches.argtypes = [_vp]
_lib.dx_kernel_launches.restype = _i64
_lib.dx_last_error.restype = ctypes.c_char_p
_lib.dx_version.restype = ctypes.c_char_p

EXPORTED = sorted(list(_SIG) + ["dx_slot_bytes", "dx_solve_n_hot", "dx_kernel_launches", "dx_last_error",
                                "dx_version"])


def _check(code: int, where: str):
    if code != DX_OK:
        raise DxError(code, where)


def _ptr(t):
    """Pointer of a torch tensor / numpy array / int / None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if hasattr(t, "ctypes"):
        return t.ctypes.data
    raise TypeError(type(t))


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ---------------------------------------------------------------- raw C names
def dx_slot_bytes(H, I, g, bits) -> int:
    return _lib.dx_slot_bytes(H, I, g, bits)


def dx_solve_n_hot(M, N, S_h, S_l, s) -> int:
    return _lib.dx_solve_n_hot(M, N, S_h, S_l, s)


def dx_version() -> str:
    return _lib.dx_version().decode()


def dx_last_error() -> str:
    return _lib.dx_last_error().decode(errors="replace")


def dx_get_unique_id() -> bytes:
    """128-byte NCCL unique id for dx_pool_create_ep (create on one rank, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.dx_get_unique_id(buf), "dx_get_unique_id")
    return buf.raw


def dx_moe_step_group(pools, layer, xs, Ts, ys, router_w=None, router_bias=None, logits=None):
    """dx_moe_step for every pool of a local EP group (lists, one entry per rank)."""
    n = len(pools)
    arr = lambda v: None if v is None else (ctypes.c_void_p * n)(*[_ptr(q) for q in v])
    hp = (ctypes.c_void_p * n)(*[q.h for q in pools])
    Ta = (ctypes.c_int32 * n)(*Ts)
    _check(_lib.dx_moe_step_group(hp, n, layer, arr(xs), Ta, arr(router_w), arr(router_bias), arr(logits), arr(ys)),
           "dx_moe_step_group")


def dx_quantize(w, N, K, g, bits, codes, scales, zeros, stream=None):
    _check(_lib.dx_quantize(_ptr(w), N, K, g, bits, _ptr(codes), _ptr(scales), _ptr(zeros), _stream(stream)),
           "dx_quantize")


def dx_dequantize(codes, scales, zeros, N, K, g, bits, w, stream=None):
    _check(_lib.dx_dequantize(_ptr(codes), _ptr(scales), _ptr(zeros), N, K, g, bits, _ptr(w), _stream(stream)),
           "dx_dequantize")


class Pool:
    """Owns one dx_pool; methods are the dx_* calls of include/dx.h with the pool bound."""

    def __init__(self, cfg: dx_config, master_ptrs, compute_stream=None, side_stream=None, nccl_id: bytes = None,
                 ssd_path: str = None, dram_cache_images: int = 0):
        """nccl_id (bytes from dx_get_unique_id): dx_pool_create_ep -- a collective over cfg.ep_size ranks;
        nccl_id = b"local": a member of a local EP group (dx_moe_step_group).
        ssd_path: dx_pool_create_ssd with a DRAM cache of dram_cache_images HIGH images."""
        arr = (ctypes.c_void_p * len(master_ptrs))(*[int(p) for p in master_ptrs])
        self._keep = arr
        h = ctypes.c_void_p()
        self.cfg = cfg
        if nccl_id == b"local":
            _check(_lib.dx_pool_create_ep(ctypes.byref(cfg), ctypes.cast(arr, ctypes.c_void_p), _stream(compute_stream),
                                          _stream(side_stream), None, ctypes.byref(h)), "dx_pool_create_ep(local)")
        elif ssd_path is not None:
            _check(_lib.dx_pool_create_ssd(ctypes.byref(cfg), ctypes.cast(arr, ctypes.c_void_p), _stream(compute_stream),
                                           _stream(side_stream), ssd_path.encode(), dram_cache_images, ctypes.byref(h)),
                   "dx_pool_create_ssd")
        elif nccl_id is None:
            _check(_lib.dx_pool_create(ctypes.byref(cfg), ctypes.cast(arr, ctypes.c_void_p), _stream(compute_stream),
                                       _stream(side_stream), ctypes.byref(h)), "dx_pool_create")
        else:
            idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
            _check(_lib.dx_pool_create_ep(ctypes.byref(cfg), ctypes.cast(arr, ctypes.c_void_p), _stream(compute_stream),
                                          _stream(side_stream), idb, ctypes.byref(h)), "dx_pool_create_ep")
        self.h = h.value
        self.info = dx_info()
        _check(_lib.dx_pool_info(self.h, ctypes.byref(self.info)), "dx_pool_info")

    def close(self):
        if getattr(self, "h", None):
            _lib.dx_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def dx_moe_forward(self, layer, x, T, y, router_w=None, router_bias=None, logits=None, topk_idx=None,
                       topk_gate=None):
        _check(_lib.dx_moe_forward(self.h, layer, _ptr(x), T, _ptr(router_w), _ptr(router_bias), _ptr(logits),
                                   _ptr(y), _ptr(topk_idx), _ptr(topk_gate)), "dx_moe_forward")

    def dx_moe_step(self, layer, x, T, y, router_w=None, router_bias=None, logits=None, topk_idx=None,
                    topk_gate=None):
        _check(_lib.dx_moe_step(self.h, layer, _ptr(x), T, _ptr(router_w), _ptr(router_bias), _ptr(logits),
                                _ptr(y), _ptr(topk_idx), _ptr(topk_gate)), "dx_moe_step")

    @staticmethod
    def ptr_array(ptrs):
        """A C array of device pointers (ints / tensors) for dx_moe_step_layers; keep it alive across calls."""
        return (ctypes.c_void_p * len(ptrs))(*[_ptr(q) for q in ptrs])

    def dx_moe_step_layers(self, layer0, n_layers, x_arr, T, y_arr, router_w_arr=None, router_bias_arr=None,
                           logits_arr=None):
        """Arrays from Pool.ptr_array (one entry per layer)."""
        _check(_lib.dx_moe_step_layers(self.h, layer0, n_layers, x_arr, T, router_w_arr, router_bias_arr, logits_arr,
                                       y_arr), "dx_moe_step_layers")

    def dx_get_logits(self, T):
        import numpy as np
        out = np.zeros((T, self.cfg.num_experts), np.float32)
        _check(_lib.dx_get_logits(self.h, _ptr(out), out.size), "dx_get_logits")
        return out

    def dx_ep_dispatch(self, layer, x, T, send_rows, send_meta, send_counts, router_w=None, router_bias=None,
                       logits=None, topk_idx=None, topk_gate=None):
        _check(_lib.dx_ep_dispatch(self.h, layer, _ptr(x), T, _ptr(router_w), _ptr(router_bias), _ptr(logits),
                                   _ptr(send_rows), _ptr(send_meta), _ptr(send_counts), _ptr(topk_idx),
                                   _ptr(topk_gate)), "dx_ep_dispatch")

    def dx_moe_forward_routed(self, layer, rows, R, meta, y_rows, tokens_global):
        _check(_lib.dx_moe_forward_routed(self.h, layer, _ptr(rows), R, _ptr(meta), _ptr(y_rows), tokens_global),
               "dx_moe_forward_routed")

    def dx_ep_combine(self, layer, back_rows, T, y):
        _check(_lib.dx_ep_combine(self.h, layer, _ptr(back_rows), T, _ptr(y)), "dx_ep_combine")

    def dx_hotness_update(self, layer):
        _check(_lib.dx_hotness_update(self.h, layer), "dx_hotness_update")

    def dx_hotness_update_from(self, layer, topk_idx, topk_gate, T):
        _check(_lib.dx_hotness_update_from(self.h, layer, _ptr(topk_idx), _ptr(topk_gate), T),
               "dx_hotness_update_from")

    def dx_plan_precision(self, layer, want_plan: bool = False):
        """None if want_plan is False; else (due, finalize, step, publish_step, [(e, dir, dst, src)])."""
        if not want_plan:
            _check(_lib.dx_plan_precision(self.h, layer, None), "dx_plan_precision")
            return None
        pl = dx_plan()
        _check(_lib.dx_plan_precision(self.h, layer, ctypes.byref(pl)), "dx_plan_precision")
        cmds = [(pl.cmd[i].expert, pl.cmd[i].dir, pl.cmd[i].dst_slot, pl.cmd[i].src_slot) for i in range(pl.n)]
        return bool(pl.due), bool(pl.finalize), pl.step, pl.publish_step, cmds

    def _cmd(self, fn, layer, experts):
        arr = (ctypes.c_int32 * len(experts))(*experts)
        return fn(self.h, layer, ctypes.cast(arr, ctypes.c_void_p), len(experts))

    def dx_promote(self, layer, experts) -> int:
        """returns the dx_status (manual commands report per-call status rather than raising)"""
        return self._cmd(_lib.dx_promote, layer, experts)

    def dx_demote(self, layer, experts) -> int:
        return self._cmd(_lib.dx_demote, layer, experts)

    def dx_sync(self):
        _check(_lib.dx_sync(self.h), "dx_sync")

    def dx_get_table(self, layer):
        import numpy as np
        E = self.info.experts_local
        tier, slot, fl = (np.zeros(E, np.int32) for _ in range(3))
        ver = np.zeros(E, np.uint32)
        _check(_lib.dx_get_table(self.h, layer, _ptr(tier), _ptr(slot), _ptr(ver), _ptr(fl)), "dx_get_table")
        return dict(tier=tier, slot=slot, version=ver, in_flight=fl)

    def dx_query_expert(self, layer, e):
        vals = [ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint32(), ctypes.c_int32()]
        _check(_lib.dx_query_expert(self.h, layer, e, *[ctypes.byref(v) for v in vals]), "dx_query_expert")
        return tuple(v.value for v in vals)

    def dx_occupancy(self, layer):
        vals = [ctypes.c_int32() for _ in range(4)]
        _check(_lib.dx_occupancy(self.h, layer, *[ctypes.byref(v) for v in vals]), "dx_occupancy")
        return dict(used_hi=vals[0].value, cap_hi=vals[1].value, used_lo=vals[2].value, cap_lo=vals[3].value)

    def dx_get_hotness(self, layer):
        import numpy as np
        E = self.info.experts_local
        S = np.zeros(E, np.float64)
        cnt = np.zeros(E, np.uint32)
        mass = np.zeros(E, np.uint64)
        tau, nh, st = ctypes.c_double(), ctypes.c_int32(), ctypes.c_int64()
        _check(_lib.dx_get_hotness(self.h, layer, _ptr(S), _ptr(cnt), _ptr(mass), ctypes.byref(tau),
                                   ctypes.byref(nh), ctypes.byref(st)), "dx_get_hotness")
        return dict(S=S, cnt=cnt, mass=mass, tau=tau.value, n_hot=nh.value, t=st.value)

    def dx_export_expert(self, layer, e):
        import numpy as np
        cap = max(self.info.export_bytes_hi, self.info.export_bytes_lo)
        buf = np.zeros(cap, np.uint8)
        wr = ctypes.c_int64()
        _check(_lib.dx_export_expert(self.h, layer, e, _ptr(buf), cap, ctypes.byref(wr)), "dx_export_expert")
        return buf[: wr.value]

    def dx_kernel_launches(self) -> int:
        return _lib.dx_kernel_launches(self.h)

    def dx_set_ffn_path(self, path: int):
        _check(_lib.dx_set_ffn_path(self.h, path), "dx_set_ffn_path")

    def dx_set_prefetch(self, fanout: int, lead: int = 2):
        _check(_lib.dx_set_prefetch(self.h, fanout, lead), "dx_set_prefetch")

    def dx_get_corr(self, layer: int):
        import numpy as np
        E = self.info.experts_local
        out = np.zeros((E, E), dtype=np.uint32)
        _check(_lib.dx_get_corr(self.h, layer, out.ctypes.data), "dx_get_corr")
        return out

    def dx_get_prefetch(self, layer: int):
        import numpy as np
        ex, bl, n = np.zeros(8, np.int32), np.zeros(8, np.int32), ctypes.c_int32()
        _check(_lib.dx_get_prefetch(self.h, layer, ex.ctypes.data, bl.ctypes.data, ctypes.byref(n)), "dx_get_prefetch")
        return list(zip(ex[:n.value].tolist(), bl[:n.value].tolist()))

    def dx_ep_traffic(self):
        rows, ents = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.dx_ep_traffic(self.h, ctypes.byref(rows), ctypes.byref(ents)), "dx_ep_traffic")
        return dict(rows_sent=rows.value, entries_sent=ents.value)

    def dx_set_teleport(self, on: bool):
        """Timing baseline only: plans publish on schedule but no transfer runs (weights become garbage)."""
        _check(_lib.dx_set_teleport(self.h, 1 if on else 0), "dx_set_teleport")

    def dx_profile_enable(self, enable=True):
        """enable: False/0 off, True/1 every forward, n > 1 every n-th forward."""
        _check(_lib.dx_profile_enable(self.h, int(enable)), "dx_profile_enable")

    def dx_profile_read(self) -> dict:
        pr = dx_profile_t()
        _check(_lib.dx_profile_read(self.h, ctypes.byref(pr)), "dx_profile_read")
        return dict(forwards=pr.forwards, fwd_ms=pr.fwd_ms, ffn_ms=[pr.ffn_ms[0], pr.ffn_ms[1]],
                    weight_bytes=[int(pr.weight_bytes[0]), int(pr.weight_bytes[1])],
                    active_experts=int(pr.active_experts), route_ms=pr.route_ms, exposed_ms=pr.exposed_ms,
                    publishes=pr.publishes, xfer_ms=pr.xfer_ms, xfer_max_ms=pr.xfer_max_ms, plans=pr.plans,
                    promotions=pr.promotions, demotions=pr.demotions, copy_ms=pr.copy_ms,
                    copy_bytes=int(pr.copy_bytes), prefetch_issued=pr.prefetch_issued, prefetch_hits=pr.prefetch_hits,
                    ssd_reads=pr.ssd_reads, ssd_bytes=int(pr.ssd_bytes), ssd_read_ms=pr.ssd_read_ms,
                    dram_cache_hits=pr.dram_cache_hits, ffn_fused=pr.ffn_fused)
