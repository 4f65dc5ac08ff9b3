"""k_dec timeline study (DX_GEMM_DBG=9): one Q30B layer at a tier mix, a B-token decode forward, per-CTA item events.
python scripts/dec_trace.py n_hot B    (n_hot 0 = all int4, 128 = all bf16)"""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("DX_GEMM_DBG", "9")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth  # noqa: E402
from dxtest import Masters, bf16_dev, budget_for, make_cfg  # noqa: E402
from paper_2511_15015_b200 import dx  # noqa: E402

E, k, H, I, g = 128, 8, 2048, 768, 128
n_hot, B = int(sys.argv[1]), int(sys.argv[2])
m = Masters(1, 1, E, H, I)
cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, n_hot, 1), 1, 0.95, 16, 1, 32, 4, 256)
pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
x0 = synth.normal_bf16(1, 0, 0, 0, (64, H))
y = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
lg0 = synth.trace_logits(1, 0, 0, 64, E, 1.2)
pool.dx_moe_forward(0, bf16_dev(x0), 64, y, logits=torch.from_numpy(lg0).cuda())
pool.dx_hotness_update(0)
pool.dx_plan_precision(0)
lib = dx._lib
lib.dx_debug_dec_trace.restype = ctypes.c_int64
lib.dx_debug_dec_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
# near-uniform routing over all experts (about min(128, 8B) touched)
lg = synth.trace_logits(1, 0, 5, B, E, 0.0)
xd = bf16_dev(synth.normal_bf16(1, 0, 5, 0, (B, H)))
lgd = torch.from_numpy(lg).cuda()
yd = torch.zeros(B, H, dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    pool.dx_moe_forward(0, xd, B, yd, logits=lgd)
torch.cuda.synchronize()
lib.dx_debug_dec_trace(None, -1)
pool.dx_moe_forward(0, xd, B, yd, logits=lgd)
torch.cuda.synchronize()
n = lib.dx_debug_dec_trace(None, 0)
buf = np.zeros(n // 8, dtype=np.uint64)
assert lib.dx_debug_dec_trace(buf.ctypes.data, n) == n
tr = buf.reshape(2, 148, 32, 8).astype(np.int64)
names = ["claim", "p_take", "p_last", "m_first", "m_last", "e_start", "e_end"]
for ph in range(2):
    t = tr[ph]
    valid = t[:, :, 1] > 0
    t0 = t[:, :, :7][t[:, :, :7] > 0].min()
    print(f"== phase {ph}: items traced {valid.sum()}, kernel span {(t[:, :, :7].max() - t0) / 1e3:.1f} us")
    for c in [0, 1, 50, 147]:
        print(f"-- CTA {c}")
        for ii in range(32):
            if t[c, ii, 1] == 0:
                break
            info = t[c, ii, 7]
            bits, mm, nst = info & 0xFF, (info >> 8) & 0xFF, info >> 16
            print(f"  item {ii:2d} bits {bits:2d} m {mm:2d} nst {nst:2d} | " +
                  " ".join(f"{nm} {(t[c, ii, f] - t0) / 1e3:7.2f}" for f, nm in enumerate(names)))
    d = (t[:, :, 6] - t[:, :, 1])[valid]
    ld = (t[:, :, 2] - t[:, :, 1])[valid]
    bits = (t[:, :, 7] & 0xFF)[valid]
    for b in (4, 16):
        sel = bits == b
        if sel.any():
            print(f"  bits {b}: items {sel.sum()}, producer take->last issue mean {ld[sel].mean() / 1e3:.2f} us, "
                  f"take->epilogue end mean {d[sel].mean() / 1e3:.2f} us")
pool.close()
