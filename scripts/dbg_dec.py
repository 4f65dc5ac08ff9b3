"""Decode-GEMM isolation: one Q30B (or Q80B) layer at a fixed tier mix, T tokens routed in trace mode, y against
the oracle.  Usage: python scripts/dbg_dec.py [q30b|q80b] [n_hot] [T ...]   (DX_DEC_OLD=1 selects k_gemm)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from dxtest import Masters, bf16_dev, budget_for, make_cfg, rel_err, to_u16  # noqa: E402
from paper_2511_15015_b200 import dx  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "q30b"
if shape == "q30b":
    E, k, H, I, g, hb, lb = 128, 8, 2048, 768, 128, 16, 4
else:
    E, k, H, I, g, hb, lb = 512, 10, 2048, 512, 128, 4, 2
n_hot = int(sys.argv[2]) if len(sys.argv) > 2 else E // 5
Ts = [int(t) for t in sys.argv[3:]] or [1, 8, 16, 24, 32, 48, 64]
m = Masters(1, 1, E, H, I)
cfg = make_cfg(dx, 1, E, k, H, I, g, hb, lb, budget_for(E, H, I, g, hb, lb, n_hot, 1), 1, 0.95, 16, 1, 32, 4, 256)
pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
lg0 = synth.trace_logits(1, 0, 0, 64, E, 1.2)
x0 = synth.normal_bf16(1, 0, 0, 0, (64, H))
y = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
pool.dx_moe_forward(0, bf16_dev(x0), 64, y, logits=torch.from_numpy(lg0).cuda())
pool.dx_hotness_update(0)
pool.dx_plan_precision(0)
tab = pool.dx_get_table(0)
cache = {}
for T in Ts:
    lg = synth.trace_logits(1, 0, 1, T, E, 1.2)
    x = synth.normal_bf16(1, 0, 1, 0, (T, H))
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x), T, y, logits=torch.from_numpy(lg).cuda())
    torch.cuda.synchronize()
    idx_o, gate_o = oracle.route(lg, k)
    for e in np.unique(idx_o):
        e = int(e)
        if e not in cache:
            cache[e] = oracle.expert_tier(m.get(0, e), H, I, g, hb, lb, bool(tab["tier"][e]))
    _, y_o = oracle.moe_ffn(x, idx_o, gate_o, {e: cache[e] for e in np.unique(idx_o).tolist()}, H, I, nthreads=16)
    yg = to_u16(y)
    err = rel_err(yg, y_o)
    cnt = np.bincount(idx_o.ravel(), minlength=E)
    bad = []
    yf = oracle.bits_to_f32(yg).astype(np.float64)
    of = oracle.bits_to_f32(y_o).astype(np.float64)
    den = np.abs(of).max()
    for t in range(T):
        if np.abs(yf[t] - of[t]).max() / den > 2e-2:
            bad.append(t)
    print(f"{shape} n_hot={n_hot} T={T}: rel err {err:.3e}; max m_e {cnt.max()}; bad tokens {bad[:16]}"
          + (f" (their experts m: {[int(cnt[e]) for e in idx_o[bad[0]]]}, tiers {[int(tab['tier'][e]) for e in idx_o[bad[0]]]})" if bad else ""),
          flush=True)
pool.close()
