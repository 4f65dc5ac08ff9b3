"""Reproduce tests/test_gpu_route.py::test_router_mode_logits_and_layer for one (shape, T) and report bad tokens:
python scripts/dbg_router.py q30b 37"""
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

shape, T = sys.argv[1], int(sys.argv[2])
if shape == "q30b":
    E, k, H, I, g, hb, lb = 128, 8, 2048, 768, 128, 16, 4
else:
    E, k, H, I, g, hb, lb = 512, 10, 2048, 512, 128, 4, 2
n_hot = E // 5
m = Masters(11, 1, E, H, I)
cfg = make_cfg(dx, 1, E, k, H, I, g, hb, lb, budget_for(E, H, I, g, hb, lb, n_hot, 1), 1, 0.95, 16, 1, 32, 4, max(T, 64))
pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
wr = synth.router_bf16(11, 0, E, H)
wr = ((oracle.bits_to_f32(wr) * np.float32(3.0)).view(np.uint32) >> 16).astype(np.uint16)
bias = synth.zipf_logp(synth.rank_perm(11, 0, 0, E, n_hot, 0.0), 1.2)
wr_d, b_d = bf16_dev(wr), torch.from_numpy(bias).cuda()
x0 = synth.normal_bf16(11, 1, 0, 0, (64, H))
y0 = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
pool.dx_moe_forward(0, bf16_dev(x0), 64, y0, router_w=wr_d, router_bias=b_d)
pool.dx_hotness_update(0)
pool.dx_plan_precision(0)
tab = pool.dx_get_table(0)
x = synth.normal_bf16(11, 2, T, 0, (T, H))
for rep in range(2):
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x), T, y, router_w=wr_d, router_bias=b_d)
    lg = pool.dx_get_logits(T)
    idx_o, gate_o = oracle.route(lg, k)
    Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, hb, lb, bool(tab["tier"][e])) for e in np.unique(idx_o)}
    _, y_o = oracle.moe_ffn(x, idx_o, gate_o, Wt, H, I, nthreads=16)
    yg = to_u16(y)
    cnt = np.bincount(idx_o.ravel(), minlength=E)
    yf = oracle.bits_to_f32(yg).astype(np.float64)
    of = oracle.bits_to_f32(y_o).astype(np.float64)
    den = np.abs(of).max()
    bad = [t for t in range(T) if np.abs(yf[t] - of[t]).max() / den > 2e-2]
    print(f"{shape} T={T} rep {rep}: rel err {rel_err(yg, y_o):.3e}; m_e of touched: {sorted(cnt[cnt > 0].tolist())}")
    if bad:
        ex = [set(idx_o[t].tolist()) for t in bad]
        common = set.intersection(*ex)
        print(f"  bad tokens {bad[:20]}; experts common to all bad tokens: {[(e, int(cnt[e]), int(tab['tier'][e])) for e in common]}")
        hcols = np.where(np.abs(yf[bad[0]] - of[bad[0]]) / den > 2e-2)[0]
        print(f"  bad h columns of token {bad[0]}: n={hcols.size} first {hcols[:8].tolist()} last {hcols[-4:].tolist()}")
pool.close()
