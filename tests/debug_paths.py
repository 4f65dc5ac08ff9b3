"""Diagnostic (not collected by pytest): per-configuration error of the tcgen05 and mma.sync FFN paths
against the oracle, printed rather than asserted.  python tests/debug_paths.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle  # noqa: E402
import synth  # noqa: E402
from dxtest import Masters, bf16_dev, budget_for, make_cfg, rel_err, to_u16  # noqa: E402
from paper_2511_15015_b200 import dx  # noqa: E402


def run(name, E, k, H, I, g, hb, lb, n_hot, T, finalize):
    m = Masters(3, 1, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, hb, lb, budget_for(E, H, I, g, hb, lb, n_hot, 1), 1, 0.9, 8, 1, 8, 2, 256)
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    lg = synth.trace_logits(3, 0, 0, T, E, 1.2)
    x = synth.normal_bf16(3, 0, 0, 0, (T, H))
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    if finalize:
        pool.dx_moe_forward(0, bf16_dev(x), T, y, logits=torch.from_numpy(lg).cuda())
        pool.dx_hotness_update(0)
        pool.dx_plan_precision(0)
    tab = pool.dx_get_table(0)
    idx_o, gate_o = oracle.route(lg, k)
    W = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, hb, lb, bool(tab["tier"][e])) for e in np.unique(idx_o)}
    _, y_o = oracle.moe_ffn(x, idx_o, gate_o, W, H, I, nthreads=16)
    outs = {}
    for path in (1, 0):
        pool.dx_set_ffn_path(path)
        y.zero_()
        pool.dx_moe_forward(0, bf16_dev(x), T, y, logits=torch.from_numpy(lg).cuda())
        torch.cuda.synchronize()
        outs[path] = to_u16(y)
    e1, e0 = rel_err(outs[1], y_o), rel_err(outs[0], y_o)
    d = np.abs(oracle.bits_to_f32(outs[0]).astype(np.float64) - oracle.bits_to_f32(y_o))
    bad = np.argwhere(d > 0.05 * np.abs(oracle.bits_to_f32(y_o)).max())
    print(f"{name:28s} hiHIGH={int(tab['tier'].sum()):3d} mma={e1:.2e} tcgen05={e0:.2e} bad={len(bad)} "
          f"first_bad={bad[:4].tolist()}", flush=True)
    pool.close()


if __name__ == "__main__":
    run("c1 low T=32", 8, 2, 64, 128, 32, 16, 4, 2, 32, False)
    run("c1 mixed T=32", 8, 2, 64, 128, 32, 16, 4, 2, 32, True)
    run("small g128 low T=8", 8, 2, 256, 128, 128, 16, 4, 2, 8, False)
    run("small g128 mixed T=8", 8, 2, 256, 128, 128, 16, 4, 2, 8, True)
    run("small g128 all-high T=8", 8, 2, 256, 128, 128, 16, 4, 8, 8, True)
    run("q30b low T=64", 128, 8, 2048, 768, 128, 16, 4, 24, 64, False)
    run("q30b mixed T=64", 128, 8, 2048, 768, 128, 16, 4, 24, 64, True)
    run("q30b mixed T=200", 128, 8, 2048, 768, 128, 16, 4, 24, 200, True)
    run("q30b mixed T=1", 128, 8, 2048, 768, 128, 16, 4, 24, 1, True)
    run("q80b mixed T=64", 512, 10, 2048, 512, 128, 4, 2, 128, 64, True)
