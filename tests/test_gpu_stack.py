"""GPU parity at BASELINE.json's full size, in the launch configuration bench.py times (C2):
the 48-layer Qwen3-30B-A3B-shaped stack (E=128, k=8, H=2048, I=768, g=128, bf16/int4) under the 24e9 B
expert budget, decode batch 64 (the tcgen05 decode GEMM configuration), controller Tp=16, W=32, dwell=16,
L=4 with a drifting Zipf(1.2) trace, run through warm-up, finalize, a plan period with promotions and
demotions, and their publication.

Checked against the CPU oracle: for two sampled layers at every step, top-k indices, gates, hotness
counters, EMA scores and the tier/slot/version table (bit-exact); at sampled steps, the layer output rows
of sampled tokens (the oracle computes them one by one) within 2e-2 (DESIGN.md R-F1)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from dxtest import Masters, bf16_dev, make_cfg, rel_err, to_u16

pytestmark = pytest.mark.gpu

TOL = 2e-2
C2 = dict(L=48, E=128, k=8, H=2048, I=768, g=128, high=16, low=4, budget=24 * 10**9, s=1, alpha=0.95, Tp=16,
          W=32, dwell=16, lag=4, B=64, zipf=1.2, drift=32, frac=0.25, n_top=24)
LAYERS = (0, 23, 47)          # sampled layers
Y_STEPS = (31, 40, 48, 53, 55)   # warm-up (all LOW), finalized, the plan step (old tiers), after publication
TOKENS = (0, 9, 21, 38, 50, 63)  # sampled token rows


@pytest.fixture(scope="module")
def dx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_15015_b200 import dx as _dx
    return _dx


def test_c2_stack_sampled_parity(dx):
    p = C2
    L, E, k, H, I, g, B = p["L"], p["E"], p["k"], p["H"], p["I"], p["g"], p["B"]
    m = Masters(3, L, E, H, I)
    cfg = make_cfg(dx, L, E, k, H, I, g, p["high"], p["low"], p["budget"], p["s"], p["alpha"], p["Tp"], p["W"],
                   p["dwell"], p["lag"], B)
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    n_hot = pool.info.n_hot
    assert n_hot == 24                                   # 24e9 B, s = 1
    ctrl = {l: oracle.Controller(E, n_hot, p["s"], p["alpha"], p["Tp"], p["W"], p["dwell"], p["lag"]) for l in LAYERS}
    y = torch.zeros(L, B, H, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(L, B, k, dtype=torch.int32, device="cuda")
    gate = torch.zeros(L, B, k, dtype=torch.float32, device="cuda")
    n_trans = {l: 0 for l in LAYERS}
    worst = 0.0
    for step in range(p["W"] + 24):
        lgs, xs, st_before = {}, {}, {}
        for l in range(L):
            lg = synth.trace_logits(3, l, step, B, E, p["zipf"], p["drift"], p["frac"], n_top=p["n_top"])
            x = synth.normal_bf16(3, 50 + l, step, 0, (B, H))
            if l in LAYERS:
                lgs[l], xs[l], st_before[l] = lg, x, ctrl[l].state()
            pool.dx_moe_forward(l, bf16_dev(x), B, y[l], logits=torch.from_numpy(lg).cuda(), topk_idx=idx[l],
                                topk_gate=gate[l])
            if l in LAYERS:
                hot = pool.dx_get_hotness(l)
            pool.dx_hotness_update(l)
            plan = pool.dx_plan_precision(l, want_plan=l in LAYERS)
            if l not in LAYERS:
                continue
            idx_o, gate_o = oracle.route(lgs[l], k)
            assert np.array_equal(idx[l].cpu().numpy(), idx_o), (step, l)
            assert np.array_equal(gate[l].cpu().numpy().view(np.uint32), gate_o.view(np.uint32)), (step, l)
            cnt_o, mass_o = oracle.counts(idx_o, gate_o, E)
            assert np.array_equal(hot["cnt"], cnt_o) and np.array_equal(hot["mass"], mass_o), (step, l)
            ctrl[l].fold(mass_o, B)
            plan_o = ctrl[l].plan()
            assert plan[0] == (plan_o is not None), (step, l)
            if plan_o is not None:
                assert [(e, d, s) for e, d, s, _ in plan[4]] == plan_o[0], (step, l)
                if not plan_o[1]:
                    n_trans[l] += len(plan_o[0])
            so, tab = ctrl[l].state(), pool.dx_get_table(l)
            assert np.array_equal(pool.dx_get_hotness(l)["S"].view(np.uint64), so["S"].view(np.uint64)), (step, l)
            for key in ("tier", "slot", "version", "in_flight"):
                assert np.array_equal(tab[key].astype(np.int64), so[key].astype(np.int64)), (step, l, key)
            if step in Y_STEPS:
                # the forward of this step used the tiers stable at its start
                tiers = st_before[l]["tier"]
                rows = list(TOKENS)
                used = np.unique(idx_o[rows])
                Wt = {int(e): oracle.expert_tier(m.get(l, int(e)), H, I, g, p["high"], p["low"], bool(tiers[e]))
                      for e in used}
                _, y_o = oracle.moe_ffn(xs[l][rows], idx_o[rows], gate_o[rows], Wt, H, I, nthreads=16)
                err = rel_err(to_u16(y[l])[rows], y_o)
                worst = max(worst, err)
                assert err <= TOL, (step, l, err)
    pool.dx_sync()
    assert all(v > 0 for v in n_trans.values()), n_trans
    print(f"C2 stack: transitions at sampled layers {n_trans}, worst sampled rel err {worst:.3e}")
    pool.close()


def test_c2_stack_layers_entry_matches_per_layer_calls(dx):
    """The bench's entry point -- dx_moe_step_layers over the 48 layers in router mode -- against
    48 separate dx_moe_step calls on a second pool fed the same steps: every layer's output, every step, bitwise,
    and the controller state (scores and tables) of every layer at the end, through warm-up, finalize and a plan
    period with copy-engine promotions."""
    p = C2
    L, E, k, H, I, g, B = p["L"], p["E"], p["k"], p["H"], p["I"], p["g"], p["B"]
    m = Masters(4, L, E, H, I)
    cfg = make_cfg(dx, L, E, k, H, I, g, p["high"], p["low"], p["budget"], p["s"], p["alpha"], p["Tp"], p["W"],
                   p["dwell"], p["lag"], B)
    pa = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    pb = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    wr = torch.stack([bf16_dev(synth.router_bf16(4, l, E, H)) for l in range(L)])
    bias = torch.stack([torch.from_numpy(synth.zipf_logp(synth.rank_perm(4, l, 0, E, 24, 0.25), 1.2)) for l in range(L)]).cuda()
    ya = torch.zeros(L, B, H, dtype=torch.bfloat16, device="cuda")
    yb = torch.zeros(L, B, H, dtype=torch.bfloat16, device="cuda")
    P = dx.Pool.ptr_array
    y_arr, wr_arr, b_arr = P([ya[l] for l in range(L)]), P([wr[l] for l in range(L)]), P([bias[l] for l in range(L)])
    for step in range(p["W"] + 22):
        x = bf16_dev(synth.normal_bf16(4, 7, step, 0, (B, H)))
        pa.dx_moe_step_layers(0, L, P([x] * L), B, y_arr, router_w_arr=wr_arr, router_bias_arr=b_arr)
        for l in range(L):
            pb.dx_moe_step(l, x, B, yb[l], router_w=wr[l], router_bias=bias[l])
        assert torch.equal(ya.view(torch.int16), yb.view(torch.int16)), step
    pa.dx_sync()
    pb.dx_sync()
    for l in range(L):
        ha, hb = pa.dx_get_hotness(l), pb.dx_get_hotness(l)
        assert np.array_equal(ha["S"].view(np.uint64), hb["S"].view(np.uint64)), l
        ta, tb = pa.dx_get_table(l), pb.dx_get_table(l)
        for key in ("tier", "slot", "version"):
            assert np.array_equal(ta[key], tb[key]), (l, key)
    assert int(sum(pa.dx_get_table(l)["version"].sum() for l in range(L))) > 0      # transitions happened
    pa.close()
    pb.close()
