"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): bit-exact top-k indices, gates, hotness counters, EMA scores,
precision plans, tables and packed quantisation codes/scales/zeros; layer outputs within
max relative error 2e-2 (||y - y_ref||_inf / ||y_ref||_inf, DESIGN.md R-F1).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from dxtest import C1, Masters, budget_for, bf16_dev, canon_expected, elem_err, make_cfg, rel_err, to_u16

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def dx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_15015_b200 import dx as _dx
    return _dx


# ------------------------------------------------------------------ K8 quantiser
@pytest.mark.parametrize("N,K,g,bits", [(64, 64, 32, 4), (37, 256, 32, 2), (768, 2048, 128, 4),
                                        (2048, 768, 128, 4), (512, 2048, 128, 2), (33, 192, 64, 4)])
def test_quantize_dequantize_bitexact(dx, N, K, g, bits):
    w = synth.weights_bf16(9, N, K, bits, N, K)
    w[0, :g] = 0                                   # all-zero group
    w[1, 3] = 0x8000                               # -0.0
    wd = bf16_dev(w)
    codes = torch.zeros(N * K * bits // 8, dtype=torch.uint8, device="cuda")
    scales = torch.zeros(N * K // g, dtype=torch.int16, device="cuda")
    zeros = torch.zeros(N * K // g, dtype=torch.uint8, device="cuda")
    dx.dx_quantize(wd, N, K, g, bits, codes, scales, zeros)
    deq = torch.zeros(N * K, dtype=torch.int16, device="cuda")
    dx.dx_dequantize(codes, scales, zeros, N, K, g, bits, deq)
    torch.cuda.synchronize()
    c_o, s_o, z_o = oracle.quantize(w, g, bits)
    per = 8 // bits
    packed = codes.cpu().numpy()
    unpacked = np.stack([(packed >> (bits * i)) & ((1 << bits) - 1) for i in range(per)], 1).reshape(N, K)
    assert np.array_equal(unpacked, c_o)
    assert np.array_equal(scales.cpu().numpy().view(np.uint16).reshape(N, -1), s_o)
    assert np.array_equal(zeros.cpu().numpy().reshape(N, -1), z_o)
    assert np.array_equal(deq.cpu().numpy().view(np.uint16).reshape(N, K), oracle.dequantize(c_o, s_o, z_o, g))


# ------------------------------------------------------------------ C1 full replay
def _c1_pool(dx, seed=0, T=None, W=None):
    p = dict(C1)
    if T is not None:
        p["T"] = T
    if W is not None:
        p["W"] = W
    m = Masters(seed, p["L"], p["E"], p["H"], p["I"])
    budget = budget_for(p["E"], p["H"], p["I"], p["g"], p["high"], p["low"], p["n_hot"], p["s"])
    cfg = make_cfg(dx, p["L"], p["E"], p["k"], p["H"], p["I"], p["g"], p["high"], p["low"], budget, p["s"],
                   p["alpha"], p["Tp"], p["W"], p["dwell"], p["lag"], max_tokens=max(64, p["T"]))
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    return p, m, pool


def test_pool_create_low_images_bitexact(dx):
    p, m, pool = _c1_pool(dx)
    assert pool.info.n_hot == 2
    for e in range(p["E"]):
        got = pool.dx_export_expert(0, e)
        exp = canon_expected(m.get(0, e), p["H"], p["I"], p["g"], p["high"], p["low"], False)
        assert np.array_equal(got, exp), e
    pool.close()


def test_c1_replay_bitexact(dx):
    """300 steps of C1: routing, counters, EMA, plans, tables, exported images
    bit-exact at every step; y within 2e-2; at least 10 transitions."""
    p, m, pool = _c1_pool(dx)
    E, k, T, H, I, g = p["E"], p["k"], p["T"], p["H"], p["I"], p["g"]
    ctrl = oracle.Controller(E, pool.info.n_hot, p["s"], p["alpha"], p["Tp"], p["W"], p["dwell"], p["lag"])
    W_tier = {(e, th): oracle.expert_tier(m.get(0, e), H, I, g, p["high"], p["low"], th)
              for e in range(E) for th in (False, True)}
    y_dev = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    idx_dev = torch.zeros(T, k, dtype=torch.int32, device="cuda")
    gate_dev = torch.zeros(T, k, dtype=torch.float32, device="cuda")
    n_trans = 0
    worst = 0.0
    for step in range(300):
        lg = synth.trace_logits(0, 0, step, T, E, p["zipf"], p["drift"], p["frac"], n_top=4)
        x = synth.normal_bf16(0, 7, step, 0, (T, H))
        st = ctrl.state()
        idx_o, gate_o = oracle.route(lg, k)
        _, y_o = oracle.moe_ffn(x, idx_o, gate_o, {e: W_tier[(e, bool(st["tier"][e]))] for e in range(E)}, H, I)
        pool.dx_moe_forward(0, bf16_dev(x), T, y_dev, logits=torch.from_numpy(lg).cuda(), topk_idx=idx_dev,
                            topk_gate=gate_dev)
        assert np.array_equal(idx_dev.cpu().numpy(), idx_o), step
        assert np.array_equal(gate_dev.cpu().numpy().view(np.uint32), gate_o.view(np.uint32)), step
        err = rel_err(to_u16(y_dev), y_o)
        worst = max(worst, err)
        assert err <= TOL, (step, err)
        hot = pool.dx_get_hotness(0)
        cnt_o, mass_o = oracle.counts(idx_o, gate_o, E)
        assert np.array_equal(hot["cnt"], cnt_o) and np.array_equal(hot["mass"], mass_o), step
        pool.dx_hotness_update(0)
        ctrl.fold(mass_o, T)
        plan = pool.dx_plan_precision(0, want_plan=True)
        plan_o = ctrl.plan()
        assert plan[0] == (plan_o is not None), step
        if plan_o is not None:
            assert [(e, d, s) for e, d, s, _ in plan[4]] == plan_o[0], (step, plan[4], plan_o[0])
            if not plan_o[1]:
                n_trans += len(plan_o[0])
        tab = pool.dx_get_table(0)
        so = ctrl.state()
        assert np.array_equal(pool.dx_get_hotness(0)["S"].view(np.uint64), so["S"].view(np.uint64)), step
        for key in ("tier", "slot", "version", "in_flight"):
            assert np.array_equal(tab[key].astype(np.int64), so[key].astype(np.int64)), (step, key)
        if step % 10 == 0 or plan_o is not None:
            pool.dx_sync()
            for e in range(E):
                if so["in_flight"][e] == 0:
                    exp = canon_expected(m.get(0, e), H, I, g, p["high"], p["low"], bool(so["tier"][e]))
                    assert np.array_equal(pool.dx_export_expert(0, e), exp), (step, e)
    occ = pool.dx_occupancy(0)
    assert occ["used_hi"] <= occ["cap_hi"] and occ["used_lo"] <= occ["cap_lo"]
    assert n_trans >= 10, n_trans
    print(f"C1 replay: {n_trans} transitions, worst rel err {worst:.3e}")
    pool.close()


def test_manual_commands(dx):
    p, m, pool = _c1_pool(dx, W=0)
    pool.dx_plan_precision(0)                      # finalize at t = W = 0
    tab = pool.dx_get_table(0)
    hi = [e for e in range(p["E"]) if tab["tier"][e] == 1]
    lo = [e for e in range(p["E"]) if tab["tier"][e] == 0]
    assert len(hi) == 2
    assert pool.dx_promote(0, [hi[0]]) == dx.DX_ERR_INVALID_ARG      # already HIGH
    assert pool.dx_promote(0, [99]) == dx.DX_ERR_RANGE
    assert pool.dx_promote(0, [lo[0]]) == dx.DX_OK                   # uses the spare HIGH block
    assert pool.dx_promote(0, [lo[0]]) == dx.DX_ERR_BUSY
    assert pool.dx_promote(0, [lo[1]]) == dx.DX_ERR_POOL_EXHAUSTED   # s = 1 spare only
    for _ in range(p["lag"]):
        pool.dx_hotness_update(0)
    pool.dx_sync()
    assert pool.dx_query_expert(0, lo[0])[0] == 1
    exp = canon_expected(m.get(0, lo[0]), p["H"], p["I"], p["g"], p["high"], p["low"], True)
    assert np.array_equal(pool.dx_export_expert(0, lo[0]), exp)
    assert pool.dx_demote(0, [hi[0]]) == dx.DX_OK
    for _ in range(p["lag"]):
        pool.dx_hotness_update(0)
    pool.dx_sync()
    exp = canon_expected(m.get(0, hi[0]), p["H"], p["I"], p["g"], p["high"], p["low"], False)
    assert np.array_equal(pool.dx_export_expert(0, hi[0]), exp)
    pool.close()


def test_errors(dx):
    p = dict(C1)
    m = Masters(0, 1, p["E"], p["H"], p["I"])
    Sl = oracle.slot_bytes(p["H"], p["I"], p["g"], p["low"])
    cfg = make_cfg(dx, 1, p["E"], p["k"], p["H"], p["I"], p["g"], 16, 4, (p["E"] + 1) * Sl - 1, 1, 0.9, 8, 16,
                   16, 2, 64)
    with pytest.raises(dx.DxError) as ei:
        dx.Pool(cfg, m.ptrs())
    assert ei.value.code == dx.DX_ERR_INFEASIBLE_BUDGET
    unpinned = [np.zeros(3 * p["I"] * p["H"], np.uint16) for _ in range(p["E"])]
    cfg = make_cfg(dx, 1, p["E"], p["k"], p["H"], p["I"], p["g"], 16, 4, 10**9, 1, 0.9, 8, 16, 16, 2, 64)
    with pytest.raises(dx.DxError) as ei:
        dx.Pool(cfg, [a.ctypes.data for a in unpinned])
    assert ei.value.code == dx.DX_ERR_INVALID_ARG
    _, _, pool = _c1_pool(dx)
    y = torch.zeros(8, p["H"], dtype=torch.bfloat16, device="cuda")
    x = torch.zeros(8, p["H"], dtype=torch.bfloat16, device="cuda")
    with pytest.raises(dx.DxError) as ei:
        pool.dx_moe_forward(3, x, 8, y, logits=torch.zeros(8, p["E"], device="cuda"))
    assert ei.value.code == dx.DX_ERR_RANGE
    pool.dx_moe_forward(0, x, 0, y, logits=torch.zeros(8, p["E"], device="cuda"))      # T = 0: no-op
    idx = torch.tensor([[1, 1]] * 4, dtype=torch.int32, device="cuda")
    gate = torch.full((4, 2), 0.5, device="cuda")
    with pytest.raises(dx.DxError) as ei:
        pool.dx_hotness_update_from(0, idx, gate, 4)
    assert ei.value.code == dx.DX_ERR_INVALID_ARG                   # duplicate expert
    pool.close()


# ------------------------------------------------------------------ router mode
def test_router_mode_logits_and_routing(dx):
    p, m, pool = _c1_pool(dx)
    E, k, H, T = p["E"], p["k"], p["H"], 40
    wr = synth.router_bf16(0, 0, E, H)
    rank = synth.rank_perm(0, 0, 0, E, 4, 0.0)
    bias = synth.zipf_logp(rank, 1.2)
    x = synth.normal_bf16(0, 3, 0, 0, (T, H))
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(T, k, dtype=torch.int32, device="cuda")
    gate = torch.zeros(T, k, dtype=torch.float32, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x), T, y, router_w=bf16_dev(wr), router_bias=torch.from_numpy(bias).cuda(),
                        topk_idx=idx, topk_gate=gate)
    lg = oracle.router_logits(x, wr, bias)
    idx_o, _ = oracle.route(lg.astype(np.float32), k)
    srt = -np.sort(-lg, 1)
    margin = np.min(srt[:, :k] - srt[:, 1:k + 1], 1)
    clear = margin > 1e-4 * np.abs(lg).max()            # selections decided beyond fp32 accumulation noise
    assert clear.sum() >= T // 2
    assert np.array_equal(idx.cpu().numpy()[clear], idx_o[clear])
    pool.close()


# ------------------------------------------------------------------ Qwen3-30B / Qwen3-Next-80B shapes
_MASTERS = {}


def _masters_cached(seed, E, H, I):
    key = (seed, E, H, I)
    if key not in _MASTERS:
        _MASTERS.clear()
        _MASTERS[key] = Masters(seed, 1, E, H, I)
    return _MASTERS[key]


@pytest.mark.parametrize("path", [0, 1], ids=["tcgen05", "mma"])
@pytest.mark.parametrize("shape", ["q30b", "q80b"])
@pytest.mark.parametrize("T", [1, 64, 200])
def test_layer_parity_paper_shapes(dx, shape, T, path):
    if shape == "q30b":
        E, k, H, I, g, hb, lb = 128, 8, 2048, 768, 128, 16, 4
    else:
        E, k, H, I, g, hb, lb = 512, 10, 2048, 512, 128, 4, 2
    n_hot = E // 5
    m = _masters_cached(1, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, hb, lb, budget_for(E, H, I, g, hb, lb, n_hot, 1), 1, 0.95, 16, 1, 32,
                   4, 256)
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    pool.dx_set_ffn_path(path)
    assert pool.info.n_hot == n_hot
    # one warm-up step, then finalize: the top n_hot by the first step's mass go HIGH
    lg0 = synth.trace_logits(1, 0, 0, 64, E, 1.2)
    x0 = synth.normal_bf16(1, 0, 0, 0, (64, H))
    y = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x0), 64, y, logits=torch.from_numpy(lg0).cuda())
    pool.dx_hotness_update(0)
    pool.dx_plan_precision(0)
    tab = pool.dx_get_table(0)
    ctrl = oracle.Controller(E, n_hot, 1, 0.95, 16, 1, 32, 4)
    i0, g0 = oracle.route(lg0, k)
    ctrl.fold(oracle.counts(i0, g0, E)[1], 64)
    ctrl.plan()
    assert np.array_equal(tab["tier"], ctrl.state()["tier"])
    lg = synth.trace_logits(1, 0, 1, T, E, 1.2)
    x = synth.normal_bf16(1, 0, 1, 0, (T, H))
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(T, k, dtype=torch.int32, device="cuda")
    gate = torch.zeros(T, k, dtype=torch.float32, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x), T, y, logits=torch.from_numpy(lg).cuda(), topk_idx=idx, topk_gate=gate)
    idx_o, gate_o = oracle.route(lg, k)
    assert np.array_equal(idx.cpu().numpy(), idx_o)
    assert np.array_equal(gate.cpu().numpy(), gate_o)
    Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, hb, lb, bool(tab["tier"][e])) for e in np.unique(idx_o)}
    _, y_o = oracle.moe_ffn(x, idx_o, gate_o, Wt, H, I, nthreads=16)
    err = rel_err(to_u16(y[:T]), y_o)
    print(f"{shape} T={T}: rel err {err:.3e}")
    assert err <= TOL
    # exported images of a HIGH and a LOW expert are bit-exact
    for e in (int(np.flatnonzero(tab["tier"] == 1)[0]), int(np.flatnonzero(tab["tier"] == 0)[0])):
        exp = canon_expected(m.get(0, e), H, I, g, hb, lb, bool(tab["tier"][e]))
        assert np.array_equal(pool.dx_export_expert(0, e), exp)
    pool.close()


# ------------------------------------------------------------------ C3 size: T = 4096 with a plan period
def test_prefill_4096_with_plan_period(dx):
    """C3 launch configuration: one Q30B-shaped layer at T = 4096 (multi-block routing, the
    prefill GEMM configuration), warm-up -> finalize -> a plan period with promotions and demotions, and
    their publication.  Every step: top-k, gates, counters, EMA scores, plans and tables bit-exact; y of 96
    sampled token rows (incl. the first and last) <= 2e-2 at a warm-up step, the plan step and after
    publication."""
    E, k, H, I, g, T = 128, 8, 2048, 768, 128, 4096
    n_hot, s, alpha, Tp, W, dwell, lag = 26, 1, 0.95, 2, 2, 0, 1
    m = _masters_cached(4, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, n_hot, s), s, alpha, Tp, W, dwell,
                   lag, T)
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    ctrl = oracle.Controller(E, n_hot, s, alpha, Tp, W, dwell, lag)
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(T, k, dtype=torch.int32, device="cuda")
    gate = torch.zeros(T, k, dtype=torch.float32, device="cuda")
    rows = np.unique(np.concatenate([[0, T - 1], np.random.default_rng(0).choice(T, 94, replace=False)]))
    n_trans, checked = 0, 0
    for step in range(9):
        lg = synth.trace_logits(4, 0, step, T, E, 1.2, 2, 0.5, n_top=n_hot)
        x = synth.normal_bf16(4, 9, step, 0, (T, H))
        st_before = ctrl.state()
        pool.dx_moe_forward(0, bf16_dev(x), T, y, logits=torch.from_numpy(lg).cuda(), topk_idx=idx, topk_gate=gate)
        idx_o, gate_o = oracle.route(lg, k)
        assert np.array_equal(idx.cpu().numpy(), idx_o), step
        assert np.array_equal(gate.cpu().numpy().view(np.uint32), gate_o.view(np.uint32)), step
        hot = pool.dx_get_hotness(0)
        cnt_o, mass_o = oracle.counts(idx_o, gate_o, E)
        assert np.array_equal(hot["cnt"], cnt_o) and np.array_equal(hot["mass"], mass_o), step
        if step in (1, 4, 6):
            tiers = st_before["tier"]
            Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, 16, 4, bool(tiers[e]))
                  for e in np.unique(idx_o[rows])}
            _, y_o = oracle.moe_ffn(x[rows], idx_o[rows], gate_o[rows], Wt, H, I, nthreads=16)
            err = rel_err(to_u16(y)[rows], y_o)
            print(f"T=4096 step {step}: rel {err:.2e}, per-element (O-5) {elem_err(to_u16(y)[rows], y_o):.2e}")
            assert err <= TOL, (step, err)
            checked += 1
        pool.dx_hotness_update(0)
        ctrl.fold(mass_o, T)
        plan = pool.dx_plan_precision(0, want_plan=True)
        plan_o = ctrl.plan()
        assert plan[0] == (plan_o is not None), step
        if plan_o is not None:
            assert [(e, d, s_) for e, d, s_, _ in plan[4]] == plan_o[0], step
            if not plan_o[1]:
                n_trans += len(plan_o[0])
        so, tab = ctrl.state(), pool.dx_get_table(0)
        assert np.array_equal(pool.dx_get_hotness(0)["S"].view(np.uint64), so["S"].view(np.uint64)), step
        for key in ("tier", "slot", "version", "in_flight"):
            assert np.array_equal(tab[key].astype(np.int64), so[key].astype(np.int64)), (step, key)
    assert n_trans > 0 and checked == 3, n_trans
    pool.close()


# ------------------------------------------------------------------ Q80B runtime int4 -> int2 and back
def test_q80b_runtime_demotion_promotion_images(dx):
    """(int4, int2) pair: a runtime demotion re-quantises the int4 HIGH block to int2 on the
    device (k_xfer), a promotion streams the int4 image from the pinned cache; after publication both
    exported images are bit-exact to the oracle's path-independent images (R-Q2)."""
    E, k, H, I, g = 512, 10, 2048, 512, 128
    n_hot = E // 5
    m = _masters_cached(1, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, 4, 2, budget_for(E, H, I, g, 4, 2, n_hot, 1), 1, 0.95, 16, 0, 32, 4, 64)
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    pool.dx_plan_precision(0)                           # finalize at t = W = 0 (all S = 0: experts 0..n_hot-1)
    tab = pool.dx_get_table(0)
    hi = int(np.flatnonzero(tab["tier"] == 1)[3])
    lo = int(np.flatnonzero(tab["tier"] == 0)[5])
    assert pool.dx_demote(0, [hi]) == dx.DX_OK
    assert pool.dx_promote(0, [lo]) == dx.DX_OK
    for _ in range(4):
        pool.dx_hotness_update(0)
    pool.dx_sync()
    tab = pool.dx_get_table(0)
    assert tab["tier"][hi] == 0 and tab["tier"][lo] == 1
    for e, th in ((hi, False), (lo, True)):
        exp = canon_expected(m.get(0, e), H, I, g, 4, 2, th)
        assert np.array_equal(pool.dx_export_expert(0, e), exp), e
    pool.close()


# ------------------------------------------------------------------ dx_moe_step == forward + update + plan
@pytest.mark.parametrize("T,router", [(32, False), (24, True), (200, False)])
def test_moe_step_equals_three_calls(dx, T, router):
    """dx_moe_step (fold + publication fused into the combine launch) is bitwise the sequence
    dx_moe_forward + dx_hotness_update + dx_plan_precision: outputs, routing, EMA scores and tables at
    every step through warm-up, finalize, plan periods and publications."""
    p = dict(C1)
    E, k, H, I, g = p["E"], p["k"], p["H"], p["I"], p["g"]
    m = Masters(0, 1, E, H, I)
    budget = budget_for(E, H, I, g, 16, 4, 2, 1)
    pools = []
    for _ in range(2):
        cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget, 1, 0.9, 4, 4, 4, 2, T)
        pools.append(dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream()))
    wr = bf16_dev(synth.router_bf16(0, 0, E, H))
    ys = [torch.zeros(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    n_pub = 0
    for step in range(40):
        x = bf16_dev(synth.normal_bf16(0, 5, step, 0, (T, H)))
        lg = torch.from_numpy(synth.trace_logits(0, 0, step, T, E, 1.2, 4, 0.5, n_top=2)).cuda()
        kw = dict(router_w=wr) if router else dict(logits=lg)
        pools[0].dx_moe_forward(0, x, T, ys[0], **kw)
        pools[0].dx_hotness_update(0)
        pools[0].dx_plan_precision(0)
        pools[1].dx_moe_step(0, x, T, ys[1], **kw)
        assert torch.equal(ys[0].view(torch.int16), ys[1].view(torch.int16)), step
        h0, h1 = pools[0].dx_get_hotness(0), pools[1].dx_get_hotness(0)
        assert np.array_equal(h0["S"].view(np.uint64), h1["S"].view(np.uint64)) and h0["t"] == h1["t"], step
        t0, t1 = pools[0].dx_get_table(0), pools[1].dx_get_table(0)
        for key in ("tier", "slot", "version", "in_flight"):
            assert np.array_equal(t0[key], t1[key]), (step, key)
        n_pub += int(t0["version"].sum())
    assert n_pub > 0
    for pl in pools:
        pl.close()


def test_routed_bad_expert_is_reported(dx):
    """an out-of-range local expert id in dx_moe_forward_routed is routed with gate 0 and reported
    by the next dx_sync (sticky device error), instead of silently indexing past the tables."""
    E, k, H, I, g = 16, 2, 64, 128, 32
    m = Masters(0, 1, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(8, H, I, g, 16, 4, 2, 1), 1, 0.9, 8, 16, 16, 2, 16)
    cfg.ep_rank, cfg.ep_size = 0, 2
    pool = dx.Pool(cfg, m.ptrs()[:8], torch.cuda.current_stream())
    R = 6
    rows = torch.zeros(R, H, dtype=torch.bfloat16, device="cuda")
    meta = torch.tensor([[1, 0], [9, 0], [2, 0], [0, 0], [3, 0], [-1, 0]], dtype=torch.int32, device="cuda")
    meta[:, 1] = torch.tensor([0.5], dtype=torch.float32).view(torch.int32).item()
    yr = torch.zeros(R, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_forward_routed(0, rows, R, meta, yr, 6)
    with pytest.raises(dx.DxError) as ei:
        pool.dx_sync()
    assert ei.value.code == dx.DX_ERR_RANGE
    pool.dx_sync()                                       # the error is cleared once reported
    pool.close()
    # EP trace-mode counters count only this rank's experts (e_cnt = E_loc), for both ranks
    idx_np = np.array([[1, 9], [8, 15], [7, 0], [3, 12]], np.int32)
    gate_np = np.array([[0.75, 0.25], [0.5, 0.5], [0.625, 0.375], [0.875, 0.125]], np.float32)
    for r in range(2):
        cfg.ep_rank = r
        pool = dx.Pool(cfg, m.ptrs()[8 * r:8 * r + 8], torch.cuda.current_stream())
        S = np.zeros(8)
        for _ in range(2):
            pool.dx_hotness_update_from(0, torch.from_numpy(idx_np).cuda(), torch.from_numpy(gate_np).cuda(), 4)
            _, mass = oracle.counts(idx_np, gate_np, 8, e_lo=8 * r)
            S = oracle.ema_fold(S, mass, 4, 0.9)
        assert np.array_equal(pool.dx_get_hotness(0)["S"].view(np.uint64), S.view(np.uint64)), r
        pool.close()
