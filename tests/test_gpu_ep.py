"""Expert parallelism on one GPU: G pools (ep_rank r of ep_size G) in one process, the all-to-all done by
tensor copies (paper_2511_15015_b200.ep.ep_forward_local), against the oracle and against the G = 1 path.

Bars: owner-side counters and EMA scores bit-exact to the oracle over the GLOBAL batch;
y within 2e-2 of the oracle; while every expert is LOW (warm-up) y is bitwise equal to the single-pool
dx_moe_forward of the same global batch.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from dxtest import Masters, bf16_dev, budget_for, make_cfg, rel_err, to_u16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_15015_b200 import dx as _dx
    return _dx


@pytest.mark.parametrize("G", [2, 4])
def test_ep_local_matches_oracle_and_single_gpu(dx, G):
    from paper_2511_15015_b200 import ep
    E, k, H, I, g, T, W = 16, 4, 256, 128, 64, 24, 3
    e_loc = E // G
    n_hot_loc = max(1, e_loc // 4)
    m = Masters(5, 1, E, H, I)
    ptrs = m.ptrs()
    pools, bufs = [], []
    for r in range(G):
        cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(e_loc, H, I, g, 16, 4, n_hot_loc, 1), 1, 0.9, 2, W,
                       2, 1, T)
        cfg.ep_rank, cfg.ep_size = r, G
        pools.append(dx.Pool(cfg, ptrs[r * e_loc:(r + 1) * e_loc], torch.cuda.current_stream()))
        bufs.append(ep.EPBuffers(T, k, H, G, e_loc, "cuda"))
    cfg1 = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, G * n_hot_loc, 1), 1, 0.9, 2, W, 2, 1,
                    G * T)
    single = dx.Pool(cfg1, ptrs, torch.cuda.current_stream())
    ctrls = [oracle.Controller(e_loc, pools[r].info.n_hot, 1, 0.9, 2, W, 2, 1) for r in range(G)]
    ys = [torch.zeros(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(G)]
    y1 = torch.zeros(G * T, H, dtype=torch.bfloat16, device="cuda")
    for step in range(8):
        lgs = [synth.trace_logits(5, 0, step * G + r, T, E, 1.2) for r in range(G)]
        xs = [synth.normal_bf16(5, 1, step * G + r, 0, (T, H)) for r in range(G)]
        tabs = [pools[r].dx_get_table(0) for r in range(G)]
        ep.ep_forward_local(pools, bufs, 0, [bf16_dev(x) for x in xs], [T] * G, ys,
                            logits_list=[torch.from_numpy(lg).cuda() for lg in lgs])
        lg_all, x_all = np.concatenate(lgs), np.concatenate(xs)
        idx_o, gate_o = oracle.route(lg_all, k)
        tier_of = {r * e_loc + e: bool(tabs[r]["tier"][e]) for r in range(G) for e in range(e_loc)}
        Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, 16, 4, tier_of[int(e)]) for e in np.unique(idx_o)}
        _, y_o = oracle.moe_ffn(x_all, idx_o, gate_o, Wt, H, I, nthreads=8)
        y_ep = np.concatenate([to_u16(y) for y in ys])
        assert rel_err(y_ep, y_o) <= 2e-2, step
        cnt_all, mass_all = oracle.counts(idx_o, gate_o, E)
        for r in range(G):
            hot = pools[r].dx_get_hotness(0)
            assert np.array_equal(hot["cnt"], cnt_all[r * e_loc:(r + 1) * e_loc]), (step, r)
            assert np.array_equal(hot["mass"], mass_all[r * e_loc:(r + 1) * e_loc]), (step, r)
        if step < W:     # all LOW on both sides: EP is bitwise the single-GPU layer
            single.dx_moe_forward(0, bf16_dev(x_all), G * T, y1, logits=torch.from_numpy(lg_all).cuda())
            assert np.array_equal(to_u16(y1), y_ep), step
            single.dx_hotness_update(0)
        for r in range(G):
            pools[r].dx_hotness_update(0)
            pools[r].dx_plan_precision(0)
            ctrls[r].fold(mass_all[r * e_loc:(r + 1) * e_loc], G * T)
            ctrls[r].plan()
            st = ctrls[r].state()
            hot = pools[r].dx_get_hotness(0)
            assert np.array_equal(hot["S"].view(np.uint64), st["S"].view(np.uint64)), (step, r)
            tab = pools[r].dx_get_table(0)
            assert np.array_equal(tab["tier"], st["tier"]) and np.array_equal(tab["slot"], st["slot"]), (step, r)
    for p in pools:
        p.close()
    single.close()


@pytest.mark.parametrize("router", [False, True], ids=["trace", "router"])
def test_ep_nccl_loopback_matches_single_pool(dx, router):
    """The in-library NCCL expert-parallel layer (dx_pool_create_ep, SURVEY §8(e) collective v1) on a one-rank
    communicator: dispatch, NCCL count exchange + host sync, grouped send/recv of rows and metadata (to self),
    owner-side FFN, return exchange, combine -- through dx_moe_step over warm-up, finalize, plan periods with
    transitions and their publication.  Routing, counters, EMA scores, plans and tables must be bit-exact to a
    plain pool fed the same steps; y within 2e-2 of the oracle (the owner side runs the grouped GEMMs on T*k
    k=1 rows, i.e. another tile configuration than the plain pool's)."""
    E, k, H, I, g, T, W, Tp = 16, 4, 256, 128, 64, 24, 3, 2
    n_hot = 4
    m = Masters(7, 1, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, n_hot, 1), 1, 0.9, Tp, W, 2, 1, T)
    nid = dx.dx_get_unique_id()
    ep_pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream(), nccl_id=nid)
    plain = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    wr = synth.router_bf16(7, 0, E, H)
    wr_d = bf16_dev(wr)
    for step in range(14):
        x = synth.normal_bf16(7, 1, step, 0, (T, H))
        lg = synth.trace_logits(7, 0, step, T, E, 1.2)
        kw = dict(router_w=wr_d) if router else dict(logits=torch.from_numpy(lg).cuda())
        tab = plain.dx_get_table(0)
        outs = []
        for p in (ep_pool, plain):
            y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
            idx = torch.zeros(T, k, dtype=torch.int32, device="cuda")
            gate = torch.zeros(T, k, dtype=torch.float32, device="cuda")
            p.dx_moe_step(0, bf16_dev(x), T, y, topk_idx=idx, topk_gate=gate, **kw)
            outs.append((to_u16(y), idx.cpu().numpy(), gate.cpu().numpy()))
        (y_ep, i_ep, g_ep), (y_pl, i_pl, g_pl) = outs
        assert np.array_equal(i_ep, i_pl) and np.array_equal(g_ep.view(np.uint32), g_pl.view(np.uint32)), step
        Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, 16, 4, bool(tab["tier"][e])) for e in np.unique(i_pl)}
        _, y_o = oracle.moe_ffn(x, i_pl, g_pl, Wt, H, I, nthreads=8)
        assert rel_err(y_ep, y_o) <= 2e-2 and rel_err(y_pl, y_o) <= 2e-2, step
        h_ep, h_pl = ep_pool.dx_get_hotness(0), plain.dx_get_hotness(0)
        assert np.array_equal(h_ep["S"].view(np.uint64), h_pl["S"].view(np.uint64)), step
        assert h_ep["t"] == h_pl["t"] == step + 1
        t_ep, t_pl = ep_pool.dx_get_table(0), plain.dx_get_table(0)
        for key in ("tier", "slot", "version", "in_flight"):
            assert np.array_equal(t_ep[key], t_pl[key]), (step, key)
    transitions = int(np.sum(plain.dx_get_table(0)["version"]))
    ep_pool.dx_sync()
    plain.dx_sync()
    assert transitions > 0
    ep_pool.close()
    plain.close()


@pytest.mark.parametrize("G", [2, 4])
def test_ep_local_group_dedup_in_library(dx, G):
    """The in-library EP layer (the same code as the NCCL path, f-2 deduplicated dispatch) for G ranks' pools in one
    process (dx_moe_step_group: the exchange by device copies): owner-side counters and EMA scores bit-exact to the
    oracle over the global batch, plans and tables equal to the oracle controller per rank, y within 2e-2 of the
    oracle, bitwise equal to a single pool while every expert is LOW; and fewer x rows sent than dispatch entries."""
    E, k, H, I, g, T, W = 16, 4, 256, 128, 64, 24, 3
    e_loc = E // G
    n_hot_loc = max(1, e_loc // 4)
    m = Masters(6, 1, E, H, I)
    ptrs = m.ptrs()
    pools = []
    for r in range(G):
        cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(e_loc, H, I, g, 16, 4, n_hot_loc, 1), 1, 0.9, 2, W, 2, 1, T)
        cfg.ep_rank, cfg.ep_size = r, G
        pools.append(dx.Pool(cfg, ptrs[r * e_loc:(r + 1) * e_loc], torch.cuda.current_stream(), nccl_id=b"local"))
    cfg1 = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, G * n_hot_loc, 1), 1, 0.9, 2, W, 2, 1,
                    G * T)
    single = dx.Pool(cfg1, ptrs, torch.cuda.current_stream())
    ctrls = [oracle.Controller(e_loc, pools[r].info.n_hot, 1, 0.9, 2, W, 2, 1) for r in range(G)]
    ys = [torch.zeros(T, H, dtype=torch.bfloat16, device="cuda") for _ in range(G)]
    y1 = torch.zeros(G * T, H, dtype=torch.bfloat16, device="cuda")
    for step in range(10):
        lgs = [synth.trace_logits(6, 0, step * G + r, T, E, 1.2) for r in range(G)]
        xs = [synth.normal_bf16(6, 1, step * G + r, 0, (T, H)) for r in range(G)]
        tabs = [pools[r].dx_get_table(0) for r in range(G)]
        xd = [bf16_dev(x) for x in xs]
        dx.dx_moe_step_group(pools, 0, xd, [T] * G, ys, logits=[torch.from_numpy(lg).cuda() for lg in lgs])
        lg_all, x_all = np.concatenate(lgs), np.concatenate(xs)
        idx_o, gate_o = oracle.route(lg_all, k)
        tier_of = {r * e_loc + e: bool(tabs[r]["tier"][e]) for r in range(G) for e in range(e_loc)}
        Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, 16, 4, tier_of[int(e)]) for e in np.unique(idx_o)}
        _, y_o = oracle.moe_ffn(x_all, idx_o, gate_o, Wt, H, I, nthreads=8)
        y_ep = np.concatenate([to_u16(y) for y in ys])
        assert rel_err(y_ep, y_o) <= 2e-2, step
        if step < W:                       # all LOW on both sides: bitwise the single-pool layer
            single.dx_moe_forward(0, bf16_dev(x_all), G * T, y1, logits=torch.from_numpy(lg_all).cuda())
            single.dx_hotness_update(0)
            assert np.array_equal(to_u16(y1), y_ep), step
        _, mass_all = oracle.counts(idx_o, gate_o, E)
        for r in range(G):
            ctrls[r].fold(mass_all[r * e_loc:(r + 1) * e_loc], G * T)
            ctrls[r].plan()
            st = ctrls[r].state()
            hot = pools[r].dx_get_hotness(0)
            assert np.array_equal(hot["S"].view(np.uint64), st["S"].view(np.uint64)), (step, r)
            tab = pools[r].dx_get_table(0)
            assert np.array_equal(tab["tier"], st["tier"]) and np.array_equal(tab["slot"], st["slot"]), (step, r)
    tr = [p.dx_ep_traffic() for p in pools]
    rows, ents = sum(t["rows_sent"] for t in tr), sum(t["entries_sent"] for t in tr)
    print(f"EP local group G={G}: {rows} x rows sent for {ents} dispatch entries ({ents / max(rows, 1):.2f}x fewer)")
    assert ents == 10 * G * T * k and rows < ents
    for p in pools:
        p.close()
    single.close()
