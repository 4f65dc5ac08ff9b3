"""GPU parity of f-1, cross-layer correlation prefetch, through the C ABI against
the oracle (or_corr_update, or_prefetch_candidates, the controller replay):
- the per-layer-pair correlation counts (dx_get_corr) bit-exact at every step;
- every prefetch decision (dx_get_prefetch: experts and the HIGH blocks they are staged into) equal to the
  oracle's candidates from the same counts, the same routing and the oracle controller's state;
- results unchanged: routing, controller state and y (<= 2e-2) as without prefetch, and on a coupled trace the
  plans' promotions hit staged images (dx_profile_t prefetch_hits > 0)."""
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


def test_prefetch_parity_and_hits(dx):
    L, E, k, H, I, g, T = 3, 16, 2, 256, 128, 64, 24
    n_hot, s, alpha, Tp, W, dwell, lag, f, lead = 4, 1, 0.9, 4, 4, 4, 1, 2, 2
    m = Masters(9, L, E, H, I)
    cfg = make_cfg(dx, L, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, n_hot, s, L), s, alpha, Tp, W, dwell,
                   lag, T)
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    pool.dx_set_prefetch(f, lead)
    ctrl = [oracle.Controller(E, n_hot, s, alpha, Tp, W, dwell, lag) for _ in range(L)]
    corr = [np.zeros((E, E), np.uint32) for _ in range(L - 1)]
    pool.dx_profile_enable(True)
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    idx_d = torch.zeros(T, k, dtype=torch.int32, device="cuda")
    gate_d = torch.zeros(T, k, dtype=torch.float32, device="cuda")
    decisions = hits = 0
    worst = 0.0
    for step in range(44):
        lgs = synth.coupled_trace_logits(9, L, step, T, E, k)
        x = synth.normal_bf16(9, 3, step, 0, (T, H))
        prev_idx = None
        for l in range(L):
            st = ctrl[l].state()
            pool.dx_moe_step(l, bf16_dev(x), T, y, logits=torch.from_numpy(lgs[l]).cuda(), topk_idx=idx_d,
                             topk_gate=gate_d)
            idx_o, gate_o = oracle.route(lgs[l], k)
            assert np.array_equal(idx_d.cpu().numpy(), idx_o), (step, l)
            Wt = {int(e): oracle.expert_tier(m.get(l, int(e)), H, I, g, 16, 4, bool(st["tier"][e])) for e in np.unique(idx_o)}
            _, y_o = oracle.moe_ffn(x, idx_o, gate_o, Wt, H, I, nthreads=8)
            err = rel_err(to_u16(y), y_o)
            worst = max(worst, err)
            assert err <= 2e-2, (step, l, err)
            # the prefetch decision for layer l+1, made right after layer l's routing (its counts include the
            # previous steps only: pair (l, l+1) is counted at layer l+1's forward)
            nl = l + 1
            if nl < L:
                sn = ctrl[nl].state()
                if sn["t"] > W and (sn["t"] + lead) % Tp == 0 and not sn["in_flight"].any():
                    own = np.array([ctrl[nl].owner(True, b) for b in range(sn["cap_hi"])], np.int32)
                    exp = oracle.prefetch_candidates(corr[l], idx_o, sn["tier"], sn["in_flight"], own, f)
                    assert pool.dx_get_prefetch(nl) == exp, (step, l, exp)
                    decisions += 1
            if prev_idx is not None:
                oracle.corr_update(corr[l - 1], prev_idx, idx_o)
            prev_idx = idx_o
            _, mass = oracle.counts(idx_o, gate_o, E)
            ctrl[l].fold(mass, T)
            ctrl[l].plan()
            so, tab = ctrl[l].state(), pool.dx_get_table(l)
            for key in ("tier", "slot", "version", "in_flight"):
                assert np.array_equal(tab[key].astype(np.int64), so[key].astype(np.int64)), (step, l, key)
        for l in range(L - 1):
            assert np.array_equal(pool.dx_get_corr(l), corr[l]), (step, l)
    pool.dx_sync()
    pr = pool.dx_profile_read()
    hits, issued = pr["prefetch_hits"], pr["prefetch_issued"]
    print(f"prefetch: {decisions} decisions checked, {issued} images staged, {hits} promotion hits, "
          f"{pr['promotions']} promotions; worst rel err {worst:.2e}")
    assert decisions > 0 and issued > 0 and hits > 0
    pool.close()
