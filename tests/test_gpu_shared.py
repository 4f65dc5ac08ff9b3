"""GPU parity of f-3, the shared expert of Eq. 1 (first sum; DESIGN.md R-S1), through the C ABI:
y = bf16(E^s(x) + sum_j g_j E_j(x)) against the oracle (or_shared_ffn + the routed oracle + or_combine_shared)
within 2e-2 at the two precision pairs (bf16/int4 and int4/int2: the shared expert at the HIGH tier), decode and
prefill token counts, router and trace mode; and a pool whose shared expert is all zeros bitwise equal to a pool
without one (the shared term enters the combine exactly once, first)."""
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


def _pool(dx, m, shared_ptrs, E, k, H, I, g, hb, lb, n_hot, T):
    cfg = make_cfg(dx, 1, E, k, H, I, g, hb, lb, budget_for(E, H, I, g, hb, lb, n_hot, 1), 1, 0.95, 16, 1, 32, 4,
                   max(T, 64))
    cfg.n_shared = 1 if shared_ptrs is not None else 0
    ptrs = m.ptrs() + (list(shared_ptrs) if shared_ptrs is not None else [])
    return dx.Pool(cfg, ptrs, torch.cuda.current_stream())


@pytest.mark.parametrize("shape", ["q30b", "q80b"])
@pytest.mark.parametrize("T", [1, 48, 300])
def test_shared_expert_layer(dx, shape, T):
    if shape == "q30b":
        E, k, H, I, g, hb, lb = 32, 8, 2048, 768, 128, 16, 4
    else:
        E, k, H, I, g, hb, lb = 64, 10, 2048, 512, 128, 4, 2
    n_hot = E // 4
    m = Masters(13, 1, E, H, I)
    sh = torch.empty(3 * I * H, dtype=torch.int16, pin_memory=True)
    sh.numpy().view(np.uint16)[:] = synth.expert_master(13, 0, E + 7, H, I)      # a distinct seeded expert
    pool = _pool(dx, m, [sh.data_ptr()], E, k, H, I, g, hb, lb, n_hot, T)
    x0 = synth.normal_bf16(13, 0, 0, 0, (64, H))
    y0 = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x0), 64, y0, logits=torch.from_numpy(synth.trace_logits(13, 0, 0, 64, E, 1.2)).cuda())
    pool.dx_hotness_update(0)
    pool.dx_plan_precision(0)                                   # finalize: HIGH / LOW mix
    tab = pool.dx_get_table(0)
    x = synth.normal_bf16(13, 1, T, 0, (T, H))
    lg = synth.trace_logits(13, 0, 1, T, E, 1.2)
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x), T, y, logits=torch.from_numpy(lg).cuda())
    idx_o, gate_o = oracle.route(lg, k)
    Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, hb, lb, bool(tab["tier"][e])) for e in np.unique(idx_o)}
    Ws = oracle.expert_tier(sh.numpy().view(np.uint16), H, I, g, hb, lb, True)  # the shared expert at the HIGH tier
    _, _, y_o = oracle.moe_ffn_shared(x, idx_o, gate_o, Wt, Ws, H, I, nthreads=16)
    err = rel_err(to_u16(y), y_o)
    print(f"shared expert {shape} T={T}: rel err {err:.2e}")
    assert err <= 2e-2
    pool.close()


def test_zero_shared_expert_is_bitwise_the_plain_layer(dx):
    E, k, H, I, g, T = 16, 4, 256, 128, 64, 40
    m = Masters(14, 1, E, H, I)
    zero = torch.zeros(3 * I * H, dtype=torch.int16, pin_memory=True)
    a = _pool(dx, m, [zero.data_ptr()], E, k, H, I, g, 16, 4, 4, T)
    b = _pool(dx, m, None, E, k, H, I, g, 16, 4, 4, T)
    wr = bf16_dev(synth.router_bf16(14, 0, E, H))
    for step in range(40):
        x = bf16_dev(synth.normal_bf16(14, 2, step, 0, (T, H)))
        ya = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
        yb = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
        a.dx_moe_step(0, x, T, ya, router_w=wr)
        b.dx_moe_step(0, x, T, yb, router_w=wr)
        assert torch.equal(ya.view(torch.int16), yb.view(torch.int16)), step
    ta, tb = a.dx_get_table(0), b.dx_get_table(0)
    assert np.array_equal(ta["tier"], tb["tier"]) and np.array_equal(ta["version"], tb["version"])
    a.close()
    b.close()
