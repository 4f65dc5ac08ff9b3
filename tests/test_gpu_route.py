"""GPU parity of the routing steps on the benched path (router mode, fused decode routing kernel) and their
edge cases, through the C ABI, against the CPU oracle.

- a1 router logits (the fused decode kernel for T*k <= 512, the tiled prefill router otherwise): the GPU's fp32
  logits (dx_get_logits = exactly what its top-k consumed) against the fp64
  oracle (or_router_logits) element by element, within the fp32 summation bound gamma_n * sum|x w| (n = H),
  and row-wise max |d| / max |ref| <= 1e-3, at C2 / Q80B sizes.
- a2-a8 in router mode: the oracle routes the GPU's own logits; idx / gates / counters bit-exact, y <= 2e-2.
- Edge cases (R-G1, R-G3): all-equal and pairwise-tied logits, +-0, -inf (masked) entries, k = 1 (gate 1.0),
  on the fused decode kernel (T*k <= 512) and the multi-block prefill kernels (T*k > 512).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from dxtest import Masters, bf16_dev, budget_for, dot_bound, elem_err, make_cfg, rel_err, to_u16

pytestmark = pytest.mark.gpu
TOL = 2e-2


@pytest.fixture(scope="module")
def dx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2511_15015_b200 import dx as _dx
    return _dx


_M = {}


def _masters(seed, E, H, I):
    key = (seed, E, H, I)
    if key not in _M:
        _M.clear()
        _M[key] = Masters(seed, 1, E, H, I)
    return _M[key]


def _shape(name):
    if name == "q30b":
        return dict(E=128, k=8, H=2048, I=768, g=128, hb=16, lb=4)
    return dict(E=512, k=10, H=2048, I=512, g=128, hb=4, lb=2)


@pytest.mark.parametrize("shape,T", [("q30b", 64), ("q30b", 1), ("q30b", 37), ("q80b", 51), ("q80b", 64),
                                     ("q30b", 300), ("q80b", 200)])
def test_router_mode_logits_and_layer(dx, shape, T):
    s = _shape(shape)
    E, k, H, I, g, hb, lb = s["E"], s["k"], s["H"], s["I"], s["g"], s["hb"], s["lb"]
    n_hot = E // 5
    m = _masters(11, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, hb, lb, budget_for(E, H, I, g, hb, lb, n_hot, 1), 1, 0.95, 16, 1, 32, 4,
                   max(T, 64))
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    wr = synth.router_bf16(11, 0, E, H)
    wr = ((oracle.bits_to_f32(wr) * np.float32(3.0)).view(np.uint32) >> 16).astype(np.uint16)  # x3 spread
    bias = synth.zipf_logp(synth.rank_perm(11, 0, 0, E, n_hot, 0.0), 1.2)
    wr_d, b_d = bf16_dev(wr), torch.from_numpy(bias).cuda()
    # warm-up step (router mode) then finalize: a HIGH/LOW mix for the measured step
    x0 = synth.normal_bf16(11, 1, 0, 0, (64, H))
    y0 = torch.zeros(64, H, dtype=torch.bfloat16, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x0), 64, y0, router_w=wr_d, router_bias=b_d)
    pool.dx_hotness_update(0)
    pool.dx_plan_precision(0)
    tab = pool.dx_get_table(0)
    assert tab["tier"].sum() == n_hot
    x = synth.normal_bf16(11, 2, T, 0, (T, H))
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(T, k, dtype=torch.int32, device="cuda")
    gate = torch.zeros(T, k, dtype=torch.float32, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x), T, y, router_w=wr_d, router_bias=b_d, topk_idx=idx, topk_gate=gate)
    lg_gpu = pool.dx_get_logits(T)
    ref = oracle.router_logits(x, wr, bias)
    d = np.abs(lg_gpu.astype(np.float64) - ref)
    bound = dot_bound(x, wr, bias) * (H * 2.0**-24) + 1e-30
    assert np.all(d <= bound), float((d / bound).max())
    row_rel = d.max(1) / np.abs(ref).max(1)
    assert row_rel.max() <= 1e-3, row_rel.max()
    # the rest of the layer on the GPU's own logits
    idx_o, gate_o = oracle.route(lg_gpu, k)
    assert np.array_equal(idx.cpu().numpy(), idx_o)
    assert np.array_equal(gate.cpu().numpy().view(np.uint32), gate_o.view(np.uint32))
    hot = pool.dx_get_hotness(0)
    cnt_o, mass_o = oracle.counts(idx_o, gate_o, E)
    assert np.array_equal(hot["cnt"], cnt_o) and np.array_equal(hot["mass"], mass_o)
    Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, hb, lb, bool(tab["tier"][e])) for e in np.unique(idx_o)}
    _, y_o = oracle.moe_ffn(x, idx_o, gate_o, Wt, H, I, nthreads=16)
    err, eerr = rel_err(to_u16(y), y_o), elem_err(to_u16(y), y_o)
    print(f"router mode {shape} T={T}: logits max |d|/bound {float((d / bound).max()):.3f}, row rel "
          f"{row_rel.max():.2e}; y rel {err:.2e}, per-element (O-5) {eerr:.2e}")
    assert err <= TOL
    pool.close()


def _edge_logits(T, E, seed):
    lg = synth.trace_logits(seed, 0, 0, T, E, 1.2)
    lg[0, :] = 0.25                                         # all equal -> experts 0..k-1, gates 1/k
    lg[1, 1::2] = lg[1, 0::2][: lg[1, 1::2].size]           # pairwise ties
    lg[2, :] = 0.0
    lg[2, 1::3] = -0.0                                      # +0 / -0 ties
    lg[3, ::2] = -np.inf                                    # masked experts (R-G3)
    lg[4, :] = -np.inf
    lg[4, E - 1] = 1.0                                      # one finite expert: gates (1, 0, ...)
    lg[5, :] = -1e30                                        # huge negative, equal
    lg[6, E // 2] = 80.0                                    # dominant expert: other gates underflow to 0
    return lg


@pytest.mark.parametrize("k,T", [(2, 40), (8, 64), (1, 100), (8, 300), (2, 1000)])
def test_route_edge_cases(dx, k, T):
    """T*k <= 512: the fused decode routing kernel; T*k > 512: the multi-block prefill kernels."""
    E, H, I, g = 32, 64, 128, 32
    m = _masters(3, E, H, I)
    cfg = make_cfg(dx, 1, E, k, H, I, g, 16, 4, budget_for(E, H, I, g, 16, 4, 4, 1), 1, 0.9, 8, 16, 16, 2, T)
    pool = dx.Pool(cfg, m.ptrs(), torch.cuda.current_stream())
    lg = _edge_logits(T, E, 7)
    x = synth.normal_bf16(3, 4, T, 0, (T, H))
    y = torch.zeros(T, H, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(T, k, dtype=torch.int32, device="cuda")
    gate = torch.zeros(T, k, dtype=torch.float32, device="cuda")
    pool.dx_moe_forward(0, bf16_dev(x), T, y, logits=torch.from_numpy(lg).cuda(), topk_idx=idx, topk_gate=gate)
    idx_o, gate_o = oracle.route(lg, k)
    assert np.array_equal(idx.cpu().numpy(), idx_o)
    assert np.array_equal(gate.cpu().numpy().view(np.uint32), gate_o.view(np.uint32))
    if k == 1:
        assert np.all(gate.cpu().numpy() == 1.0)
    assert idx_o[0].tolist() == list(range(k))
    hot = pool.dx_get_hotness(0)
    cnt_o, mass_o = oracle.counts(idx_o, gate_o, E)
    assert np.array_equal(hot["cnt"], cnt_o) and np.array_equal(hot["mass"], mass_o)
    Wt = {int(e): oracle.expert_tier(m.get(0, int(e)), H, I, g, 16, 4, False) for e in np.unique(idx_o)}
    _, y_o = oracle.moe_ffn(x, idx_o, gate_o, Wt, H, I, nthreads=8)
    assert rel_err(to_u16(y), y_o) <= TOL
    pool.close()
