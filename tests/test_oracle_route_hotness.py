"""Pins for O-1 (top-k + gates) and O-2 (hotness counters + EMA).

Pinned against: math.exp (ulp bound), numpy's stable lexsort (brute-force top-k), fp64 softmax,
HuggingFace Qwen3-MoE's router (softmax -> topk -> renormalise, PAPER.md:277 models),
numpy bincount recounts, and SPEC.md's worked EMA values / closed form.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth


def _ulp_err(got: float, ref: float) -> float:
    if ref == 0:
        return 0.0 if got == 0 else float("inf")
    sp = np.spacing(np.float32(ref))
    return abs(got - ref) / float(sp)


def test_expf_exact_at_zero_and_ulp_bound():
    assert oracle.expf(0.0) == 1.0
    assert oracle.expf(-0.0) == 1.0
    xs = np.concatenate([-np.linspace(0, 87, 20001, dtype=np.float32),
                         -np.random.default_rng(0).random(5000, dtype=np.float32) * 30])
    worst = max(_ulp_err(oracle.expf(float(x)), math.exp(float(x))) for x in xs)
    assert worst <= 2.0, worst
    assert oracle.expf(-104.0) == 0.0


def _brute_topk(logits, k):
    T, E = logits.shape
    out = np.zeros((T, k), np.int32)
    for t in range(T):
        order = np.lexsort((np.arange(E), -logits[t].astype(np.float64)))  # logit desc, id asc
        out[t] = order[:k]
    return out


@pytest.mark.parametrize("T,E,k", [(64, 8, 2), (37, 128, 8), (9, 512, 10), (5, 3, 3)])
def test_topk_matches_brute_force_and_gates_softmax(T, E, k):
    lg = synth.trace_logits(11, 2, 5, T, E, 1.2)
    lg[0, :] = 0.5                                  # all ties -> experts 0..k-1, gates 1/k
    lg[1, 1::2] = lg[1, 0::2][: lg[1, 1::2].size]   # pairwise ties
    idx, gate = oracle.route(lg, k)
    assert np.array_equal(idx, _brute_topk(lg, k))
    sel = np.take_along_axis(lg.astype(np.float64), idx.astype(np.int64), 1)
    ref = np.exp(sel - sel[:, :1])
    ref /= ref.sum(1, keepdims=True)
    assert np.allclose(gate, ref, rtol=2e-6, atol=1e-7)
    assert np.all(np.abs(gate.astype(np.float64).sum(1) - 1) <= 1e-6)
    assert idx[0].tolist() == list(range(k))
    assert np.all(gate[0] == np.float32(1.0) / np.float32(k)) or np.allclose(gate[0], 1.0 / k, rtol=1e-7)


def test_k1_gate_is_exactly_one():
    lg = synth.trace_logits(1, 0, 0, 50, 16)
    _, gate = oracle.route(lg, 1)
    assert np.all(gate == 1.0)


def test_nonfinite_logits_rejected():
    for bad in (np.nan, np.inf):
        lg = np.zeros((2, 4), np.float32)
        lg[1, 2] = bad
        with pytest.raises(ValueError):
            oracle.route(lg, 2)
    with pytest.raises(ValueError):                       # no finite logit in a token (R-G3)
        oracle.route(np.full((1, 4), -np.inf, np.float32), 2)


def test_masked_experts_neg_inf():
    """R-G3: -inf = masked expert: ranked after every finite logit (ties among masked experts to the
    lower id), gate exactly 0; the finite part of the selection is the plain top-k of the finite logits."""
    lg = synth.trace_logits(4, 0, 0, 20, 16, 1.2)
    lg[:, ::2] = -np.inf
    idx, gate = oracle.route(lg, 4)
    assert np.array_equal(idx, _brute_topk(np.where(np.isinf(lg), -1e30, lg), 4))
    assert np.all(idx % 2 == 1)                           # 8 finite experts >= k: masked never chosen
    one = np.full((3, 8), -np.inf, np.float32)
    one[:, 5] = 0.25
    idx, gate = oracle.route(one, 3)
    assert idx.tolist() == [[5, 0, 1]] * 3                # then masked ones by ascending id
    assert gate[:, 0].tolist() == [1.0] * 3 and np.all(gate[:, 1:] == 0.0)


def test_signed_zero_logits_tie():
    """-0 and +0 compare equal, so they tie and the lower id wins (R-G1)."""
    lg = np.array([[-0.0, 0.0, -1.0, -0.0]], np.float32)
    idx, gate = oracle.route(lg, 3)
    assert idx.tolist() == [[0, 1, 3]]
    assert np.all(gate == np.float32(1) / np.float32(3)) or np.allclose(gate, 1 / 3, rtol=1e-7)


def test_router_logits_pins():
    """or_router_logits (O-1 step 1, Eq. 1 router, full precision PAPER.md:281): (a) equals numpy's fp64
    x @ W_r^T + b (a transposed or mis-strided W_r, a dropped bias or a wrong K range fails it on these
    non-square shapes); (b) closed form: one-hot token rows pick out a column of W_r exactly."""
    for (T, E, H) in [(7, 8, 64), (5, 128, 2048), (3, 512, 256)]:
        x = synth.normal_bf16(2, T, E, H, (T, H))
        wr = synth.router_bf16(2, 1, E, H)
        b = synth.zipf_logp(synth.rank_perm(2, 1, 0, E, 4, 0.0), 1.2)
        got = oracle.router_logits(x, wr, b)
        ref = oracle.bits_to_f32(x).astype(np.float64) @ oracle.bits_to_f32(wr).astype(np.float64).T + b
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)
        nob = oracle.router_logits(x, wr)
        assert np.allclose(got - nob, np.broadcast_to(b.astype(np.float64), got.shape), atol=1e-12)
    E, H = 16, 96
    wr = synth.router_bf16(5, 0, E, H)
    onehot = np.zeros((H, H), np.uint16)
    onehot[np.arange(H), np.arange(H)] = 0x3F80            # bf16 1.0
    got = oracle.router_logits(onehot, wr)
    assert np.array_equal(got, oracle.bits_to_f32(wr).astype(np.float64).T)


def test_route_matches_hf_qwen3_router():
    """Qwen3-MoE routes by softmax -> top-k -> renormalise (norm_topk_prob); top-k of a softmax is
    top-k of the logits, and the renormalised mass equals softmax over the selected logits."""
    from transformers.models.qwen3_moe.configuration_qwen3_moe import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeTopKRouter
    E, k, H, T = 32, 4, 64, 40
    cfg = Qwen3MoeConfig(hidden_size=H, num_experts=E, num_experts_per_tok=k, norm_topk_prob=True,
                         moe_intermediate_size=32)
    r = Qwen3MoeTopKRouter(cfg).double()
    x = oracle.bits_to_f32(synth.normal_bf16(0, 0, 0, 0, (T, H)))
    wr = oracle.bits_to_f32(synth.router_bf16(0, 0, E, H))
    with torch.no_grad():
        r.weight.copy_(torch.from_numpy(wr.astype(np.float64)))
        _, w_hf, i_hf = r(torch.from_numpy(x.astype(np.float64)))
    lg = (x.astype(np.float64) @ wr.astype(np.float64).T).astype(np.float32)
    idx, gate = oracle.route(lg, k)
    assert np.array_equal(idx, i_hf.numpy())
    assert np.allclose(gate, w_hf.numpy(), rtol=1e-5, atol=1e-6)


def test_counts_match_bincount_and_mass_bound():
    for (T, E, k) in [(32, 8, 2), (300, 128, 8), (77, 512, 10)]:
        lg = synth.trace_logits(5, 1, 3, T, E, 1.2)
        idx, gate = oracle.route(lg, k)
        cnt, mass = oracle.counts(idx, gate, E)
        assert np.array_equal(cnt, np.bincount(idx.ravel(), minlength=E).astype(np.uint32))
        ref_mass = np.zeros(E, np.int64)
        np.add.at(ref_mass, idx.ravel(), np.rint(gate.astype(np.float64).ravel() * 2**24).astype(np.int64))
        assert np.array_equal(mass.astype(np.int64), ref_mass)
        assert cnt.sum() == T * k
        assert abs(int(mass.sum()) - T * 2**24) <= T * k
        # EP: local range counts are the slice of the global counts
        c2, m2 = oracle.counts(idx, gate, E // 2, e_lo=E // 2)
        assert np.array_equal(c2, cnt[E // 2:]) and np.array_equal(m2, mass[E // 2:])


def test_ema_spec_examples():
    """(S=0, a=0.9, g=1) -> 0.1; (S=0.5 inactive) -> 0.45; a=0.5, g=1,1,1 -> 0.875."""
    one = np.array([2**24], np.uint64)
    assert abs(oracle.ema_fold([0.0], one, 1, 0.9)[0] - 0.1) < 1e-15
    assert abs(oracle.ema_fold([0.5], np.zeros(1, np.uint64), 1, 0.9)[0] - 0.45) < 1e-15
    S = np.zeros(1)
    for _ in range(3):
        S = oracle.ema_fold(S, one, 1, 0.5)
    assert S[0] == 0.875


def test_ema_closed_form_and_bounds():
    """constant gate g from S=0 gives S = g(1 - a^t) to 1e-12; S stays in [0,1]."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        a = float(rng.uniform(0.5, 0.999))
        gq = int(rng.integers(0, 2**24 + 1))
        t = int(rng.integers(1, 2000))
        S = np.zeros(1)
        for _ in range(t):
            S = oracle.ema_fold(S, np.array([gq], np.uint64), 1, a)
        g = gq / 2**24
        assert abs(S[0] - g * (1 - a**t)) <= 1e-12
        assert 0.0 <= S[0] <= 1.0
