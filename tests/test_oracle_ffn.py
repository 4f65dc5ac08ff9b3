"""Pins for O-5 (routed MoE FFN, Eq. 1).

Pinned against: HuggingFace Qwen3-MoE experts run in fp64 (an independent, library
implementation of the same routed-expert sum), torch's SiLU for the E=k=1 special case,
and exact algebraic properties (zero input, power-of-two gate scaling).
"""
import numpy as np
import torch

import oracle
import synth


def _layer(seed, E, H, I, T, k, high_bits=16, low_bits=4, g=32, tiers=None):
    masters = {e: synth.expert_master(seed, 0, e, H, I) for e in range(E)}
    tiers = tiers if tiers is not None else {e: (e % 3 == 0) for e in range(E)}
    W = {e: oracle.expert_tier(masters[e], H, I, g, high_bits, low_bits, tiers[e]) for e in range(E)}
    x = synth.normal_bf16(seed, 1, 0, 0, (T, H))
    lg = synth.trace_logits(seed, 0, 0, T, E, 1.2)
    idx, gate = oracle.route(lg, k)
    return W, x, idx, gate


def test_matches_hf_qwen3_moe_experts_fp64():
    from transformers.models.qwen3_moe.configuration_qwen3_moe import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeExperts
    E, H, I, T, k = 8, 64, 128, 32, 2
    W, x, idx, gate = _layer(0, E, H, I, T, k)
    _, y = oracle.moe_ffn(x, idx, gate, W, H, I)
    cfg = Qwen3MoeConfig(hidden_size=H, num_experts=E, num_experts_per_tok=k, moe_intermediate_size=I,
                         hidden_act="silu")
    ex = Qwen3MoeExperts(cfg).double()
    n = I * H
    with torch.no_grad():
        for e in range(E):
            w = oracle.bits_to_f32(W[e]).astype(np.float64)
            ex.gate_up_proj[e].copy_(torch.from_numpy(w[: 2 * n].reshape(2 * I, H)))
            ex.down_proj[e].copy_(torch.from_numpy(w[2 * n:].reshape(H, I)))
        ref = ex(torch.from_numpy(oracle.bits_to_f32(x).astype(np.float64)),
                 torch.from_numpy(idx.astype(np.int64)), torch.from_numpy(gate.astype(np.float64))).numpy()
    yf = oracle.bits_to_f32(y).astype(np.float64)
    rel = np.abs(yf - ref).max() / np.abs(ref).max()
    assert rel <= 1e-2, rel


def test_single_expert_is_swiglu():
    """E = k = 1, gate = 1: y is one SwiGLU FFN (torch silu, fp64) up to the bf16 rounding points."""
    H, I, T = 64, 96, 7
    m = synth.expert_master(4, 0, 0, H, I)
    W = {0: oracle.expert_tier(m, H, I, 32, 16, 4, True)}
    x = synth.normal_bf16(4, 0, 0, 0, (T, H))
    idx = np.zeros((T, 1), np.int32)
    gate = np.ones((T, 1), np.float32)
    Y, y = oracle.moe_ffn(x, idx, gate, W, H, I)
    w = oracle.bits_to_f32(W[0]).astype(np.float64)
    n = I * H
    xt = torch.from_numpy(oracle.bits_to_f32(x).astype(np.float64))
    u = xt @ torch.from_numpy(w[:n].reshape(I, H)).T
    v = xt @ torch.from_numpy(w[n:2 * n].reshape(I, H)).T
    a = (torch.nn.functional.silu(u) * v).to(torch.bfloat16).double()
    o = a @ torch.from_numpy(w[2 * n:].reshape(H, I)).T
    ref = o.to(torch.bfloat16).double().numpy()
    yf = oracle.bits_to_f32(y).astype(np.float64)
    assert np.abs(yf - ref).max() <= 2**-7 * np.abs(ref).max()
    assert np.array_equal(Y[:, 0], y)                 # k = 1: combine is the identity


def test_zero_input_and_gate_scaling():
    E, H, I, T, k = 4, 64, 128, 6, 2
    W, x, idx, _ = _layer(2, E, H, I, T, k)
    g1 = np.full((T, k), 0.25, np.float32)
    g2 = np.full((T, k), 0.5, np.float32)
    Y1, _ = oracle.moe_ffn(x, idx, g1, W, H, I)
    Y2, _ = oracle.moe_ffn(x, idx, g2, W, H, I)
    assert np.array_equal(oracle.bits_to_f32(Y2), 2 * oracle.bits_to_f32(Y1))
    _, y0 = oracle.moe_ffn(np.zeros_like(x), idx, g1, W, H, I)
    assert np.all(oracle.bits_to_f32(y0) == 0)


def test_expert_relabeling_invariance():
    """Permuting expert ids together with their weights leaves y unchanged (Eq. 1 sums over K)."""
    E, H, I, T, k = 6, 64, 64, 9, 3
    W, x, idx, gate = _layer(5, E, H, I, T, k)
    perm = np.array([3, 5, 0, 1, 4, 2])
    W2 = {int(perm[e]): W[e] for e in range(E)}
    _, y1 = oracle.moe_ffn(x, idx, gate, W, H, I)
    _, y2 = oracle.moe_ffn(x, perm[idx].astype(np.int32), gate, W2, H, I)
    assert np.array_equal(y1, y2)
