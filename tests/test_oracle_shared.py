"""Pins of the oracle's f-3 shared expert (Eq. 1's first sum; DESIGN.md R-S1): or_shared_ffn against a
torch fp64 SwiGLU (bf16 rounding at the same two points), the zero shared expert reducing to the routed-only
oracle bitwise, and or_combine_shared's order (shared term first, then the routed rows)."""
import numpy as np
import torch

import oracle
import synth


def _f32(u16):
    return oracle.bits_to_f32(u16).astype(np.float64)


def test_shared_ffn_matches_torch_swiglu():
    H, I, T = 64, 128, 5
    w = synth.expert_master(21, 0, 0, H, I)
    x = synth.normal_bf16(21, 1, 0, 0, (T, H))
    Ys, _, _ = oracle.moe_ffn_shared(x, np.zeros((T, 1), np.int32), np.zeros((T, 1), np.float32),
                                     {0: np.zeros(3 * I * H, np.uint16)}, w, H, I)
    Wg = torch.from_numpy(_f32(w[:I * H]).reshape(I, H))
    Wu = torch.from_numpy(_f32(w[I * H:2 * I * H]).reshape(I, H))
    Wd = torch.from_numpy(_f32(w[2 * I * H:]).reshape(H, I))
    xt = torch.from_numpy(_f32(x))
    u, v = xt @ Wg.T, xt @ Wu.T
    a = (torch.nn.functional.silu(u) * v).to(torch.bfloat16).to(torch.float64)
    o = (a @ Wd.T).to(torch.float32).numpy()
    ref = oracle.bits_to_f32(np.array([[oracle.f64_to_bf16_rn(float(val)) for val in row] for row in o], np.uint16))
    got = oracle.bits_to_f32(Ys)
    # one bf16 ulp of slack: torch's fp64 -> bf16 cast of a goes through fp32 (double rounding) in rare ties
    assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0**-7 + 1e-30)


def test_zero_shared_expert_is_the_routed_oracle():
    E, k, H, I, T = 8, 2, 64, 128, 7
    W = {e: synth.expert_master(22, 0, e, H, I) for e in range(E)}
    x = synth.normal_bf16(22, 1, 0, 0, (T, H))
    idx, gate = oracle.route(synth.trace_logits(22, 0, 0, T, E, 1.2), k)
    _, y_plain = oracle.moe_ffn(x, idx, gate, W, H, I)
    Ys, _, y = oracle.moe_ffn_shared(x, idx, gate, W, np.zeros(3 * I * H, np.uint16), H, I)
    assert not Ys.any() and np.array_equal(y, y_plain)


def test_combine_shared_order_and_terms():
    T, k, H = 3, 2, 8
    rng = np.random.default_rng(0)
    Ys = np.array([[oracle.f32_to_bf16_rn(float(v)) for v in rng.standard_normal(H)] for _ in range(T)], np.uint16)
    Y = np.zeros((T, k, H), np.uint16)
    y = np.zeros((T, H), np.uint16)
    oracle._L().or_combine_shared(oracle._p(Ys), oracle._p(Y), T, k, H, oracle._p(y))
    assert np.array_equal(y, Ys)                                    # routed rows zero: y is the shared term
    Y[:, 0] = Ys                                                    # y = bf16(2 Ys) exactly
    oracle._L().or_combine_shared(oracle._p(Ys), oracle._p(Y), T, k, H, oracle._p(y))
    assert np.array_equal(_f32(y), 2 * _f32(Ys))
