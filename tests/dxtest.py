"""Shared helpers for the GPU parity tests: seeded pools, oracle replays (tests only)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth

C1 = dict(L=1, E=8, k=2, H=64, I=128, g=32, high=16, low=4, T=32, n_hot=2, s=1, alpha=0.9, Tp=8, W=16,
          dwell=16, lag=2, zipf=1.2, drift=16, frac=0.5)


def budget_for(E, H, I, g, high, low, n_hot, s, L=1):
    Sh, Sl = oracle.slot_bytes(H, I, g, high), oracle.slot_bytes(H, I, g, low)
    return L * ((n_hot + s) * Sh + (E - n_hot + s) * Sl)


class Masters:
    """Pinned host bf16 masters [L][E] of 3*I*H each, from synth (the only shared input code)."""

    def __init__(self, seed, L, E, H, I):
        n = 3 * I * H
        self.t = torch.empty(L * E * n, dtype=torch.int16, pin_memory=True)
        self.np = self.t.numpy().view(np.uint16)
        self.n, self.L, self.E = n, L, E
        for l in range(L):
            for e in range(E):
                synth.expert_master_into(seed, l, e, H, I, self.np[(l * E + e) * n:(l * E + e + 1) * n])

    def ptrs(self):
        base = self.t.data_ptr()
        return [base + i * self.n * 2 for i in range(self.L * self.E)]

    def get(self, l, e):
        return self.np[(l * self.E + e) * self.n:(l * self.E + e + 1) * self.n]


def make_cfg(dx, L, E, k, H, I, g, high, low, budget, s, alpha, Tp, W, dwell, lag, max_tokens):
    c = dx.dx_config()
    c.num_layers, c.num_experts, c.top_k, c.hidden, c.inter, c.group_size = L, E, k, H, I, g
    c.high_bits, c.low_bits = high, low
    c.expert_budget_bytes = budget
    c.n_spare = s
    c.ema_alpha = alpha
    c.period, c.warmup_steps, c.dwell_min, c.publish_lag = Tp, W, dwell, lag
    c.max_tokens = max_tokens
    c.ep_rank, c.ep_size = 0, 1
    return c


def canon_expected(master, H, I, g, high, low, tier_high):
    """Oracle canonical export image of one expert at a tier (bytes as dx_export_expert writes them)."""
    bits = high if tier_high else low
    if bits == 16:
        w = oracle.expert_tier(master, H, I, g, high, low, tier_high)
        return w.view(np.uint8)
    w, c, s, z = oracle.expert_tier(master, H, I, g, high, low, tier_high, want_codes=True)
    return np.concatenate([c, s.view(np.uint8), z])


def rel_err(y, ref):
    y = oracle.bits_to_f32(y).astype(np.float64)
    ref = oracle.bits_to_f32(ref).astype(np.float64)
    den = np.abs(ref).max()
    return float(np.abs(y - ref).max() / den) if den > 0 else float(np.abs(y).max())


def bf16_dev(a_u16: np.ndarray, dev="cuda"):
    return torch.from_numpy(np.ascontiguousarray(a_u16).view(np.int16)).to(dev).view(torch.bfloat16)


def to_u16(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def elem_err(y, ref):
    """SURVEY §8(c) O-5 per-element metric: max |y - ref| / (|ref| + 1e-2 * ||ref||_inf)."""
    y = oracle.bits_to_f32(y).astype(np.float64)
    ref = oracle.bits_to_f32(ref).astype(np.float64)
    den = np.abs(ref) + 1e-2 * np.abs(ref).max()
    return float((np.abs(y - ref) / np.where(den > 0, den, 1.0)).max())


def dot_bound(x_u16, wr_u16, bias=None):
    """Per-element scale sum_h |x_h w_eh| + |b_e| of a router logit: the fp32-summation error of an n-term
    dot product of exact bf16 products is <= gamma_n times this (gamma_n ~ n * 2^-24)."""
    x = np.abs(oracle.bits_to_f32(x_u16).astype(np.float64))
    w = np.abs(oracle.bits_to_f32(wr_u16).astype(np.float64))
    s = x @ w.T
    if bias is not None:
        s = s + np.abs(np.asarray(bias, np.float64))
    return s
