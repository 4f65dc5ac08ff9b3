"""Pins for the oracle's numeric formats and group quantiser (O-4).

Pinned against: torch's bf16 cast (library RNE), brute-force enumeration of bf16 neighbours,
hand-worked examples (tests/golden/quant_worked_examples.txt, DESIGN.md R-Q1), the paper's
memory footprints and mathematical round-trip bounds.
"""
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "quant_worked_examples.txt")


def _bf16_neighbors(x: float):
    """All finite bf16 values as exact Fractions near x (brute force over the 2^16 codes)."""
    codes = np.arange(1 << 16, dtype=np.uint32)
    vals = (codes << 16).view(np.float32).astype(np.float64)
    ok = np.isfinite(vals)
    return codes[ok], vals[ok]


_CODES, _VALS = _bf16_neighbors(0.0)
_ORDER = np.argsort(_VALS, kind="stable")


def _brute_rn(x: float) -> float:
    """nearest bf16 (ties to even mantissa) by exhaustive search with exact Fractions"""
    fx = Fraction(x)
    i = np.searchsorted(_VALS[_ORDER], x)
    cands = []
    for j in range(max(0, i - 2), min(len(_ORDER), i + 3)):
        c = int(_CODES[_ORDER[j]])
        v = float(_VALS[_ORDER[j]])
        cands.append((abs(Fraction(v) - fx), c & 1, v))
    cands.sort()
    return cands[0][2]


def _brute_ru(x: float) -> float:
    v = _VALS[_ORDER]
    i = np.searchsorted(v, x, side="left")
    return float(v[i])


def test_bf16_rn_matches_torch_cast():
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 20000),
                         np.array([0.0, -0.0, 1e-40, -1e-40, 3.4e38, 1.0 + 2**-8, 1.0 + 3 * 2**-8], np.float32)])
    xs = xs.astype(np.float32)
    ref = torch.from_numpy(xs).to(torch.bfloat16).view(torch.int16).numpy().astype(np.uint16)
    got = np.array([oracle.f32_to_bf16_rn(float(v)) for v in xs], dtype=np.uint16)
    assert np.array_equal(got, ref)


def test_bf16_ru_brute_force():
    rng = np.random.default_rng(1)
    xs = np.abs(rng.standard_normal(3000).astype(np.float32)) * np.float32(0.01)
    for v in list(xs) + [np.float32(0.1), np.float32(1.0), np.float32(1e-39)]:
        got = oracle.bf16_to_f32(oracle.f32_to_bf16_ru(float(v)))
        assert got == _brute_ru(float(v)), v
        assert got >= float(v)


def test_f64_to_bf16_single_rounding():
    rng = np.random.default_rng(2)
    xs = list(rng.standard_normal(2000) * 10.0 ** rng.integers(-20, 20, 2000))
    # double-rounding trap: just above a bf16 tie, which fp64->fp32->bf16 would round to even wrongly
    xs += [1.0 + 2**-8 + 2**-30, -(1.0 + 2**-8 + 2**-30), 1.0 + 2**-8, 1e-39, 5e-41]
    for x in xs:
        got = oracle.bf16_to_f32(oracle.f64_to_bf16_rn(float(x)))
        assert got == _brute_rn(float(x)), x


def _golden():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f = [p.strip() for p in line.split("|")]
        bits, g = map(int, f[0].split())
        rows.append((bits, g, [float(v) for v in f[1].split()], float(f[2]), int(f[3]),
                     [int(v) for v in f[4].split()], [float(v) for v in f[5].split()]))
    return rows


@pytest.mark.parametrize("row", _golden())
def test_quantizer_worked_examples(row):
    bits, g, w, s, z, codes, deq = row
    wb = np.array([[oracle.f32_to_bf16_rn(v) for v in w]], dtype=np.uint16)
    c, sc, zr = oracle.quantize(wb, g, bits)
    assert oracle.bf16_to_f32(int(sc[0, 0])) == s
    assert int(zr[0, 0]) == z
    assert c[0].tolist() == codes
    assert oracle.bits_to_f32(oracle.dequantize(c, sc, zr, g))[0].tolist() == deq


@pytest.mark.parametrize("bits", [4, 2])
def test_quantizer_roundtrip_bound_and_invariants(bits):
    """|w - (q-z)s| <= s/2 (RTN), codes/zeros in [0, qmax], w=0 -> code z (exact zero),
    deq = bf16_rn of the exact product (single rounding)."""
    g = 128
    w = synth.weights_bf16(7, 0, 0, 0, 256, 1024)
    w[3, :128] = 0                                # an all-zero group
    w[5, 0:128:7] = 0                             # zeros inside a group
    c, sc, zr = oracle.quantize(w, g, bits)
    qmax = (1 << bits) - 1
    assert c.max() <= qmax and zr.max() <= qmax
    wf = oracle.bits_to_f32(w).astype(np.float64)
    s = np.repeat(oracle.bits_to_f32(sc).astype(np.float64), g, axis=1)
    zz = np.repeat(zr.astype(np.float64), g, axis=1)
    prod = (c.astype(np.float64) - zz) * s
    assert np.all(np.abs(wf - prod) <= s * (0.5 + 2.0**-20))
    deq = oracle.bits_to_f32(oracle.dequantize(c, sc, zr, g)).astype(np.float64)
    ref = torch.from_numpy(prod).to(torch.bfloat16).to(torch.float64).numpy()  # exact prod -> one RNE
    assert np.array_equal(deq, ref)
    assert np.all(deq[wf == 0] == 0)
    assert oracle.bits_to_f32(sc[3, 0]) == 1.0 and zr[3, 0] == 0 and np.all(c[3, :128] == 0)


def test_scale_round_up_keeps_range():
    """s >= (wmax-wmin)/qmax, so (wmax-wmin) fits in qmax steps (DESIGN.md R-Q1 step 3)."""
    w = synth.weights_bf16(3, 1, 2, 1, 64, 512)
    for bits in (4, 2):
        _, sc, _ = oracle.quantize(w, 128, bits)
        wf = oracle.bits_to_f32(w).reshape(64, 4, 128).astype(np.float64)
        rng_ = np.maximum(wf.max(-1), 0) - np.minimum(wf.min(-1), 0)
        assert np.all(oracle.bits_to_f32(sc) * ((1 << bits) - 1) >= rng_ * (1 - 2**-23))


def test_path_independence_high_int4():
    """LOW = Q_low(deq(HIGH)) (DESIGN.md R-Q2): int2 codes of an int4 HIGH image equal quantising
    the dequantised HIGH weights directly."""
    H, I, g = 256, 128, 128
    m = synth.expert_master(0, 0, 3, H, I)
    hi, hc, hs, hz = oracle.expert_tier(m, H, I, g, 4, 2, True, want_codes=True)
    lo, lc, ls, lz = oracle.expert_tier(m, H, I, g, 4, 2, False, want_codes=True)
    n = I * H
    c2, s2, z2 = oracle.quantize(hi[:n].reshape(I, H), g, 2)
    assert np.array_equal(lc[:n], c2.reshape(-1)) and np.array_equal(ls[:n // g], s2.reshape(-1))


def test_slot_bytes_match_paper_footprints():
    """Appendix A of SURVEY: with g=128, bf16 scale, u8 zero, the expert totals reproduce the paper's
    footprints: Qwen3-30B 57 GB bf16 -> 17 GB int4 incl. ~1.5B non-expert params
    (PAPER.md:332); Qwen3-80B 152/41/21 GB.  2 % bound on the expert share."""
    q30 = [oracle.slot_bytes(2048, 768, 128, b) * 48 * 128 for b in (16, 4)]
    q80 = [oracle.slot_bytes(2048, 512, 128, b) * 48 * 512 for b in (16, 4, 2)]
    assert abs(q30[0] / 57e9 - 1) < 0.02
    assert abs(q80[0] / 152e9 - 1) < 0.02
    assert abs(q80[1] / 41e9 - 1) < 0.02
    assert abs(q80[2] / 21e9 - 1) < 0.02
    assert q30[1] < 17e9 < q30[1] + 3e9          # + non-expert weights (< 3 GB)
    # C1 slot sizes stated in SURVEY §8(c) O-3 step 1
    assert oracle.slot_bytes(64, 128, 32, 16) == 49152
    assert oracle.slot_bytes(64, 128, 32, 4) == 15360
