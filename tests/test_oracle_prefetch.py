"""Pins of the oracle's f-1 functions (cross-layer correlation prefetch):
or_corr_update (update_correlation) and or_prefetch_candidates, against SPEC.md's worked examples, a numpy
brute force of the plain definitions, the k*k increment invariant and SPEC's convergence property (empirical
conditional frequencies of a coupled generator converge to its coupling within 0.05 after 10^4 tokens)."""
import numpy as np

import oracle


def test_corr_spec_examples():
    E = 4
    c = np.zeros((E, E), np.uint32)
    oracle.corr_update(c, np.array([[0]]), np.array([[1]]))          # token activates {a} then {b}
    assert c[0, 1] == 1 and c.sum() == 1                             # count[a, b] += 1
    c = np.zeros((E, E), np.uint32)
    oracle.corr_update(c, np.array([[0, 2]]), np.array([[1, 3]]))    # k = 2: cartesian product
    assert c.sum() == 4 and c[0, 1] == c[0, 3] == c[2, 1] == c[2, 3] == 1


def test_corr_brute_force_and_invariant():
    rng = np.random.default_rng(3)
    for T, k, E in ((1, 1, 8), (17, 2, 8), (64, 8, 128), (33, 10, 512)):
        a = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
        b = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
        c = np.zeros((E, E), np.uint32)
        c[5 % E, 1] = 7                                               # counts only increase from any start
        ref = c.astype(np.int64).copy()
        oracle.corr_update(c, a, b)
        for t in range(T):
            for x in a[t]:
                for y in b[t]:
                    ref[x, y] += 1
        assert np.array_equal(c.astype(np.int64), ref)
        assert int(c.sum()) == 7 + T * k * k


def test_corr_converges_to_generator_coupling():
    """stationary coupled distribution -> empirical conditional frequencies within 0.05 of the
    generator's conditional matrix after 10^4 tokens."""
    rng = np.random.default_rng(11)
    E, coupling, n = 16, 0.9, 10_000
    pi = rng.permutation(E)
    a = rng.integers(0, E, n)
    follow = rng.random(n) < coupling
    b = np.where(follow, pi[a], rng.integers(0, E, n))
    c = np.zeros((E, E), np.uint32)
    oracle.corr_update(c, a.reshape(-1, 1).astype(np.int32), b.reshape(-1, 1).astype(np.int32))
    emp = c / c.sum(1, keepdims=True)
    true = np.full((E, E), (1 - coupling) / E)
    true[np.arange(E), pi] += coupling
    assert np.abs(emp - true).max() <= 0.05


def _brute_candidates(corr, idx, tier, infl, own, f):
    E = corr.shape[0]
    score = corr[idx.ravel()].astype(np.int64).sum(0)
    elig = [e for e in range(E) if tier[e] == 0 and infl[e] == 0 and score[e] > 0]
    elig.sort(key=lambda e: (-score[e], e))
    free = [b for b in range(own.size) if own[b] < 0]
    n = min(f, len(free), len(elig))
    return [(elig[i], free[i]) for i in range(n)]


def test_prefetch_spec_examples():
    E = 4
    corr = np.zeros((E, E), np.uint32)
    corr[0, 1], corr[0, 2] = 50, 3                                   # row: b >> c
    tier, infl = np.zeros(E, np.int32), np.zeros(E, np.int32)
    own = np.array([2, -1, -1], np.int32)                            # HIGH blocks 1, 2 free
    idx = np.array([[0]], np.int32)
    assert oracle.prefetch_candidates(corr, idx, tier, infl, own, 0) == []          # f = 0: disabled
    assert oracle.prefetch_candidates(corr, idx, tier, infl, own, 1) == [(1, 1)]    # argmax, lowest free block
    assert oracle.prefetch_candidates(corr, idx, tier, infl, own, 4) == [(1, 1), (2, 2)]   # two free blocks
    tier[1] = 1                                                      # already HIGH: filtered
    assert oracle.prefetch_candidates(corr, idx, tier, infl, own, 1) == [(2, 1)]
    infl[2] = 1                                                      # in flight: filtered
    assert oracle.prefetch_candidates(corr, idx, tier, infl, own, 1) == []


def test_prefetch_brute_force():
    rng = np.random.default_rng(5)
    for E, k, T, f in ((8, 2, 5, 2), (128, 8, 64, 3), (512, 10, 16, 8)):
        corr = rng.integers(0, 4, (E, E)).astype(np.uint32)
        corr[rng.random((E, E)) < 0.5] = 0
        idx = np.stack([rng.choice(E, k, replace=False) for _ in range(T)]).astype(np.int32)
        tier = (rng.random(E) < 0.3).astype(np.int32)
        infl = (rng.random(E) < 0.1).astype(np.int32)
        own = np.where(rng.random(9) < 0.5, -1, 3).astype(np.int32)
        assert oracle.prefetch_candidates(corr, idx, tier, infl, own, f) == _brute_candidates(corr, idx, tier, infl, own, f)
