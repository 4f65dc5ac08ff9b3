"""Pins for O-3 / O-6: budget solver, pool ledger and Alg. 1 controller replay.

Pinned against: SPEC.md worked examples (init_budget :156-158, warmup_threshold :163-168,
schedule :176-178, alloc/free :253-265), brute-force max-feasible n_hot, a brute-force
sort-and-filter hot set, a Python set-based reference allocator, and invariants
(budget, |HIGH| <= n_hot, one stable slot per expert, monotone versions, periodicity,
determinism, corner cases n_hot = 0 / N).
"""
import numpy as np
import pytest

import oracle
import synth


# ------------------------------------------------------------------ budget
def test_init_budget_spec_examples():
    # SPEC.md:156-158 (no spare slots: the SPEC solver has none)
    assert oracle.n_hot(256, 128, 2, 1, 0) == 128
    assert oracle.n_hot(128, 128, 2, 1, 0) == 0
    assert oracle.n_hot(200, 128, 4, 1, 0) == 24
    assert oracle.n_hot(127, 128, 2, 1, 0) == -1           # infeasible: all-LOW does not fit


def test_n_hot_brute_force():
    rng = np.random.default_rng(0)
    for _ in range(10000):
        N = int(rng.integers(1, 513))
        Sl = int(rng.integers(1, 1000))
        Sh = Sl + int(rng.integers(1, 4000))
        s = int(rng.integers(0, 3))
        M = int(rng.integers(0, (N + 2 * s) * Sh + 1))
        feas = [n for n in range(N + 1) if (n + s) * Sh + (N - n + s) * Sl <= M]
        assert oracle.n_hot(M, N, Sh, Sl, s) == (max(feas) if feas else -1)


def test_c2_budget():
    """Q30B, 24e9 B over 48 layers -> M = 5e8 -> n_hot 24 with one spare per tier."""
    Sh, Sl = oracle.slot_bytes(2048, 768, 128, 16), oracle.slot_bytes(2048, 768, 128, 4)
    M = 24 * 10**9 // 48
    assert oracle.n_hot(M, 128, Sh, Sl, 1) == 24
    assert oracle.n_hot(M, 128, Sh, Sl, 0) == 26


# ------------------------------------------------------------------ ledger
def test_alloc_free_spec_examples():
    own = np.full(4, -1, np.int32)
    assert oracle.ledger_alloc(own, 10) == 0                     # fresh -> block 0
    a = 0
    b = oracle.ledger_alloc(own, 11)
    c = oracle.ledger_alloc(own, 12)
    assert (a, b, c) == (0, 1, 2)
    assert oracle.ledger_free(own, b, 11) == 0
    assert oracle.ledger_alloc(own, 13) == 1                     # d reuses block 1
    assert oracle.ledger_alloc(own, 14) == 3
    assert oracle.ledger_alloc(own, 15) == -1                    # exhausted
    assert oracle.ledger_free(own, 3, 14) == 0
    assert oracle.ledger_free(own, 3, 14) == -1                  # double free is corruption


def test_ledger_random_replay():
    rng = np.random.default_rng(1)
    cap = 64
    own = np.full(cap, -1, np.int32)
    ref_free = set(range(cap))
    held = {}
    for op in range(100000):
        if held and (rng.random() < 0.5 or not ref_free):
            who = int(rng.choice(list(held)))
            slot = held.pop(who)
            assert oracle.ledger_free(own, slot, who) == 0
            ref_free.add(slot)
        else:
            who = op
            slot = oracle.ledger_alloc(own, who)
            assert slot == min(ref_free)
            ref_free.remove(slot)
            held[who] = slot
        if op % 997 == 0:
            assert ref_free == set(np.flatnonzero(own < 0).tolist())
        assert len(ref_free) + len(held) == cap


# ------------------------------------------------------------------ Alg. 1 on hand-built states
def test_schedule_spec_examples():
    # n_hot=2, tau=0.4, {a:.9, b:.5, c:.3} all LOW -> [UP a, UP b]
    c = oracle.Controller(3, 2, 1, 0.9, 8, 0, 0, 1)
    c.debug_set([0.9, 0.5, 0.3], [0, 0, 0], 0.4, 8)
    plan, fin = c.plan()
    assert not fin and [(e, d) for e, d, _ in plan] == [(0, 1), (1, 1)]
    # {a:.9, b:.35, c:.3}, a,b HIGH -> [DOWN b] (b fails S >= tau although rank < n_hot)
    c = oracle.Controller(3, 2, 1, 0.9, 8, 0, 0, 1)
    c.debug_set([0.9, 0.35, 0.3], [1, 1, 0], 0.4, 16)
    plan, _ = c.plan()
    assert [(e, d) for e, d, _ in plan] == [(1, -1)]
    # off-period -> nothing
    c.debug_set([0.9, 0.35, 0.3], [1, 1, 0], 0.4, 7)
    assert c.plan() is None
    # idempotence: second call at the same step emits nothing
    c.debug_set([0.9, 0.35, 0.3], [1, 1, 0], 0.4, 16)
    assert len(c.plan()[0]) == 1 and c.plan()[0] == []


def _brute_hot(S, n_hot, tau):
    order = sorted(range(len(S)), key=lambda e: (-S[e], e))
    return {e for r, e in enumerate(order) if r < n_hot and S[e] >= tau}


def test_hot_set_matches_brute_force_with_ample_spares():
    """With spares >= E and dwell 0 every mismatch is fixed in one period, so after publication the
    HIGH set equals the brute-force sort-and-filter hot set."""
    rng = np.random.default_rng(2)
    for _ in range(1000):
        E = int(rng.integers(1, 40))
        n_hot = int(rng.integers(0, E + 1))
        S = np.round(rng.random(E), 2)                            # coarse values -> many ties
        tau = float(rng.choice(S)) if rng.random() < 0.8 else float(rng.random())
        tier = np.zeros(E, np.int32)
        tier[rng.permutation(E)[: int(rng.integers(0, n_hot + 1))]] = 1
        c = oracle.Controller(E, n_hot, E, 0.9, 4, 0, 0, 1)
        c.debug_set(S, tier, tau, 8)
        plan, _ = c.plan()
        c.fold(np.zeros(E, np.uint64), 0)    # B_tot = 0 -> S unchanged except *alpha: publishes at t+1
        st = c.state()
        assert set(np.flatnonzero(st["tier"] == 1).tolist()) == _brute_hot(S, n_hot, tau)


# ------------------------------------------------------------------ replay invariants
def _replay(E=32, k=4, T=16, n_hot=6, s=1, alpha=0.9, Tp=4, W=8, dwell=8, L=2, steps=200,
            zipf=1.2, drift=16, frac=0.5, seed=0):
    c = oracle.Controller(E, n_hot, s, alpha, Tp, W, dwell, L)
    hist = []
    prev_ver = np.zeros(E, np.uint32)
    ntrans = 0
    for t in range(steps):
        lg = synth.trace_logits(seed, 0, t, T, E, zipf, drift, frac, n_top=n_hot)
        idx, gate = oracle.route(lg, k)
        _, mass = oracle.counts(idx, gate, E)
        c.fold(mass, T)
        p = c.plan()
        st = c.state()
        if p is not None:
            plan, fin = p
            if not fin:
                ntrans += len(plan)
                assert all(d != 0 for _, d, _ in plan)
            assert st["t"] == W or st["t"] % Tp == 0              # periodicity
        # invariants
        assert np.all(st["version"] >= prev_ver)
        prev_ver = st["version"].copy()
        nhigh = int((st["tier"] == 1).sum())
        pend_up = int((st["in_flight"] == 1).sum())
        pend_dn = int((st["in_flight"] == -1).sum())
        if st["t"] >= W:
            assert nhigh <= n_hot and nhigh + pend_up - pend_dn <= n_hot
        assert st["used_hi"] <= st["cap_hi"] and st["used_lo"] <= st["cap_lo"]
        for e in range(E):                                       # one stable slot per expert
            assert c.owner(st["tier"][e] == 1, int(st["slot"][e])) == e
        assert st["used_hi"] + st["used_lo"] == E + pend_up + pend_dn
        assert 0 <= st["S"].min() and st["S"].max() <= 1
        hist.append((st["tier"].tolist(), st["slot"].tolist(), st["version"].tolist()))
    return hist, ntrans, c


def test_replay_invariants_and_determinism():
    h1, n1, _ = _replay()
    h2, n2, _ = _replay()
    assert h1 == h2 and n1 == n2
    assert n1 >= 10                      # the drifting trace forces transitions (C1-like)


def test_budget_never_exceeded():
    H, I, g = 64, 128, 32
    Sh, Sl = oracle.slot_bytes(H, I, g, 16), oracle.slot_bytes(H, I, g, 4)
    E, s = 8, 1
    M = 2 * Sh + 6 * Sl + s * (Sh + Sl)
    n_hot = oracle.n_hot(M, E, Sh, Sl, s)
    assert n_hot == 2                                       # C1
    _, _, c = _replay(E=E, k=2, T=32, n_hot=n_hot, s=s, steps=120, drift=16)
    st = c.state()
    assert st["cap_hi"] * Sh + st["cap_lo"] * Sl <= M
    assert E * Sl <= M                                      # warmup layout fits too


@pytest.mark.parametrize("n_hot", [0, 32])
def test_corner_cases_no_transitions(n_hot):
    """n_hot = N: all HIGH after finalize, zero transitions; n_hot = 0: tau = +inf, zero."""
    _, ntrans, c = _replay(E=32, n_hot=n_hot, steps=100)
    st = c.state()
    assert ntrans == 0
    assert int((st["tier"] == 1).sum()) == n_hot
    if n_hot == 0:
        assert st["tau"] == float("inf")


def test_warmup_threshold_is_nth_score():
    """tau_h = n_hot-th largest score after warmup, then fixed."""
    c = oracle.Controller(4, 2, 1, 0.5, 4, 1, 0, 1)
    c.fold(np.array([0.9 * 2**24, 0.5 * 2**24, 0.1 * 2**24, 0], np.uint64), 1)
    plan, fin = c.plan()
    st = c.state()
    assert fin and st["tau"] == 0.5 * 0.5 and set(np.flatnonzero(st["tier"]).tolist()) == {0, 1}
    c2 = oracle.Controller(4, 2, 1, 0.5, 4, 1, 0, 1)
    c2.fold(np.array([0.3 * 2**24] * 4, np.uint64), 1)
    plan, _ = c2.plan()
    assert set(np.flatnonzero(c2.state()["tier"]).tolist()) == {0, 1}   # ties -> lower ids


def test_convergence_to_true_top_set():
    """Stationary Zipf(1.2): the HIGH set approaches the true top-n_hot (weakened to
    Jaccard >= 0.7 because near-equal Zipf ranks are not separable from a finite EMA window)."""
    E, n_hot, k, T = 128, 16, 8, 256
    js = []
    for seed in range(3):
        c = oracle.Controller(E, n_hot, 2, 0.95, 8, 32, 16, 2)
        for t in range(32 + 10 * 8 + 4):
            lg = synth.trace_logits(seed, 0, t, T, E, 1.2, 0, 0.0)
            idx, gate = oracle.route(lg, k)
            _, mass = oracle.counts(idx, gate, E)
            c.fold(mass, T)
            c.plan()
        hot = set(np.flatnonzero(c.state()["tier"] == 1).tolist())
        rank_of = synth.rank_perm(seed, 0, 0, E, 16, 0.0)
        true = set(np.flatnonzero(rank_of < n_hot).tolist())
        js.append(len(hot & true) / len(hot | true))
    assert np.mean(js) >= 0.7, js


def test_manual_command_semantics():
    """or_ctrl_command (Alg. 1 EnqueueUpgrade/EnqueueDowngrade for a chosen expert) against
    SPEC.md's op rules: range check, warm-up not finished, already at the tier, busy while in
    flight, lowest-free destination, exhausted -> deferred with the pool unchanged
    (SPEC.md:251), and publication L folds later with one alloc/free per transition."""
    E, n_hot, s, L = 6, 2, 1, 2
    c = oracle.Controller(E, n_hot, s, 0.9, 8, 4, 0, L)
    assert c.command(0, 1) == 1                              # warm-up not finished
    c.debug_set([0.9, 0.8, 0.1, 0.1, 0.1, 0.1], [1, 1, 0, 0, 0, 0], 0.5, 10)
    st0 = c.state()
    assert st0["cap_hi"] == n_hot + s and st0["cap_lo"] == E - n_hot + s
    assert c.command(6, 1) == 2 and c.command(-1, -1) == 2 and c.command(2, 0) == 2
    assert c.command(0, 1) == 1                              # already HIGH
    assert c.command(2, -1) == 1                             # already LOW
    assert c.command(2, 1) == 0                              # the one spare HIGH block
    st = c.state()
    assert st["in_flight"][2] == 1 and st["tier"][2] == 0   # not visible before publication
    free_hi = [b for b in range(st0["cap_hi"]) if c.owner(True, b) in (-1, 2)]
    assert c.owner(True, min(free_hi)) == 2                  # lowest free block
    assert c.command(2, 1) == 5                              # busy
    assert c.command(3, 1) == 4                              # exhausted: deferred, ledger unchanged
    assert c.state()["used_hi"] == st["used_hi"] and c.state()["in_flight"][3] == 0
    assert c.command(0, -1) == 0                             # demotion into the spare LOW block
    for _ in range(L - 1):
        c.fold(np.zeros(E, np.uint64), 1)
        assert c.state()["tier"][2] == 0
    c.fold(np.zeros(E, np.uint64), 1)                        # t + L: registration + reclaim
    st = c.state()
    assert st["tier"][2] == 1 and st["tier"][0] == 0 and st["in_flight"][2] == 0 and st["in_flight"][0] == 0
    assert st["version"][2] == st0["version"][2] + 1 and st["version"][0] == st0["version"][0] + 1
    assert st["used_hi"] == n_hot and st["used_lo"] == E - n_hot   # one alloc + one free per transition
    assert c.command(3, 1) == 0                              # the block expert 0 released is free again
