"""Pins for Eq. 1 (anchor), Alg. 1 top-k spawn and Eq. 2 verify/select in the oracle.

Expected values come from SPEC.md examples (tests/golden/, cited), literal set-builder /
exhaustive-subset evaluation (oracle/brute.py) and exact rational arithmetic.
"""
import itertools
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import brute
from oracle import lopa_oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_decode_examples.json")))


def dense(case):
    """Golden conf values are taken as fp32 numbers (reading R14: tau and conf are compared
    as fp32 values widened to double, so S:203's 'conf = 0.9 = tau' stays a tie)."""
    W = case["window"]
    conf = np.zeros(W)
    mask = np.zeros(W, dtype=np.uint8)
    for k, v in case["conf"].items():
        conf[int(k)] = float(np.float32(v))
        mask[int(k)] = 1
    return conf, mask


@pytest.mark.parametrize("case", GOLD["select_fill_set"], ids=lambda c: c["cite"])
def test_spec_select_fill_set(case):
    conf, mask = dense(case)
    d = O.select_fill_set(conf, mask, case["tau"])
    assert sorted(d.i_fill) == case["i_fill"] and d.fallback == case["fallback"]


@pytest.mark.parametrize("case", GOLD["anchor_step"], ids=lambda c: c["cite"])
def test_spec_anchor_step(case):
    conf, mask = dense(case)
    W = case["window"]
    argmax = np.arange(100, 100 + W)
    tokens = np.full(W, 7)
    a = O.anchor_fill(conf, argmax, tokens, mask, case["tau"])
    filled = [i for i in range(W) if mask[i] and not a.mask[i]]
    assert filled == case["filled"]
    assert [i for i in range(W) if a.mask[i]] == case["unfilled"]
    for i in range(W):
        assert a.tokens[i] == (argmax[i] if i in filled else 7)


@pytest.mark.parametrize("case", GOLD["spawn_lookahead"], ids=lambda c: c["cite"])
def test_spec_spawn(case):
    conf, mask = dense(case)
    W = case["window"]
    argmax = np.arange(50, 50 + W)
    s = O.spawn_branches(conf, argmax, np.zeros(W), mask, case["k"])
    assert s.lookahead == case["lookahead"]
    assert s.tokens.shape[0] == len(case["lookahead"]) + 1


@pytest.mark.parametrize("case", GOLD["branch_confidence"], ids=lambda c: c["cite"])
def test_spec_branch_confidence(case):
    conf, mask = dense(case)
    # inputs are fp32-rounded (see dense()), so the mean is exact only to ~1e-8
    assert O.branch_score(conf, mask) == pytest.approx(case["score"], abs=1e-7)


@pytest.mark.parametrize("case", GOLD["verify_branches"], ids=lambda c: c["cite"])
def test_spec_verify(case):
    assert O.verify_select(case["scores"]) == case["winner"]


def rand_map(rng, W, ties=True):
    """A random confidence map with deliberate ties and values on the tau boundary."""
    pool = [0.1, 0.25, 0.5, 0.9, float(np.float32(0.9)), 0.95, 0.99, 1.0]
    conf = np.array([rng.choice(pool) if (ties and rng.random() < 0.4) else rng.random() for _ in range(W)])
    mask = np.array([1 if rng.random() < 0.7 else 0 for _ in range(W)], dtype=np.uint8)
    return conf, mask


def test_eq1_law_1000_maps():
    """S:265 / S:509: 1000 random maps satisfy Eq. 1's piecewise definition exactly."""
    rng = random.Random(1)
    n = 0
    while n < 1000:
        W = rng.randint(1, 64)
        conf, mask = rand_map(rng, W)
        if not mask.any():
            with pytest.raises(O.EmptyMaskError):
                O.select_fill_set(conf, mask, 0.9)
            continue
        tau = rng.choice([0.5, 0.9, 0.95, 1.0, rng.random()])
        d = O.select_fill_set(conf, mask, tau)
        ref, fb = brute.brute_fill_set(conf, mask, float(np.float32(tau)))
        assert set(d.i_fill) == ref and d.fallback == fb
        assert len(d.i_fill) >= 1 and all(mask[i] for i in d.i_fill)
        n += 1


def test_anchor_all_masks_w8():
    """Brute force over every mask of an 8-position window (plus invariants)."""
    rng = random.Random(2)
    W = 8
    for trial in range(6):
        conf, _ = rand_map(rng, W)
        tau = [0.5, 0.9, 1.0][trial % 3]
        t32 = float(np.float32(tau))
        for bits_ in itertools.product([0, 1], repeat=W):
            mask = np.array(bits_, dtype=np.uint8)
            if not mask.any():
                continue
            argmax = np.arange(W) + 10
            a = O.anchor_fill(conf, argmax, np.zeros(W), mask, tau)
            fill = {i for i in range(W) if mask[i] and not a.mask[i]}
            ref, fb = brute.brute_fill_set(conf, mask, t32)
            assert fill == ref
            assert fill and fill <= {i for i in range(W) if mask[i]}
            if not fb:
                assert all(conf[i] > t32 for i in fill)
            rest = [conf[i] for i in range(W) if a.mask[i]]
            if rest:
                assert max(rest) <= t32      # nothing above tau survives the anchor
            assert all(a.tokens[i] == argmax[i] for i in fill)


def test_spawn_exhaustive_subsets():
    rng = random.Random(3)
    for _ in range(400):
        W = rng.randint(1, 8)
        conf, mask = rand_map(rng, W)
        k = rng.randint(0, 9)
        argmax = np.arange(W) + 1000
        s = O.spawn_branches(conf, argmax, np.arange(W), mask, k)
        assert s.lookahead == brute.brute_topk(conf, mask, k)
        nM = int(mask.sum())
        assert len(s.lookahead) == min(k, nM)
        # branches: distinct, each B0 plus exactly one more filled position
        rows = {tuple(s.tokens[j]) + tuple(s.mask[j]) for j in range(len(s.tokens))}
        assert len(rows) == len(s.tokens)
        for j, p in enumerate(s.lookahead, start=1):
            diff = [i for i in range(W) if s.mask[0][i] != s.mask[j][i]]
            assert diff == [p] and s.mask[0][p] == 1 and s.mask[j][p] == 0
            assert s.tokens[j][p] == argmax[p]


def test_scores_match_exact_rationals():
    rng = random.Random(4)
    for _ in range(300):
        n, W = rng.randint(1, 16), rng.randint(1, 64)
        confs = [[rng.random() for _ in range(W)] for _ in range(n)]
        masks = [[1 if rng.random() < 0.6 else 0 for _ in range(W)] for _ in range(n)]
        if rng.random() < 0.3:                      # an exact duplicate branch -> tie
            confs.append(list(confs[0]))
            masks.append(list(masks[0]))
        ours = [O.branch_score(c, m) for c, m in zip(confs, masks)]
        exact = brute.brute_branch_scores(confs, masks)
        for a, e in zip(ours, exact):
            assert abs(Fraction(a) - e) <= Fraction(1, 10 ** 15)
        w = O.verify_select(ours)
        assert w == brute.brute_winner(exact)
        assert all(ours[w] >= s for s in ours)


# ----------------------------------------------------------------------------- Eq. 2 variants
def test_spec_sliding_window_example():
    """confs in position order [.9,.2,.8], sliding_window(2) -> min(.55, .5) = 0.5."""
    conf = np.array([0.9, 0.2, 0.8])
    mask = np.ones(3, dtype=np.uint8)
    assert O.branch_score(conf, mask, O.METRIC_SLIDING_MIN, 2) == pytest.approx(0.5, abs=1e-15)


@pytest.mark.parametrize("seed", range(30))
def test_metric_variants_reduce_and_bound(seed):
    """Closed-form reductions of the Eq. 2 variants, exact rational checks, and
    the ordering min <= bottom-fraction <= mean <= ... that any correct implementation obeys."""
    rng = random.Random(seed)
    W = rng.randint(1, 20)
    conf = np.array([float(np.float32(rng.random())) for _ in range(W)])
    mask = np.array([rng.random() < 0.7 for _ in range(W)], dtype=np.uint8)
    vals = [conf[i] for i in range(W) if mask[i]]
    if not vals:
        for m, p in ((O.METRIC_SLIDING_MIN, 3), (O.METRIC_BOTTOM_FRACTION, 0.5)):
            assert O.branch_score(conf, mask, m, p) == 1.0
        return
    n = len(vals)
    mean = O.branch_score(conf, mask)
    # window >= n -> the mean; window 1 -> the minimum
    assert O.branch_score(conf, mask, O.METRIC_SLIDING_MIN, n + 3) == mean
    assert O.branch_score(conf, mask, O.METRIC_SLIDING_MIN, 1) == min(vals)
    # eta = 1 -> the mean; eta -> 0+ -> the minimum
    assert O.branch_score(conf, mask, O.METRIC_BOTTOM_FRACTION, 1.0) == pytest.approx(mean, abs=1e-15)
    assert O.branch_score(conf, mask, O.METRIC_BOTTOM_FRACTION, 1e-6) == min(vals)
    # exact rational recompute of a window / bottom mean
    w = rng.randint(1, n)
    exact_w = min(sum(Fraction(v) for v in vals[s:s + w]) / w for s in range(n - w + 1))
    assert abs(O.branch_score(conf, mask, O.METRIC_SLIDING_MIN, w) - float(exact_w)) < 1e-15
    eta = float(np.float32(rng.random()))
    b = -(-(Fraction(eta) * n).numerator // (Fraction(eta) * n).denominator)   # exact ceil
    exact_b = sum(sorted(Fraction(v) for v in vals)[:b]) / b
    assert abs(O.branch_score(conf, mask, O.METRIC_BOTTOM_FRACTION, eta) - float(exact_b)) < 1e-15
    # ordering
    assert min(vals) <= O.branch_score(conf, mask, O.METRIC_SLIDING_MIN, w) <= max(vals)
    assert min(vals) <= O.branch_score(conf, mask, O.METRIC_BOTTOM_FRACTION, eta) <= mean + 1e-15


# ----------------------------------------------------------------------------- per-position tau
@pytest.mark.parametrize("seed", range(40))
def test_per_position_tau_equals_blockwise_brute(seed):
    """Eq. 1 with a per-position threshold (D2F window, R25) equals the literal set-builder with
    each position's own tau (brute force), and reduces to the scalar rule for a constant map."""
    rng = random.Random(seed)
    W = rng.randint(1, 40)
    conf = np.array([float(np.float32(rng.choice([0.5, 0.9, 0.95, rng.random()]))) for _ in range(W)])
    mask = np.array([rng.random() < 0.7 for _ in range(W)], dtype=np.uint8)
    if not mask.any():
        mask[rng.randrange(W)] = 1
    taus = np.array([float(np.float32(rng.choice([0.9, 0.95, 0.7]))) for _ in range(W)])
    d = O.select_fill_set(conf, mask, taus)
    M = [i for i in range(W) if mask[i]]
    high = {i for i in M if conf[i] > taus[i]}
    if high:
        assert set(d.i_fill) == high and not d.fallback
    else:
        best = max(conf[i] for i in M)
        assert d.i_fill == [min(i for i in M if conf[i] == best)] and d.fallback
    const = O.select_fill_set(conf, mask, np.full(W, 0.9))
    assert const.i_fill == O.select_fill_set(conf, mask, 0.9).i_fill
