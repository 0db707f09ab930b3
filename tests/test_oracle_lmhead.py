"""Pins for the LM-head + Conf oracle (oracle/lmhead_oracle.py; NEXT-4, reading R27).  CPU."""
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import syngen
from oracle import lmhead_oracle as LO
from oracle import lopa_oracle as O


def test_one_hot_hidden_rows_reduce_to_row_confidence():
    """h = e_k (bf16 1.0 at k) makes the logits exactly column k of W, so Conf must be the
    already-pinned row Conf of that column's bf16 values."""
    _, W, _ = syngen.lmhead_inputs(3, 1, 64, 500)
    for k in (0, 17, 63):
        h = np.zeros((1, 64), np.uint16)
        h[0, k] = 0x3F80
        c, a, ok, _ = LO.lmhead_confidence(h, W)
        rc, ra, st = O.row_confidence(W[:, k])
        assert ok[0] and st == 0 and a[0] == ra and c[0] == rc


def test_brute_force_exact_arithmetic():
    """Tiny shapes against exact rational logits and 50-digit exp sums."""
    getcontext().prec = 50
    h, W, _ = syngen.lmhead_inputs(5, 3, 64, 7)
    c, a, ok, _ = LO.lmhead_confidence(h, W)
    Hf = [[Fraction(float(x)) for x in row] for row in syngen.bf16_bits_to_f32(h)]
    Wf = [[Fraction(float(x)) for x in row] for row in syngen.bf16_bits_to_f32(W)]
    for r in range(3):
        l = [sum(hk * wk for hk, wk in zip(Hf[r], Wf[v])) for v in range(7)]
        m = max(l)
        am = l.index(m)
        s = sum(Decimal(float(x - m)).exp() for x in l)
        assert a[r] == am
        assert abs(c[r] - float(1 / s)) < 1e-15


def test_ties_take_lowest_token():
    W = np.zeros((6, 64), np.uint16)
    W[2, 0] = W[4, 0] = 0x4000   # 2.0 at tokens 2 and 4
    h = np.zeros((1, 64), np.uint16)
    h[0, 0] = 0x3F80
    c, a, ok, _ = LO.lmhead_confidence(h, W)
    assert a[0] == 2
    assert abs(c[0] - 1.0 / (2 + 4 * np.exp(-2.0))) < 1e-15


def test_nonfinite_row_flagged():
    W = np.zeros((4, 64), np.uint16)
    W[1, 3] = 0x3F80
    h = np.zeros((2, 64), np.uint16)
    h[0, 3] = 0x7F80   # +inf in row 0's hidden state: +inf and NaN (inf * 0) logits
    h[1, 5] = 0x3F80
    c, a, ok, _ = LO.lmhead_confidence(h, W)
    assert not ok[0] and ok[1] and a[0] == -1


@pytest.mark.parametrize("seed", range(3))
def test_error_bound_covers_fp32_accumulation(seed):
    """R27: every fp32 evaluation of the K-term sums (here: sequential and NumPy's float32
    matmul) stays within the bound, and the bound is not vacuous (< 1e-2 logit units)."""
    h, W, _ = syngen.lmhead_inputs(seed, 6, 512, 300)
    E = LO.logit_error_bound(h, W)
    L = LO.logits(h, W)
    H32 = syngen.bf16_bits_to_f32(h)
    W32 = syngen.bf16_bits_to_f32(W)
    mm = (H32 @ W32.T).astype(np.float64)
    seq = np.zeros_like(mm, dtype=np.float32)
    for k in range(512):
        seq = seq + np.outer(H32[:, k], W32[:, k]).astype(np.float32)
    for approx in (mm, seq.astype(np.float64)):
        assert np.all(np.abs(approx - L).max(axis=1) <= E)
    assert E.max() < 1e-2


def test_conf_perturbation_bound():
    """Logits each moved by at most E give a conf within conf·(exp(2E) - 1) (R27)."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        l = rng.normal(0, 3, 200)
        l[rng.integers(200)] += rng.uniform(0, 15)
        E = 10 ** rng.uniform(-6, -2)
        c, _, _ = LO.conf_from_logits(l)
        c2, _, _ = LO.conf_from_logits(l + rng.uniform(-E, E, 200))
        assert abs(c2 - c) <= c * np.expm1(2 * E) * (1 + 1e-9)


def test_generator_shape_and_spread():
    h, W, t = syngen.lmhead_inputs(9, 16, 128, 2000)
    assert h.shape == (16, 128) and W.shape == (2000, 128) and h.dtype == np.uint16
    c, a, ok, _ = LO.lmhead_confidence(h, W)
    assert ok.all() and (a == t).mean() > 0.8 and c.min() < 0.5 < c.max()


def test_neg_inf_logits_are_zero_probability():
    """R20 applied to exact logits: -inf entries are tokens of probability 0; only an all -inf
    row (or NaN / +inf) is not a distribution."""
    c, a, ok = LO.conf_from_logits(np.array([-np.inf, 1.0, 1.0, -np.inf]))
    assert ok and a == 1 and c == 0.5
    assert not LO.conf_from_logits(np.array([-np.inf, -np.inf]))[2]
    assert not LO.conf_from_logits(np.array([0.0, np.inf]))[2]
