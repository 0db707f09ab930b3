"""Pins for the oracle's row reduction Conf(·) (readings R1, R2, R4).

Nothing here compares the oracle with itself: every expected value comes from a closed
form, 50-digit decimal arithmetic (oracle/brute.py), or a metamorphic relation.
"""
import math

import numpy as np
import pytest

from oracle import brute
from oracle import lopa_oracle as O
import syngen


def bits(vals):
    """float values -> bf16 bit patterns; asserts every value is bf16-exact."""
    f = np.asarray(vals, dtype=np.float32)
    b = f.view(np.uint32)
    assert np.all((b & 0xFFFF) == 0)
    return (b >> 16).astype(np.uint16)


NEG_INF = float("-inf")


@pytest.mark.parametrize("V,m,a,b", [(64, 1, 3.0, 0.0), (64, 3, 1.5, -0.25), (1000, 7, 8.0, 2.0),
                                     (151936, 1, 12.5, 0.0), (151936, 5, 20.0, -2.0), (8, 8, 1.0, 0.0)])
def test_two_level_row_closed_form(V, m, a, b):
    """A row holding a at m positions and b elsewhere: conf = 1/(m + (V-m) e^{b-a}),
    argmax = first a-position."""
    rng = np.random.default_rng(V * 31 + m)
    pos = np.sort(rng.choice(V, size=m, replace=False))
    row = np.full(V, b, dtype=np.float32)
    row[pos] = a
    conf, am, st = O.row_confidence(bits(row))
    expect = 1.0 / (m + (V - m) * math.exp(b - a))
    assert st == 0
    assert am == int(pos[0])
    assert abs(conf - expect) <= 1e-13 * max(1.0, expect)


@pytest.mark.parametrize("V", [1, 4, 64, 151936])
def test_flat_row(V):
    conf, am, st = O.row_confidence(bits(np.full(V, 0.75)))
    assert st == 0 and am == 0
    assert conf == pytest.approx(1.0 / V, rel=1e-14)


def test_uniform_over_four_is_quarter():
    """uniform over 4 -> 0.25 (exactly: exp(0) = 1 four times)."""
    conf, am, _ = O.row_confidence(bits([-1.0, -1.0, -1.0, -1.0]))
    assert conf == 0.25 and am == 0


@pytest.mark.parametrize("V,p", [(64, 17), (151936, 151935), (3, 0)])
def test_spike_over_neg_inf_is_one(V, p):
    """one-hot -> 1.0 (all other logits -inf)."""
    row = np.full(V, NEG_INF, dtype=np.float32)
    row[p] = 3.5
    conf, am, st = O.row_confidence(bits(row))
    assert (conf, am, st) == (1.0, p, 0)


def test_neg_inf_entries_contribute_nothing():
    rng = np.random.default_rng(5)
    row = (rng.integers(-128, 128, 64) / 64.0).astype(np.float32)
    row2 = row.copy()
    row2[::3] = NEG_INF
    c_sub, _, _ = O.row_confidence(bits(row[np.arange(64) % 3 != 0]))
    c2, _, _ = O.row_confidence(bits(row2))
    assert c2 == pytest.approx(c_sub, rel=1e-14)


@pytest.mark.parametrize("seed", range(40))
def test_matches_50_digit_exact(seed):
    """Oracle conf within 1e-12 of 50-digit decimal truth on random tiny bf16 rows."""
    rng = np.random.default_rng(seed)
    V = int(rng.integers(1, 65))
    scale = [1 / 64, 1 / 8, 1.0][seed % 3]
    row = (rng.integers(-200, 200, V) * scale).astype(np.float32)
    if seed % 5 == 0:          # duplicate maxima -> argmax tie
        row[rng.integers(0, V)] = row.max()
    b = bits(row)
    conf, am, st = O.row_confidence(b)
    exact, am_exact = brute.exact_row_confidence(b)
    assert st == 0
    assert am == am_exact
    assert abs(conf - float(exact)) <= 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_generator_rows_match_exact_at_moderate_V(seed):
    """Same pin on SYN-D2F rows at V=4096 (noise + spike structure of the workload)."""
    V, W = 4096, 8
    tok, msk = syngen.fresh_block(W)
    msk[seed % W] = 0
    row = syngen.gen_row(seed, 0, (seed + 1) % W, V, tok, msk)
    conf, am, _ = O.row_confidence(row)
    exact, am_exact = brute.exact_row_confidence(row)
    assert am == am_exact
    assert abs(conf - float(exact)) <= 1e-12


@pytest.mark.parametrize("seed", range(5))
def test_shift_invariance(seed):
    """Adding 1.0 to every entry of a generator row is bf16-exact and leaves softmax unchanged."""
    V = 151936 if seed == 0 else 4096
    tok, msk = syngen.fresh_block(8)
    row = syngen.gen_row(seed, 0, 3, V, tok, msk)
    f = syngen.bf16_bits_to_f32(row).astype(np.float64)
    shifted = bits((f + 1.0).astype(np.float32))
    c0, a0, _ = O.row_confidence(row)
    c1, a1, _ = O.row_confidence(shifted)
    assert a0 == a1
    assert c1 == pytest.approx(c0, rel=1e-13)


def test_permutation_invariance():
    rng = np.random.default_rng(9)
    V = 2048
    row = (rng.integers(-128, 128, V) / 64.0).astype(np.float32)
    row[77] = 9.0                      # unique max
    perm = rng.permutation(V)
    c0, a0, _ = O.row_confidence(bits(row))
    c1, a1, _ = O.row_confidence(bits(row[perm]))
    assert c1 == pytest.approx(c0, rel=1e-12)
    assert perm[a1] == a0 == 77


@pytest.mark.parametrize("bad", ["nan", "pinf", "allneg"])
def test_nonfinite_rows_flagged(bad):
    row = np.zeros(32, dtype=np.float32)
    if bad == "nan":
        row[5] = np.nan
    elif bad == "pinf":
        row[9] = np.inf
    else:
        row[:] = NEG_INF
    conf, am, st = O.row_confidence(bits(row) if bad != "nan" else
                                    (row.view(np.uint32) >> 16).astype(np.uint16))
    assert st == O.DEV_NONFINITE and am == -1 and math.isnan(conf)


def test_confidence_skips_unmasked_rows():
    L = np.stack([bits([0.0, 1.0]), bits([2.0, 0.0]), bits([0.0, 0.0])])
    conf, am, st = O.confidence(L, [1, 0, 1])
    assert am.tolist() == [1, -1, 0]
    assert math.isnan(conf[1])
    assert conf[0] == pytest.approx(1 / (1 + math.exp(-1)), rel=1e-15)
    assert conf[2] == 0.5
