"""LM-head + Conf ORACLE — plain NumPy float64.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this module.  It shares no code with the
CUDA path (paper_2512_16229_b200/csrc/lopa_lmhead.cu).

Citation keys: ``P:n`` = PAPER.md line n; readings R1-R4, R27 are DESIGN.md §2.

The fused kernel computes, for each hidden-state row h_r (bf16) and the output projection W
(bf16, one row per token), the logits l_rv = sum_k h_rk W_vk and from them the paper's
Conf(·) (R1 top-1 softmax probability, R2 T = 1) and greedy token (R3, R4).  The
definition is written out here: the logits by a float64 matrix product of the exactly
widened bf16 values (each product h_rk W_vk is exact in float64; only the K-term sums round,
relative error ~K·2^-53), then conf = 1 / sum_v exp(l_v - max l), argmax = lowest v at max.

:func:`logit_error_bound` is reading R27's tolerance: the device accumulates in fp32, so
|l~_rv - l_rv| <= K·2^-23·sum_k |h_rk W_vk| (the classical bound for a K-term fp32 sum of
exact products, any order); a conf computed from logits that are each within E of the
exact ones lies within conf·(exp(2E) - 1) of the exact conf.

Parity pins: tests/test_oracle_lmhead.py — one-hot hidden rows reduce to the pinned row Conf,
exact rational logits with 50-digit exp sums, ties, non-finite rows, the error bound checked
against real fp32 evaluations, the conf perturbation bound.  No function is "parity unpinned".
"""
from __future__ import annotations

import numpy as np


def bf16_to_f64(u16) -> np.ndarray:
    """bf16 bit patterns -> float64 (exact widening)."""
    u = np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)


def logits(hidden_u16, weight_u16, rows=None, chunk: int = 16384) -> np.ndarray:
    """l[r][v] = sum_k h[r][k] W[v][k] in float64 for the selected rows (all by default)."""
    H = bf16_to_f64(hidden_u16 if rows is None else np.asarray(hidden_u16)[rows])
    Wu = np.asarray(weight_u16, dtype=np.uint16)
    out = np.empty((H.shape[0], Wu.shape[0]))
    with np.errstate(invalid="ignore", over="ignore"):
        for v0 in range(0, Wu.shape[0], chunk):
            out[:, v0:v0 + chunk] = H @ bf16_to_f64(Wu[v0:v0 + chunk]).T
    return out


def conf_from_logits(l):
    """Conf / greedy token of one row of exact logits (R1, R2, R4).  Returns
    (conf, argmax, ok).  As for rows of bf16 logits (R20): a row with a NaN or +inf logit,
    or whose logits are all -inf, is not a distribution (ok = False); a -inf logit is a
    token of probability 0."""
    l = np.asarray(l, dtype=np.float64)
    if np.isnan(l).any() or np.isposinf(l).any() or np.isneginf(l).all():
        return float("nan"), -1, False
    m = l.max()
    return float(1.0 / np.exp(l - m).sum()), int(np.argmax(l)), True


def lmhead_confidence(hidden_u16, weight_u16, rows=None):
    """conf[r], argmax[r], ok[r] for every (selected) row, straight from the definition."""
    L = logits(hidden_u16, weight_u16, rows)
    res = [conf_from_logits(L[i]) for i in range(L.shape[0])]
    return (np.array([r[0] for r in res]), np.array([r[1] for r in res], dtype=np.int64),
            np.array([r[2] for r in res]), L)


def logit_error_bound(hidden_u16, weight_u16, rows=None, chunk: int = 16384) -> np.ndarray:
    """E_r = K·2^-23·max_v sum_k |h_rk W_vk| (R27) for the selected rows."""
    H = np.abs(bf16_to_f64(hidden_u16 if rows is None else np.asarray(hidden_u16)[rows]))
    Wu = np.asarray(weight_u16, dtype=np.uint16)
    K = H.shape[1]
    best = np.zeros(H.shape[0])
    for v0 in range(0, Wu.shape[0], chunk):
        best = np.maximum(best, (H @ np.abs(bf16_to_f64(Wu[v0:v0 + chunk])).T).max(axis=1))
    return K * 2.0 ** -23 * best
