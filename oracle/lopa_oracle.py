"""LoPA verify-step ORACLE — plain, slow, obviously correct CPU reference (NumPy float64).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this module.  It shares no code with
the CUDA path (paper_2512_16229_b200/), and the CUDA path never imports it.

Citation keys: ``P:n`` = /root/reference/PAPER.md line n; ``S:n`` = SPEC.md line n.
Readings R1..R18 refer to DESIGN.md §2 (= SURVEY.md §8(c) table).

Every function follows the paper's definition in the paper's order:

* :func:`row_confidence`   Conf(i) = top-1 softmax probability of position i's logits
  ("a confidence function Conf(·) assigns a score"; R1 top-1 prob, R2 T=1,
  R4 argmax tie -> lowest token id).  conf = 1 / sum_v exp(l_v - max l).
* :func:`select_fill_set`  Eq. 1: S_high = {i in M : Conf(i) > tau};
  I_fill = S_high if non-empty else {argmax_{i in M} Conf(i)} (R5 strict >, fallback tie ->
  lowest position; R14 tau compared as (double)(float)tau).
* :func:`anchor_fill`      Alg. 1 step 1: B0 = x_t with I_fill filled by the
  greedy token (R3), M_B0 = M_t \\ I_fill.
* :func:`spawn_branches`   Alg. 1 step 2: top-k of M_B0 by
  (conf desc, position asc) (R6), clamped to |M_B0| (R7); B_j = B0 + {p_j <- argmax}.
* :func:`branch_score`     Eq. 2: C(B_j) = mean_{i in M_Bj} Conf(i); 1.0 when
  M_Bj is empty (R8).
* :func:`verify_select`    Alg. 1 step 3: B* = argmax_j C(B_j), ties -> lowest
  j, i.e. anchor first (R9).
* :func:`step`             one verify step: reduce the branches' verify logits, score,
  select, then (logits reuse, R17) anchor + spawn on the winner's conf/argmax.
* :func:`decode_block`     Alg. 1 loop: repeat until the window is
  full; forwards = 1 (initial predict) + number of verify passes.

Parity pins: tests/test_oracle_*.py (closed forms, 50-digit exact arithmetic, brute force,
SPEC.md examples, invariants).  No function here is "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DEV_EMPTY_MASK = 1   # Eq. 1 applied with nothing masked
DEV_NONFINITE = 2    # a reduced row has NaN / +inf, or is all -inf


class EmptyMaskError(ValueError):
    """Eq. 1 on an empty masked set (S:199 'errors: empty confidence map')."""


# ----------------------------------------------------------------------------- input decode
def bf16_to_f64(u16) -> np.ndarray:
    """Exact decode of bf16 bit patterns: float64(uint32(u16) << 16 viewed as f32) (§8(c).1)."""
    u = np.asarray(u16, dtype=np.uint16)
    return (u.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def tau_as_f64(tau: float) -> float:
    """R14: tau is fp32 on the device side; the oracle compares against (double)(float)tau."""
    return float(np.float32(tau))


# ----------------------------------------------------------------------------- Conf(·)
def row_confidence(row_u16):
    """Conf and greedy token of one position (R1, R2, R4).

    Returns (conf, argmax, status).  m = max_v l_v; argmax = lowest v with l_v = m;
    conf = 1 / sum_v exp(l_v - m).  A row containing NaN or +inf, or whose entries are
    all -inf, is not a distribution: status = DEV_NONFINITE, conf = NaN, argmax = -1.
    """
    x = bf16_to_f64(row_u16)
    if x.size == 0 or np.isnan(x).any() or np.isposinf(x).any() or np.isneginf(x).all():
        return float("nan"), -1, DEV_NONFINITE
    m = x.max()
    a = int(np.argmax(x))          # first occurrence == lowest token id (R4)
    s = np.exp(x - m).sum()
    return float(1.0 / s), a, 0


def confidence(logits_u16, row_mask=None):
    """Conf / argmax for every masked row of logits[n_rows][>=V] (§8(a) a1).

    Unmasked rows are not reduced: conf = NaN, argmax = -1 in the result (the CUDA side
    leaves them untouched).  Returns (conf[n_rows], argmax[n_rows], status bits).
    """
    L = np.asarray(logits_u16, dtype=np.uint16)
    n = L.shape[0]
    conf = np.full(n, np.nan)
    amax = np.full(n, -1, dtype=np.int64)
    status = 0
    for r in range(n):
        if row_mask is not None and not row_mask[r]:
            continue
        c, a, st = row_confidence(L[r])
        conf[r], amax[r] = c, a
        status |= st
    return conf, amax, status


# ----------------------------------------------------------------------------- Eq. 1
@dataclass
class FillDecision:
    """S_high, I_fill and whether the 'otherwise' branch of Eq. 1 was taken."""
    s_high: list
    i_fill: list
    fallback: bool


def select_fill_set(conf, mask, tau) -> FillDecision:
    """Eq. 1 on the positions i with mask[i] = 1.

    ``tau`` is a scalar or, for the D2F multi-block window (reading R25), one
    threshold per window position (tau_act on the newest active block, tau_conf on older ones)."""
    taus = np.atleast_1d(np.asarray(tau, dtype=np.float64))
    M = [i for i in range(len(mask)) if mask[i]]
    if not M:
        raise EmptyMaskError("Eq. 1 with an empty masked set")
    def t_at(i):
        return tau_as_f64(taus[i] if taus.size > 1 else taus[0])
    s_high = [i for i in M if float(conf[i]) > t_at(i)]
    if s_high:
        return FillDecision(s_high, list(s_high), False)
    best = max(float(conf[i]) for i in M)
    i_star = min(i for i in M if float(conf[i]) == best)   # R5: fallback tie -> lowest i
    return FillDecision([], [i_star], True)


@dataclass
class Anchor:
    tokens: np.ndarray
    mask: np.ndarray
    decision: FillDecision


def anchor_fill(conf, argmax, tokens, mask, tau) -> Anchor:
    """Alg. 1 step 1: fill I_fill with greedy tokens; M_B0 = M_t minus I_fill."""
    d = select_fill_set(conf, mask, tau)
    tok = np.array(tokens, dtype=np.int64).copy()
    msk = np.array(mask, dtype=np.uint8).copy()
    for i in d.i_fill:
        tok[i] = int(argmax[i])
        msk[i] = 0
    return Anchor(tok, msk, d)


# ----------------------------------------------------------------------------- spawn
@dataclass
class Spawn:
    lookahead: list                 # p_1..p_n (n = min(k, |M_B0|))
    tokens: np.ndarray              # [n+1][W]; row 0 = B0
    mask: np.ndarray                # [n+1][W]


def spawn_branches(conf, argmax, tokens_b0, mask_b0, k: int) -> Spawn:
    """Alg. 1 step 2: top-k positions of M_B0 by confidence.

    Order: conf descending, then position ascending (R6); n = min(k, |M_B0|) (R7).
    B_j (j >= 1) is B0 with p_j additionally filled with its greedy token (R3).
    """
    M = [i for i in range(len(mask_b0)) if mask_b0[i]]
    order = sorted(M, key=lambda i: (-float(conf[i]), i))
    n = min(k, len(M))
    look = order[:n]
    W = len(mask_b0)
    tok = np.zeros((n + 1, W), dtype=np.int64)
    msk = np.zeros((n + 1, W), dtype=np.uint8)
    tok[0], msk[0] = tokens_b0, mask_b0
    for j, p in enumerate(look, start=1):
        tok[j], msk[j] = tokens_b0, mask_b0
        tok[j, p] = int(argmax[p])
        msk[j, p] = 0
    return Spawn(look, tok, msk)


# ----------------------------------------------------------------------------- Eq. 2 + select
METRIC_MEAN = 0            # Eq. 2
METRIC_SLIDING_MIN = 1     # P:204 "applying a sliding window to assess local quality"
METRIC_BOTTOM_FRACTION = 2 # P:204 "averaging confidence over the least confident segment"


def branch_score(conf_row, mask_row, metric: int = METRIC_MEAN, param: float = 0.0) -> float:
    """Branch confidence C(B_j) over the branch's own unfilled positions M_Bj, in position order.

    * METRIC_MEAN: Eq. 2, the arithmetic mean.
    * METRIC_SLIDING_MIN: the minimum over all length-w contiguous windows of
      the window mean, w = param clamped to |M_Bj| (reading R23: windows over the unfilled
      positions in position order, as S:228 states).
    * METRIC_BOTTOM_FRACTION: the mean of the ceil(eta * |M_Bj|) lowest
      confidences, eta = param (fp32, R14-style: ceil of (double)(float)eta * n, exact).
    1.0 if M_Bj is empty (R8).
    """
    vals = [float(conf_row[i]) for i in range(len(mask_row)) if mask_row[i]]
    if not vals:
        return 1.0
    n = len(vals)
    if metric == METRIC_MEAN:
        return float(sum(vals) / n)
    if metric == METRIC_SLIDING_MIN:
        w = min(int(param), n)
        return float(min(sum(vals[s:s + w]) / w for s in range(n - w + 1)))
    if metric == METRIC_BOTTOM_FRACTION:
        import math
        b = int(math.ceil(float(np.float32(param)) * n))
        low = sorted(vals)[:b]
        return float(sum(low) / b)
    raise ValueError("unknown branch-confidence metric")


def verify_select(scores) -> int:
    """Alg. 1 step 3: B* = argmax_j C(B_j); ties -> lowest j (anchor first, R9)."""
    best = max(scores)
    return min(j for j, s in enumerate(scores) if s == best)


# ----------------------------------------------------------------------------- one step
@dataclass
class StepResult:
    conf: np.ndarray          # [n_br][W] (NaN where unmasked)
    argmax: np.ndarray        # [n_br][W] (-1 where unmasked)
    scores: list              # [n_br]
    winner: int
    done: bool                # the winner has no masked position: block complete
    anchor: Anchor | None
    spawn: Spawn | None
    status: int = 0

    @property
    def n_branches_next(self) -> int:
        return 0 if self.done else len(self.spawn.lookahead) + 1


def step(logits_u16, branch_tokens, branch_mask, k: int, tau, metric: int = METRIC_MEAN,
         param: float = 0.0) -> StepResult:
    """One LoPA verify step over n_br branches' verify logits [n_br][W][>=V] (§8(a) a1-a4).

    a1 Conf/argmax of every masked (branch, position) row ("Compute scores ... Single
    Pass"); a2 Eq. 2 scores and argmax select; logits reuse: the winner's
    conf/argmax drive a3 the next anchor (Eq. 1) and a4 the next spawn (top-k).
    """
    L = np.asarray(logits_u16, dtype=np.uint16)
    n_br, W = np.asarray(branch_mask).shape
    conf = np.full((n_br, W), np.nan)
    amax = np.full((n_br, W), -1, dtype=np.int64)
    status = 0
    for j in range(n_br):
        c, a, st = confidence(L[j], branch_mask[j])
        conf[j], amax[j] = c, a
        status |= st
    scores = [branch_score(conf[j], branch_mask[j], metric, param) for j in range(n_br)]
    w = verify_select(scores)
    if not np.asarray(branch_mask[w]).any():
        return StepResult(conf, amax, scores, w, True, None, None, status)
    anc = anchor_fill(conf[w], amax[w], branch_tokens[w], branch_mask[w], tau)
    sp = spawn_branches(conf[w], amax[w], anc.tokens, anc.mask, k)
    return StepResult(conf, amax, scores, w, False, anc, sp, status)


# ----------------------------------------------------------------------------- the loop
@dataclass
class DecodeTrace:
    tokens: np.ndarray
    forwards: int = 0
    tokens_generated: int = 0
    per_step_fills: list = field(default_factory=list)
    winners: list = field(default_factory=list)
    branch_counts: list = field(default_factory=list)

    @property
    def tpf(self) -> float:
        return self.tokens_generated / self.forwards if self.forwards else 0.0


def decode_block(forward, tokens0, mask0, k: int, tau, max_iters: int | None = None) -> DecodeTrace:
    """Alg. 1 loop for one window.

    ``forward(branch_tokens[n][W], branch_mask[n][W]) -> logits[n][W][V]`` is the dLLM
    stand-in; one call = one forward pass regardless of how many branches are packed
    (S:278).  The first forward is the initial predict (a0, R17): its single "branch" is the
    starting state, which trivially wins.  Every later forward is a verify pass over the
    spawned branches; the winner's logits are reused for the next anchor.  The loop
    ends when the winner has no masked position; forwards = 1 + verify passes.
    per_step_fills[t] = masked(previous winner) - masked(winner of verify pass t).
    """
    tok = np.array(tokens0, dtype=np.int64)
    msk = np.array(mask0, dtype=np.uint8)
    tr = DecodeTrace(tokens=tok.copy())
    n0 = int(msk.sum())
    if n0 == 0:
        return tr
    br_tok, br_msk = tok[None, :].copy(), msk[None, :].copy()
    prev = n0
    while True:
        logits = forward(br_tok, br_msk)
        tr.forwards += 1
        r = step(logits, br_tok, br_msk, k, tau)
        if tr.forwards > 1:
            cnt = int(np.asarray(br_msk[r.winner]).sum())
            tr.per_step_fills.append(prev - cnt)
            tr.winners.append(r.winner)
            prev = cnt
        if r.done:
            tr.tokens = np.array(br_tok[r.winner], dtype=np.int64)
            break
        br_tok, br_msk = r.spawn.tokens, r.spawn.mask
        tr.branch_counts.append(len(r.spawn.lookahead) + 1)
        if max_iters is not None and tr.forwards >= max_iters:
            tr.tokens = np.array(br_tok[0], dtype=np.int64)
            break
    tr.tokens_generated = n0 - prev
    return tr


def baseline_decode(forward, tokens0, mask0, tau) -> DecodeTrace:
    """Confidence-driven sampling without lookahead: one forward per
    iteration followed by Eq. 1 fills, until the window is full.  Forwards = iterations
    (one-hot rows -> 1 forward).  Reading R19: LoPA with k=0 visits the same states
    and fills and spends exactly one more forward, its final verify pass."""
    tok = np.array(tokens0, dtype=np.int64)
    msk = np.array(mask0, dtype=np.uint8)
    tr = DecodeTrace(tokens=tok.copy())
    n0 = int(msk.sum())
    while msk.any():
        logits = forward(tok[None, :], msk[None, :])
        tr.forwards += 1
        conf, amax, _ = confidence(logits[0], msk)
        d = select_fill_set(conf, msk, tau)
        for i in d.i_fill:
            tok[i] = int(amax[i])
            msk[i] = 0
        tr.per_step_fills.append(len(d.i_fill))
    tr.tokens = tok
    tr.tokens_generated = n0
    return tr
