"""Independent checkers that pin the oracle (TEST INFRASTRUCTURE ONLY).

These re-derive the paper's definitions a second, different way — exact decimal
arithmetic, literal set-builder evaluation, exhaustive subset enumeration, unbatched
recomputation — so that a plausible mistake in `lopa_oracle.py` (a dropped term, a wrong
sign or index, a transposed operand) fails a test.  Pure Python (no NumPy) on purpose.
"""
from __future__ import annotations

import itertools
import struct
from decimal import Decimal, getcontext
from fractions import Fraction

getcontext().prec = 50


def bf16_bits_to_float(u: int) -> float:
    """Exact bf16 -> Python float via the IEEE single layout (bf16 = top half of an f32)."""
    return struct.unpack("<f", struct.pack("<I", (int(u) & 0xFFFF) << 16))[0]


def exact_row_confidence(row_bits):
    """conf = 1 / sum_v exp(l_v - m) at 50 significant digits (R1).

    Also returns the greedy token found by a literal scan (first index holding the max).
    """
    vals = [bf16_bits_to_float(u) for u in row_bits]
    m = vals[0]
    a = 0
    for v, x in enumerate(vals):
        if x > m:
            m, a = x, v
    mD = Decimal(m)
    s = Decimal(0)
    for x in vals:
        s += (Decimal(x) - mD).exp()
    return Decimal(1) / s, a


def brute_fill_set(conf, mask, tau32: float):
    """Eq. 1 evaluated literally as a set-builder over all positions.

    The fallback is 'the position i in M such that no j in M beats it', with 'beats'
    meaning larger conf, or equal conf at a lower position.
    """
    W = len(mask)
    M = {i for i in range(W) if mask[i]}
    S_high = {i for i in M if conf[i] > tau32}
    if S_high:
        return S_high, False
    cands = [i for i in M if not any(conf[j] > conf[i] or (conf[j] == conf[i] and j < i) for j in M)]
    assert len(cands) == 1
    return {cands[0]}, True


def brute_topk(conf, mask_b0, k: int):
    """Alg. 1 step 2 by exhaustive enumeration.

    Among all subsets T of M_B0 with |T| = min(k, |M_B0|), exactly one satisfies
    'every member of T beats every non-member' where beats = (conf, -position) greater.
    Returns that T ordered best first.
    """
    M = [i for i in range(len(mask_b0)) if mask_b0[i]]
    n = min(k, len(M))

    def beats(a, b):
        return conf[a] > conf[b] or (conf[a] == conf[b] and a < b)

    found = []
    for T in itertools.combinations(M, n):
        rest = [i for i in M if i not in T]
        if all(beats(a, b) for a in T for b in rest):
            found.append(T)
    assert len(found) == 1, found
    T = list(found[0])
    # order inside T: position p comes before q iff p beats q
    ordered = sorted(T, key=lambda p: sum(1 for q in T if beats(q, p)))
    return ordered


def brute_branch_scores(branch_confs, branch_masks):
    """Eq. 2 with exact rational arithmetic on each branch independently."""
    out = []
    for c, m in zip(branch_confs, branch_masks):
        idx = [i for i in range(len(m)) if m[i]]
        if not idx:
            out.append(Fraction(1))
        else:
            out.append(sum(Fraction(c[i]) for i in idx) / len(idx))
    return out


def brute_winner(scores):
    """argmax with ties -> lowest index, by scanning (R9)."""
    best = 0
    for j in range(1, len(scores)):
        if scores[j] > scores[best]:
            best = j
    return best


def brute_verify(forward, tokens_anchor_state, mask_anchor_state, conf_state, argmax_state, tau32, k):
    """S:447-455 pattern: rebuild B0..Bk from scratch, evaluate each branch with its own
    unbatched forward, compute Eq. 2 exactly, return (scores, best index, branches)."""
    W = len(mask_anchor_state)
    fill, _ = brute_fill_set(conf_state, mask_anchor_state, tau32)
    b0_tok = list(tokens_anchor_state)
    b0_msk = list(mask_anchor_state)
    for i in fill:
        b0_tok[i] = argmax_state[i]
        b0_msk[i] = 0
    look = brute_topk(conf_state, b0_msk, k)
    branches = [(b0_tok, b0_msk)]
    for p in look:
        t = list(b0_tok)
        m = list(b0_msk)
        t[p] = argmax_state[p]
        m[p] = 0
        branches.append((t, m))
    confs, masks = [], []
    for t, m in branches:
        logits = forward([t], [m])[0]          # one unbatched forward per branch
        c = [None] * W
        for i in range(W):
            if m[i]:
                cd, _ = exact_row_confidence(logits[i])
                c[i] = float(cd)
        confs.append(c)
        masks.append(m)
    scores = brute_branch_scores(confs, masks)
    return scores, brute_winner(scores), branches
