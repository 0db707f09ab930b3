"""Shared helpers for the `-m gpu` parity tests: drive liblopa through its binding and compare
with the CPU oracle on the same seeded SYN-D2F inputs.

Parity bar (BASELINE.json north_star):
* conf and branch scores within CONF_TOL = 1e-5 absolute (fp32 accumulation vs fp64 oracle);
* argmax tokens, filled-position sets, lookahead positions, branch tables, n_branches and the
  selected branch bit-exact, except "near-ties" (R16) whose governing oracle gap is < 1e-6;
* every GPU decision must ALSO be exactly the oracle's decision recomputed on the GPU's own fp32
  conf / scores (no exemption: the decisions are exact functions of those values).
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import lopa_oracle as O

CONF_TOL = 1e-5
NEAR_TIE = 1e-6


def to_np_u16(t: torch.Tensor) -> np.ndarray:
    return t.detach().view(torch.int16).cpu().numpy().view(np.uint16)


def fresh_tables(k: int, W: int, device):
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=device)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=device)
    msk[0] = 1
    nb = torch.ones(1, dtype=torch.int32, device=device)
    return tok, msk, nb


def decision_gaps(conf_w, mask_w, anchor_mask, k, tau, scores):
    """Governing gaps of the step's decisions (R16), from a conf row / scores (float64)."""
    gaps = {}
    s = sorted([x for x in scores if np.isfinite(x)], reverse=True)
    gaps["select"] = (s[0] - s[1]) if len(s) > 1 else np.inf
    M = [i for i in range(len(mask_w)) if mask_w[i]]
    if M:
        t = np.broadcast_to(np.asarray(tau, np.float32).astype(np.float64), (len(mask_w),))
        gaps["anchor"] = min(abs(float(conf_w[i]) - t[i]) for i in M)
        c = sorted((float(conf_w[i]) for i in M), reverse=True)
        gaps["fallback"] = (c[0] - c[1]) if len(c) > 1 else np.inf
    if anchor_mask is not None:
        M0 = [i for i in range(len(anchor_mask)) if anchor_mask[i]]
        c = sorted((float(conf_w[i]) for i in M0), reverse=True)[: k + 1]
        gaps["spawn"] = min((c[q] - c[q + 1] for q in range(len(c) - 1)), default=np.inf)
    return gaps


def check_step(out, logits_u16, tok, msk, n_br, k, tau, exempt_counter=None, vocab=None,
               metric=0, param=0.0):
    """Compare one fused-step output with the oracle on the same inputs.  Returns the oracle
    StepResult.  tok/msk: numpy [max_br][W]; logits_u16: numpy [>=n_br][W][ld]."""
    W = msk.shape[1]
    V_rows = logits_u16[:n_br, :, :vocab] if vocab else logits_u16[:n_br]   # the oracle reads V entries, not ld
    ref = O.step(V_rows, tok[:n_br], msk[:n_br], k, tau, metric, param)
    g_conf = out.conf.cpu().numpy()[:n_br].astype(np.float64)
    g_amax = out.argmax.cpu().numpy()[:n_br].astype(np.int64)
    g_scores = out.scores.cpu().numpy()[:n_br].astype(np.float64)
    g_w = int(out.winner.item())
    g_n = int(out.n_next.item())
    g_tok = out.next_tokens.cpu().numpy()
    g_msk = out.next_mask.cpu().numpy()
    g_look = out.lookahead.cpu().numpy()
    assert int(out.status.item()) == ref.status
    sel = msk[:n_br].astype(bool)
    # a1: conf within tolerance, argmax exact (bf16 compares are exact)
    assert np.all(np.isfinite(g_conf[sel]))
    err = np.abs(g_conf[sel] - ref.conf[sel])
    assert err.max(initial=0.0) <= CONF_TOL, f"conf err {err.max()}"
    assert np.array_equal(g_amax[sel], ref.argmax[sel])
    # a2: scores within tolerance
    assert np.max(np.abs(g_scores - np.array(ref.scores)), initial=0.0) <= CONF_TOL
    # decisions: exactly the oracle's decisions on the GPU's own fp32 values
    cs = [O.branch_score(np.where(sel, g_conf, np.nan)[j], msk[j], metric, param) for j in range(n_br)]
    # exact fp64 sums on both sides: the GPU score is the oracle's value (on GPU conf) rounded once
    assert [float(np.float32(x)) for x in cs] == [float(x) for x in g_scores]
    # fp32-rounded score ties -> lowest index (the GPU selects on its fp32 scores)
    gs32 = [float(np.float32(x)) for x in cs]
    assert g_w == O.verify_select(gs32)
    exempt = set()
    gaps = decision_gaps(ref.conf[ref.winner], msk[ref.winner],
                         None if ref.done else ref.anchor.mask, k, tau, ref.scores)
    for name, g in gaps.items():
        if g < NEAR_TIE:
            exempt.add(name)
    if exempt_counter is not None:
        for e in exempt:
            exempt_counter[e] = exempt_counter.get(e, 0) + 1
    if "select" not in exempt:
        assert g_w == ref.winner
    wref = g_w  # continue the GPU-self-consistency checks on the GPU's winner
    own_done = not np.asarray(msk[wref]).any()
    if own_done:
        assert g_n == 0
        assert np.array_equal(g_tok[0], tok[wref]) and np.array_equal(g_msk[0], msk[wref])
        return ref
    c = np.where(sel, g_conf, np.nan)
    anc = O.anchor_fill(c[wref], g_amax[wref], tok[wref], msk[wref], tau)
    sp = O.spawn_branches(c[wref], g_amax[wref], anc.tokens, anc.mask, k)
    n = len(sp.lookahead)
    assert g_n == n + 1
    assert np.array_equal(g_tok[: n + 1], sp.tokens) and np.array_equal(g_msk[: n + 1], sp.mask)
    assert g_look[:n].tolist() == sp.lookahead and all(x == -1 for x in g_look[n:k])
    # and against the fp64 oracle unless a near-tie governs
    if g_w == ref.winner and not ref.done and not (exempt & {"anchor", "fallback", "spawn"}):
        assert sp.lookahead == ref.spawn.lookahead
        assert np.array_equal(sp.tokens, ref.spawn.tokens) and np.array_equal(sp.mask, ref.spawn.mask)
    return ref
