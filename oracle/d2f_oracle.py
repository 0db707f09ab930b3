"""D2F block-pipeline ORACLE — the LoPA loop over a multi-block active window.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this module.  It shares no code with the
CUDA path or with paper_2512_16229_b200/d2f.py (the product's scheduler is written separately);
the per-iteration step is :func:`oracle.lopa_oracle.step`.

Citation keys: ``P:n`` = /root/reference/PAPER.md line n; ``S:n`` = SPEC.md line n; readings
R25/R26 are DESIGN.md §2.

The paper says only "LoPA integrates seamlessly with D2F by treating all active blocks as a
single window for branch exploration" and names D2F's parameters (block size, tau_add,
tau_act, tau_conf; Appendix table).  The block semantics are SPEC's stand-in
(S:312-320), taken here as reading R26:

* the generation region is split into blocks of ``block_size`` positions, each inactive ->
  active -> committed;
* the window is the union of the active blocks' spans, contiguous because blocks
  activate and commit in index order;
* per-position Eq. 1 threshold (S:315 (c), R25): tau_act on the newest active block, tau_conf
  on the older ones;
* after each verify step, on the selected branch B* (the new x_{t+1}):
  (a) active blocks whose span is fully filled are committed, oldest first, stopping at the
      first one that is not full (commit order monotone);
  (b) if no block is active the next inactive block is activated; otherwise the next inactive
      block is activated when the newest active block's fill ratio >= tau_add (S:315 (b)) and
      the window stays within ``max_window`` positions;
* the spawned branches (built on the old window from the reused logits) carry over:
  committed columns are dropped (identical in every branch, since every branch extends
  B* there), newly activated columns are appended fully masked.  If the step completed the
  window (R21) the next forward is the new window's initial predict (a0, R17).

Parity pins: tests/test_oracle_d2f.py — SPEC's block examples, the single-block
reduction to the pinned Alg. 1 loop (block_size >= L_gen), the tau_add = 1
reduction to the sequential per-block loop, the one-hot two-block trace
and the pipeline invariants.  No function here is "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle import lopa_oracle as O

INACTIVE, ACTIVE, COMMITTED = 0, 1, 2


def active_window(status, block_size: int):
    """Positions of the active blocks: the union of their spans, in order."""
    pos = []
    for b, s in enumerate(status):
        if s == ACTIVE:
            pos.extend(range(b * block_size, (b + 1) * block_size))
    return pos


def threshold_map(status, block_size: int, tau_act: float, tau_conf: float) -> np.ndarray:
    """Eq. 1 thresholds over the window (S:315 (c)): newest active block -> tau_act, older
    active blocks -> tau_conf."""
    act = [b for b, s in enumerate(status) if s == ACTIVE]
    taus = []
    for b in act:
        t = tau_act if b == act[-1] else tau_conf
        taus.extend([t] * block_size)
    return np.array(taus, dtype=np.float32)


def schedule_blocks(status, mask, block_size: int, tau_add: float, max_window: int):
    """Rules (a) and (b) above.  ``mask`` is the full-region mask of the selected
    branch (1 = still masked).  Returns the new status list."""
    st = list(status)
    n = len(st)
    # (a) commit the oldest active blocks that are fully filled
    for b in range(n):
        if st[b] == COMMITTED:
            continue
        if st[b] != ACTIVE:
            break
        if int(np.sum(mask[b * block_size:(b + 1) * block_size])) == 0:
            st[b] = COMMITTED
        else:
            break
    act = [b for b in range(n) if st[b] == ACTIVE]
    nxt = next((b for b in range(n) if st[b] == INACTIVE), None)
    if nxt is None:
        return st
    if not act:
        st[nxt] = ACTIVE
        return st
    newest = act[-1]
    filled = block_size - int(np.sum(mask[newest * block_size:(newest + 1) * block_size]))
    # fill ratio >= tau_add, compared exactly: filled / block_size >= tau_add
    if filled / block_size >= float(tau_add) and (len(act) + 1) * block_size <= max_window:
        st[nxt] = ACTIVE
    return st


@dataclass
class D2FTrace:
    tokens: np.ndarray
    forwards: int = 0
    tokens_generated: int = 0
    windows: list = field(default_factory=list)     # (first position, width) per forward
    winners: list = field(default_factory=list)     # selected branch per forward
    branch_counts: list = field(default_factory=list)  # branches fed to each forward
    commits: list = field(default_factory=list)     # block indices in commit order
    max_active: int = 0

    @property
    def tpf(self) -> float:
        return self.tokens_generated / self.forwards if self.forwards else 0.0


def decode_d2f(forward_block, gen_len: int, block_size: int, k: int, tau_add: float,
               tau_act: float, tau_conf: float, max_window: int = 256, tokens0=None,
               max_forwards: int | None = None) -> D2FTrace:
    """LoPA over the D2F active window (P:217-218 + R26).

    ``forward_block(b, branch_tokens[n][block_size], branch_mask[n][block_size])`` returns the
    logits (uint16 bf16 bits [n][block_size][V]) of block b's positions for n branch states;
    a window forward is one call per active block, concatenated along the window (one forward
    pass for the whole window).  The region starts fully masked (tokens ``tokens0`` or 0)."""
    if gen_len % block_size:
        raise ValueError("generation length must be a multiple of block_size (S:324)")
    nblk = gen_len // block_size
    tok = np.zeros(gen_len, np.int64) if tokens0 is None else np.array(tokens0, np.int64)
    msk = np.ones(gen_len, np.uint8)
    status = [INACTIVE] * nblk
    status[0] = ACTIVE
    tr = D2FTrace(tokens=tok.copy())
    win = active_window(status, block_size)
    br_tok, br_msk = tok[None, win].copy(), msk[None, win].copy()
    while True:
        nb = br_tok.shape[0]
        parts = []
        for b in [x for x, s in enumerate(status) if s == ACTIVE]:
            off = win.index(b * block_size)
            parts.append(forward_block(b, br_tok[:, off:off + block_size], br_msk[:, off:off + block_size]))
        logits = np.concatenate(parts, axis=1)
        tr.forwards += 1
        tr.windows.append((win[0], len(win)))
        tr.branch_counts.append(nb)
        taus = threshold_map(status, block_size, tau_act, tau_conf)
        r = O.step(logits, br_tok, br_msk, k, taus)
        tr.winners.append(r.winner)
        tr.max_active = max(tr.max_active, sum(1 for s in status if s == ACTIVE))
        # x_{t+1} = B* on the window
        tok[win] = br_tok[r.winner]
        msk[win] = br_msk[r.winner]
        new_status = schedule_blocks(status, msk, block_size, tau_add, max_window)
        tr.commits.extend(b for b in range(nblk) if status[b] != COMMITTED and new_status[b] == COMMITTED)
        status = new_status
        if all(s == COMMITTED for s in status):
            break
        new_win = active_window(status, block_size)
        if r.done:
            nt, nm = tok[None, new_win].copy(), msk[None, new_win].copy()
        else:
            # carry the spawned branches over to the new window
            nbr = r.spawn.tokens.shape[0]
            nt = np.zeros((nbr, len(new_win)), np.int64)
            nm = np.zeros((nbr, len(new_win)), np.uint8)
            for c, p in enumerate(new_win):
                if p in win:
                    nt[:, c] = r.spawn.tokens[:, win.index(p)]
                    nm[:, c] = r.spawn.mask[:, win.index(p)]
                else:
                    nt[:, c] = tok[p]
                    nm[:, c] = msk[p]
        win, br_tok, br_msk = new_win, nt, nm
        if max_forwards is not None and tr.forwards >= max_forwards:
            break
    tr.tokens = tok.copy()
    tr.tokens_generated = int(gen_len - msk.sum())
    return tr
