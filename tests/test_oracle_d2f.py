"""Pins for the D2F block-pipeline oracle (oracle/d2f_oracle.py, SPEC S:302-336,
reading R26).  CPU only."""
import numpy as np
import pytest

import syngen
from oracle import d2f_oracle as D
from oracle import lopa_oracle as O

I, A, C = D.INACTIVE, D.ACTIVE, D.COMMITTED


def test_active_window_spec_examples():
    # S:308-310
    assert D.active_window([C, A, A, I], 4) == list(range(4, 12))
    assert D.active_window([C, C, I], 4) == []
    assert D.active_window([A, A, A], 4) == list(range(12))


def test_threshold_map_newest_block_uses_tau_act():
    t = D.threshold_map([C, A, A, I], 4, 0.95, 0.9)
    assert t.tolist() == [np.float32(0.9)] * 4 + [np.float32(0.95)] * 4


def test_schedule_activation_ratio():
    """S:315 (b): activate when the newest active block's fill ratio >= tau_add.  SPEC's
    example S:318 says "3/32 filled, tau_add=0.1 -> activates (3/32 >= 0.1)", but
    3/32 = 0.094 < 0.1: the rule, not the example's arithmetic, is what R26 follows."""
    m = np.ones(64, np.uint8)
    m[:3] = 0
    assert D.schedule_blocks([A, I], m, 32, 0.1, 256) == [A, I]
    m[3] = 0
    assert D.schedule_blocks([A, I], m, 32, 0.1, 256) == [A, A]
    # window cap
    assert D.schedule_blocks([A, I], m, 32, 0.1, 32) == [A, I]


def test_schedule_commit_and_sequential():
    m = np.ones(12, np.uint8)
    m[:4] = 0                                   # block 0 full
    assert D.schedule_blocks([A, A, I], m, 4, 1.0, 256) == [C, A, I]
    # a full newer block behind a non-full older one is not committed (monotone)
    m = np.ones(12, np.uint8)
    m[4:8] = 0
    # (block 1 itself is full, so rule (b) opens block 2)
    assert D.schedule_blocks([A, A, I], m, 4, 1.0, 256) == [A, A, A]
    # tau_add = 1.0: the next block starts only when no block is active
    m = np.ones(8, np.uint8)
    m[:3] = 0
    assert D.schedule_blocks([A, I], m, 4, 1.0, 256) == [A, I]
    m[3] = 0
    assert D.schedule_blocks([A, I], m, 4, 1.0, 256) == [C, A]


def _fwd(seed, V, extras=1):
    return lambda b, t, m: syngen.gen_logits(seed, b, V, t, m, extras=extras)


@pytest.mark.parametrize("seed", range(4))
def test_single_block_equals_decode_block(seed):
    """block_size >= L_gen -> exactly the single-window Alg. 1 loop."""
    V, L, k = 64, 16, 3
    tr = D.decode_d2f(_fwd(seed, V), L, L, k, 0.1, 0.9, 0.5)
    ref = O.decode_block(lambda t, m: syngen.gen_logits(seed, 0, V, t, m, extras=1),
                         *syngen.fresh_block(L), k, 0.9)
    assert tr.forwards == ref.forwards and np.array_equal(tr.tokens, ref.tokens)
    assert tr.winners[1:] == ref.winners


@pytest.mark.parametrize("seed", range(4))
def test_tau_add_one_is_block_sequential(seed):
    """tau_add = 1.0 -> one active block at a time, and the run is exactly the
    per-block Alg. 1 loop repeated block after block (R22) with tau = tau_act."""
    V, B, nb, k = 64, 8, 4, 2
    tr = D.decode_d2f(_fwd(seed, V), B * nb, B, k, 1.0, 0.9, 0.5)
    toks, fw = [], 0
    for b in range(nb):
        r = O.decode_block(lambda t, m, b=b: syngen.gen_logits(seed, b, V, t, m, extras=1),
                           *syngen.fresh_block(B), k, 0.9)
        toks.append(r.tokens)
        fw += r.forwards
    assert tr.max_active == 1 and tr.commits == list(range(nb))
    assert tr.forwards == fw and np.array_equal(tr.tokens, np.concatenate(toks))


def test_one_hot_two_blocks_spec_example():
    """one-hot rows, tau_add = 1.0, 2 blocks of 4 -> each block is filled by one anchor
    (its initial predict fills all 4 positions), blocks in order: 2 forwards per block."""
    V = 16

    def fwd(b, t, m):
        out = np.full((t.shape[0], t.shape[1], V), 0xFF80, np.uint16)  # -inf
        for i in range(t.shape[1]):
            out[:, i, (3 * b + i) % V] = 0x3F80                        # 1.0
        return out

    tr = D.decode_d2f(fwd, 8, 4, 2, 1.0, 0.95, 0.9)
    assert tr.commits == [0, 1] and tr.forwards == 4
    assert tr.tokens.tolist() == [0, 1, 2, 3, 3, 4, 5, 6]
    assert tr.branch_counts == [1, 1, 1, 1]


@pytest.mark.parametrize("seed,tau_add,B,L", [(0, 0.1, 8, 48), (1, 0.3, 8, 48), (2, 0.5, 4, 32),
                                              (3, 0.1, 16, 64)])
def test_pipeline_invariants(seed, tau_add, B, L):
    """S:333-336 invariants on pipelined runs: commits in index order and complete, windows
    contiguous, within max_window and monotone, every position filled, tokens inside the
    vocabulary, and several blocks really overlap."""
    V, k = 64, 3
    tr = D.decode_d2f(_fwd(seed, V), L, B, k, tau_add, 0.95, 0.9, max_window=3 * B)
    assert tr.commits == list(range(L // B))
    assert tr.tokens_generated == L and np.all((tr.tokens >= 0) & (tr.tokens < V))
    starts = [w[0] for w in tr.windows]
    ends = [w[0] + w[1] for w in tr.windows]
    assert starts == sorted(starts) and ends == sorted(ends)
    assert all(w[1] % B == 0 and 0 < w[1] <= 3 * B for w in tr.windows)
    assert tr.max_active >= 2
    assert tr.forwards >= L // B


def test_no_fill_outside_window():
    """no token is ever filled in an inactive block — checked by recording every
    forward's inputs: positions outside the window are never handed to the model, and the
    committed prefix never changes after its commit."""
    V, B, L, k = 64, 8, 32, 3
    seen = []

    def fwd(b, t, m):
        seen.append((b, t.copy(), m.copy()))
        return syngen.gen_logits(5, b, V, t, m, extras=1)

    tr = D.decode_d2f(fwd, L, B, k, 0.1, 0.95, 0.9)
    first_seen = {}
    for idx, (b, t, m) in enumerate(seen):
        first_seen.setdefault(b, (t, m))
    for b, (t, m) in first_seen.items():
        assert np.all(m[0] == 1), f"block {b} had fills before it became active"
    for b in range(L // B):
        fin = tr.tokens[b * B:(b + 1) * B]
        last = [x for x in seen if x[0] == b][-1]
        # the last time a block is seen, its final tokens are its branches' filled tokens
        filled = last[2][0] == 0
        assert np.array_equal(last[1][0][filled], fin[filled])
