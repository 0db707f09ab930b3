"""Pins for the oracle's verify step and decode loop (Alg. 1)."""
import numpy as np
import pytest

from oracle import brute
from oracle import lopa_oracle as O
import syngen


def one_hot_forward(V=16):
    """Every masked position is certain: logit 0 at token (i % V), -inf elsewhere."""
    def fwd(tok, msk):
        n, W = np.asarray(msk).shape
        out = np.full((n, W, V), 0xFF80, dtype=np.uint16)   # bf16 -inf
        for j in range(n):
            for i in range(W):
                out[j, i, i % V] = 0x0000
        return out
    return fwd


def syn_forward(seed, V=64, extras=syngen.EXTRAS_TIES_FLAT, blk=0):
    def fwd(tok, msk):
        return syngen.gen_logits(seed, blk, V, tok, msk, extras=extras)
    return fwd


def test_one_hot_tpf_is_three():
    """one-hot model, tau=.9, 6 tokens -> all filled by the first anchor; TPF = 6/2."""
    tok, msk = syngen.fresh_block(6)
    tr = O.decode_block(one_hot_forward(), tok, msk, k=3, tau=0.9)
    assert tr.forwards == 2 and tr.tokens_generated == 6 and tr.tpf == 3.0
    assert tr.tokens.tolist() == list(range(6))


def test_one_hot_baseline_one_forward():
    """baseline on one-hot rows finishes in one forward, TPF = L_gen."""
    tok, msk = syngen.fresh_block(6)
    tr = O.baseline_decode(one_hot_forward(), tok, msk, tau=0.9)
    assert tr.forwards == 1 and tr.tpf == 6.0


def test_tau_one_always_falls_back():
    """tau = 1.0 (strict >) -> always the fallback; one token per forward."""
    tok, msk = syngen.fresh_block(8)
    tr = O.baseline_decode(one_hot_forward(), tok, msk, tau=1.0)
    assert tr.per_step_fills == [1] * 8 and tr.tpf == 1.0
    tr2 = O.decode_block(one_hot_forward(), tok, msk, k=0, tau=1.0)
    assert tr2.per_step_fills == [1] * 8


@pytest.mark.parametrize("seed", range(12))
def test_k0_reduces_to_baseline(seed):
    """S:251 / S:266 (reading R19): k=0 visits the same states with the same fills as the
    Eq. 1 baseline and spends exactly one more forward (its final verify pass)."""
    W, tau = 8, [0.9, 0.5, 0.95][seed % 3]
    tok, msk = syngen.fresh_block(W)
    fwd = syn_forward(seed)
    a = O.decode_block(fwd, tok, msk, k=0, tau=tau)
    b = O.baseline_decode(fwd, tok, msk, tau=tau)
    assert a.tokens.tolist() == b.tokens.tolist()
    assert a.per_step_fills == b.per_step_fills
    assert a.forwards == b.forwards + 1


@pytest.mark.parametrize("seed", range(10))
def test_loop_invariants(seed):
    """>= 1 fill per iteration, W fills in total, <= k+1 branches and exactly
    k+1 whenever |M_B0| >= k."""
    W, k = 16, [1, 3, 7][seed % 3]
    tok, msk = syngen.fresh_block(W)
    fwd = syn_forward(seed, V=64)
    tr = O.decode_block(fwd, tok, msk, k=k, tau=0.9)
    assert sum(tr.per_step_fills) == W == tr.tokens_generated
    assert all(f >= 1 for f in tr.per_step_fills)
    assert all(1 <= b <= k + 1 for b in tr.branch_counts)
    assert tr.forwards == len(tr.per_step_fills) + 1


@pytest.mark.parametrize("seed", range(8))
def test_step_winner_matches_brute_force(seed):
    """S:447-455 / S:267-268: at every iteration, rebuild the branches from scratch, run one
    unbatched forward per branch, score Eq. 2 exactly and compare with the batched step;
    the carried conf equals a fresh recomputation on the winner's state."""
    V, W, k, tau = 64, 8, [2, 3, 4][seed % 3], 0.9
    fwd = syn_forward(seed, V=V)
    t32 = float(np.float32(tau))
    tok, msk = syngen.fresh_block(W)
    br_tok, br_msk = tok[None], msk[None]
    r = O.step(fwd(br_tok, br_msk), br_tok, br_msk, k, tau)
    state_conf, state_am = r.conf[0], r.argmax[0]
    state_tok, state_msk = br_tok[0], br_msk[0]
    iters = 0
    while not r.done:
        br_tok, br_msk = r.spawn.tokens, r.spawn.mask
        scores, best, branches = brute.brute_verify(fwd, state_tok, state_msk, state_conf,
                                                    state_am, t32, k)
        assert len(branches) == len(br_tok)
        for (t, m), bt, bm in zip(branches, br_tok, br_msk):
            assert list(t) == list(bt) and list(m) == list(bm)
        r = O.step(fwd(br_tok, br_msk), br_tok, br_msk, k, tau)
        gaps = sorted(float(s) for s in scores)
        if len(gaps) < 2 or gaps[-1] - gaps[-2] > 1e-12:
            assert r.winner == best
        for j, s in enumerate(scores):
            assert abs(r.scores[j] - float(s)) <= 1e-12
        w = r.winner
        fresh = O.confidence(fwd(br_tok[w:w + 1], br_msk[w:w + 1])[0], br_msk[w])
        m = br_msk[w].astype(bool)
        assert np.array_equal(fresh[1][m], r.argmax[w][m])
        assert np.allclose(fresh[0][m], r.conf[w][m], rtol=0, atol=1e-15)
        state_conf, state_am, state_tok, state_msk = r.conf[w], r.argmax[w], br_tok[w], br_msk[w]
        iters += 1
    assert iters >= 1


def test_step_done_when_winner_complete():
    W = 4
    tok = np.arange(W)
    msk = np.zeros((1, W), dtype=np.uint8)
    r = O.step(np.zeros((1, W, 8), dtype=np.uint16), tok[None], msk, k=2, tau=0.9)
    assert r.done and r.scores == [1.0] and r.n_branches_next == 0
