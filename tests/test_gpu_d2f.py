"""GPU parity of the D2F block pipeline (paper_2512_16229_b200/d2f.py, NEXT-1, R25,
R26): the product loop — one fused `lopa_step` per iteration over the multi-block window with
per-position thresholds — against the oracle loop (oracle/d2f_oracle.py) on the same SYN-D2F
forward.  Whole traces must agree: windows, branch counts, winners, commit order, final
tokens and forward counts."""
import numpy as np
import pytest
import torch

import syngen
from oracle import d2f_oracle as D

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2512_16229_b200 import d2f, lopa
    return d2f, lopa


def _compare(mods, seed, V, L, B, k, tau_add, tau_act, tau_conf, max_window, extras):
    d2f, lopa = mods
    cfg = d2f.BlockConfig(B, tau_add, tau_act, tau_conf, max_window)
    g = d2f.decode_d2f(lambda b, t, m: lopa.syn_generate(seed, b, V, t, m, extras=extras),
                       L, k, cfg, V, DEV)
    r = D.decode_d2f(lambda b, t, m: syngen.gen_logits(seed, b, V, t, m, extras=extras),
                     L, B, k, tau_add, tau_act, tau_conf, max_window=max_window)
    assert g.windows == r.windows
    assert g.branch_counts == r.branch_counts
    assert g.winners == r.winners
    assert g.commits == r.commits
    assert g.forwards == r.forwards
    assert np.array_equal(g.tokens.cpu().numpy(), r.tokens)
    return r


@pytest.mark.parametrize("seed,tau_add,B,L,k,mw", [
    (0, 0.1, 8, 48, 3, 256), (1, 0.3, 8, 48, 3, 24), (2, 1.0, 8, 32, 2, 256),
    (3, 0.5, 4, 32, 5, 12), (4, 0.1, 16, 64, 7, 256), (5, 0.1, 32, 256, 3, 256)])
def test_d2f_toy(mods, seed, tau_add, B, L, k, mw):
    r = _compare(mods, seed, 64, L, B, k, tau_add, 0.95, 0.9, mw, extras=1)
    if tau_add < 1.0:
        assert r.max_active >= 2


def test_d2f_dream_vocab(mods):
    """Dream vocabulary (V=151936), GSM8K D2F parameters (Appendix table, PAPER.md:528:
    block 32, tau_add 0.1, tau_act 0.95, tau_conf 0.90) with k=7, 3 blocks: windows up to 96."""
    r = _compare(mods, 7, 151936, 96, 32, 7, 0.1, 0.95, 0.9, 256, extras=0)
    assert max(w[1] for w in r.windows) > 64


def test_d2f_full_decode_k15_dream_vocab(mods):
    """BASELINE configs[2] shape on one GPU: a 256-token generation at V = 151936 with k = 15
    (16 branches), D2F GSM8K parameters (block 32, tau_add 0.1, tau_act 0.95, tau_conf 0.90,
    PAPER.md:528), windows up to 256 positions (4096 rows per step).  The whole run is checked
    for the pipeline invariants, and every 6th step against the oracle step on the
    same inputs (tests/_gpu.check_step: conf, argmax, scores, winner, anchor, spawn)."""
    import _gpu as G
    d2f, lopa = mods
    V, L_gen, k, seed = 151936, 256, 15, 11
    cfg = d2f.BlockConfig(32, 0.1, 0.95, 0.9, 256)
    checked = []

    def on_step(it, logits, tok, msk, n, taus, out):
        if it % 6 == 1 and n > 1 and len(checked) < 6:
            torch.cuda.synchronize()
            W = tok.shape[1]
            G.check_step(out, G.to_np_u16(logits[:n]), tok.cpu().numpy(), msk.cpu().numpy(), n, k,
                         np.asarray(taus, np.float32), vocab=V)
            checked.append((it, W))

    r = d2f.decode_d2f(lambda b, t, m: lopa.syn_generate(seed, b, V, t, m), L_gen, k, cfg, V, DEV,
                       on_step=on_step)
    toks = r.tokens.cpu().numpy()
    assert r.commits == list(range(L_gen // 32))
    assert np.all((toks >= 0) & (toks < V))
    assert all(w[1] % 32 == 0 and 0 < w[1] <= 256 for w in r.windows)
    starts = [w[0] for w in r.windows]
    assert starts == sorted(starts)
    assert max(w[1] for w in r.windows) >= 96 and len(checked) >= 3
    assert r.forwards < L_gen            # lookahead + pipelining fill > 1 token per forward
