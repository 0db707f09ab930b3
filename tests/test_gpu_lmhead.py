"""GPU parity of the fused LM-head + Conf kernel (NEXT-4, lopa_lmhead_confidence) against the
fp64 oracle (oracle/lmhead_oracle.py) on seeded SYN-LMH inputs.  Tolerance (R27): per row,
|conf - conf_ref| <= conf_ref·(exp(2E_r) - 1) + 2e-6 with E_r the fp32-accumulation bound;
argmax exact unless the oracle's top-2 logit gap is below 2E_r (then it must be one of the
tokens within 2E_r of the max)."""
import numpy as np
import pytest
import torch

import syngen
from oracle import lmhead_oracle as LO

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2512_16229_b200 import lopa
    return lopa


def _dev(u16):
    return torch.from_numpy(np.ascontiguousarray(u16).view(np.int16)).to(DEV).view(torch.bfloat16)


def _check(L, h, W, rows=None, stats=None):
    head = L.LMHead(_dev(W), max_rows=max(256, h.shape[0]))
    c, a, st = head(_dev(h))
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    g_c = c.cpu().numpy().astype(np.float64)
    g_a = a.cpu().numpy()
    sel = np.arange(h.shape[0]) if rows is None else np.asarray(rows)
    rc, ra, ok, Lg = LO.lmhead_confidence(h, W, sel)
    E = LO.logit_error_bound(h, W, sel)
    assert ok.all()
    for i, r in enumerate(sel):
        tol = rc[i] * np.expm1(2 * E[i]) + 2e-6
        assert abs(g_c[r] - rc[i]) <= tol, (r, g_c[r], rc[i], tol)
        srt = np.sort(Lg[i])[::-1]
        if srt.size > 1 and srt[0] - srt[1] < 2 * E[i]:
            assert Lg[i][g_a[r]] >= srt[0] - 2 * E[i]
        else:
            assert g_a[r] == ra[i], (r, g_a[r], ra[i])
        if stats is not None:
            stats.append(abs(g_c[r] - rc[i]) / rc[i])
    return g_c, g_a


@pytest.mark.parametrize("M,K,V", [(1, 64, 16), (7, 64, 100), (33, 128, 1000), (128, 256, 4096),
                                   (129, 64, 8200), (200, 192, 4111), (256, 128, 16),
                                   (256, 320, 5000), (64, 3584, 2048), (300, 128, 3000),
                                   (600, 64, 1000)])
def test_lmhead_shapes(L, M, K, V):
    """Rows > 256 run in chunks of 256 rows (one pass over the weights each)."""
    h, W, _ = syngen.lmhead_inputs(M * 7 + V, M, K, V)
    st = []
    _check(L, h, W, stats=st)
    assert np.mean(st) < 1e-4     # far inside the worst-case bound in practice


def test_lmhead_dream_size(L):
    """Dream-7B shapes: V = 151936 tokens, K = 3584, the 241 masked rows of the bench step;
    32 sampled rows against the oracle, plus every row's argmax against the planted token
    where the planted margin is large."""
    M, K, V = 241, 3584, 151936
    h, W, t = syngen.lmhead_inputs(2024, M, K, V)
    rows = list(range(0, M, 8)) + [M - 1]
    _check(L, h, W, rows=rows)


def test_lmhead_nonfinite(L):
    h, W, _ = syngen.lmhead_inputs(1, 4, 64, 300)
    h = h.copy()
    h[2, 5] = 0x7FC0   # NaN
    head = L.LMHead(_dev(W))
    c, a, st = head(_dev(h))
    torch.cuda.synchronize()
    assert int(st.item()) & L.DEV_NONFINITE
    assert int(a[2].item()) == -1 and np.isnan(float(c[2].item()))
    rc, ra, ok, _ = LO.lmhead_confidence(h, W, [0, 1, 3])
    assert a.cpu().numpy()[[0, 1, 3]].tolist() == ra.tolist()


def test_lmhead_repeatable(L):
    """Same inputs -> bit-identical outputs (fixed vocabulary split and fold order)."""
    h, W, _ = syngen.lmhead_inputs(77, 100, 256, 20000)
    head = L.LMHead(_dev(W))
    hd = _dev(h)
    c1, a1, _ = head(hd)
    c1, a1 = c1.clone(), a1.clone()
    for _ in range(3):
        c2, a2, _ = head(hd)
        assert torch.equal(c1, c2) and torch.equal(a1, a2)


def _oracle_decisions(conf, amax, tok, msk, n, k, tau):
    """Alg. 1 decisions (a2-a4) from per-row conf / argmax (oracle functions, fp64)."""
    from oracle import lopa_oracle as O
    scores = [O.branch_score(conf[j], msk[j]) for j in range(n)]
    w = O.verify_select(scores)
    if not msk[w].any():
        return scores, w, None, None
    anc = O.anchor_fill(conf[w], amax[w], tok[w], msk[w], tau)
    sp = O.spawn_branches(conf[w], amax[w], anc.tokens, anc.mask, k)
    return scores, w, anc, sp


@pytest.mark.parametrize("seed,V,K,W,k", [(0, 5000, 128, 32, 7), (1, 20000, 256, 16, 3),
                                          (2, 3000, 64, 64, 3), (3, 151936, 3584, 32, 7),
                                          (4, 8000, 128, 32, 14)])
def test_step_lmhead(L, seed, V, K, W, k):
    """lopa_step_lmhead (fused LM-head a1 + the step's a2-a4) against the oracle: conf within
    R27, and every decision exactly the oracle's decision on the GPU's own conf (and on the
    fp64 conf unless a near-tie within the conf tolerance governs)."""
    from oracle import lopa_oracle as O
    rng = np.random.default_rng(seed)
    nbr = k + 1
    h, Wt, _ = syngen.lmhead_inputs(seed, nbr * W, K, V)
    tok = rng.integers(0, V, size=(nbr, W)).astype(np.int32)
    msk = (rng.random((nbr, W)) < 0.7).astype(np.uint8)
    msk[:, 0] = 1
    n = nbr - 1 if seed % 2 else nbr      # also an absent last branch
    st = L.Stepper(V, W, nbr, k, 0.9, DEV)
    head = L.LMHead(_dev(Wt))
    nb = torch.tensor([n], dtype=torch.int32, device=DEV)
    out = head.step(st, _dev(h), nb, torch.from_numpy(tok).to(DEV), torch.from_numpy(msk).to(DEV))
    torch.cuda.synchronize()
    assert int(out.status.item()) == 0
    g_conf = out.conf.cpu().numpy().astype(np.float64).reshape(-1)[: n * W].reshape(n, W)
    g_amax = out.argmax.cpu().numpy().reshape(-1)[: n * W].reshape(n, W)
    sel = [r for r in range(n * W) if msk.reshape(-1)[r]]
    rc, ra, ok, Lg = LO.lmhead_confidence(h, Wt, sel)
    E = LO.logit_error_bound(h, Wt, sel)
    ref_conf = np.full((n, W), np.nan)
    ref_amax = np.full((n, W), -1)
    tol = np.zeros((n, W))
    for i, r in enumerate(sel):
        ref_conf[r // W, r % W], ref_amax[r // W, r % W] = rc[i], ra[i]
        tol[r // W, r % W] = rc[i] * np.expm1(2 * E[i]) + 2e-6
        assert abs(g_conf[r // W, r % W] - rc[i]) <= tol[r // W, r % W]
        srt = np.sort(Lg[i])[::-1]
        if srt[0] - srt[1] >= 2 * E[i]:
            assert g_amax[r // W, r % W] == ra[i]
    m = msk[:n].astype(bool)
    gc = np.where(m, g_conf, np.nan)
    # decisions exactly the oracle's on the GPU's own conf
    scores, w, anc, sp = _oracle_decisions(gc, g_amax, tok[:n], msk[:n], n, k, 0.9)
    assert out.scores.cpu().numpy()[:n].tolist() == [float(np.float32(x)) for x in scores]
    assert int(out.winner.item()) == O.verify_select([float(np.float32(x)) for x in scores])
    nn = int(out.n_next.item())
    if sp is not None:
        assert nn == len(sp.lookahead) + 1
        assert np.array_equal(out.next_tokens.cpu().numpy()[:nn], sp.tokens)
        assert np.array_equal(out.next_mask.cpu().numpy()[:nn], sp.mask)
    # and the fp64 oracle's decisions unless a near-tie within the conf tolerance governs
    r_scores, r_w, _, _ = _oracle_decisions(ref_conf, ref_amax, tok[:n], msk[:n], n, k, 0.9)
    srt = sorted(r_scores, reverse=True)
    if len(srt) < 2 or srt[0] - srt[1] > 2 * tol.max():
        assert int(out.winner.item()) == r_w


def test_lmhead_row_mask(L):
    """Rows with row_mask = 0 are not reported (conf NaN, argmax -1) and never flag the status;
    the selected rows equal the unmasked call's."""
    h, W, _ = syngen.lmhead_inputs(12, 50, 128, 900)
    head = L.LMHead(_dev(W))
    hd = _dev(h)
    c0, a0, _ = head(hd)
    c0, a0 = c0.clone(), a0.clone()
    rm = torch.from_numpy((np.arange(50) % 3 != 0).astype(np.uint8)).to(DEV)
    c1, a1, st = head(hd, row_mask=rm)
    torch.cuda.synchronize()
    sel = rm.bool()
    assert int(st.item()) == 0
    assert torch.equal(c1[sel], c0[sel]) and torch.equal(a1[sel], a0[sel])
    assert torch.isnan(c1[~sel]).all() and (a1[~sel] == -1).all()


@pytest.mark.parametrize("N", [16, 48, 112, 144, 240, 256, 272])
def test_lmhead_pair_tile_widths(L, N):
    """Rows 129..256 run on CTA pairs (tcgen05 cta_group::2, M = 256).  V = 74·N gives every pair
    of a B200 tiles of N columns (N = 272: two tiles of 128 + 144), so tile widths of an odd number
    of 16-column units (computed 16 columns wider, the extra columns ignored) are all exercised."""
    M, K, V = 256, 64, 74 * N
    h, W, _ = syngen.lmhead_inputs(N + 3, M, K, V)
    st = []
    _check(L, h, W, stats=st)
    assert np.mean(st) < 1e-4


def test_lmhead_pair_planted_columns(L):
    """Planted logits (row r: 8 at column c_r, 0 elsewhere) through the pair kernel: every argmax is
    exactly c_r and every conf equals 1 / (1 + (V - 1) e^-8) — a misplaced or duplicated weight
    row of either CTA's half shows up as a wrong column or a larger sum."""
    M = K = 256
    for V in (8200, 18944, 151936 // 4):
        h = np.zeros((M, K), np.float32)
        h[np.arange(M), np.arange(M)] = 1.0
        Wf = np.zeros((V, K), np.float32)
        c = (np.arange(M) * 7919) % V
        Wf[c, np.arange(M)] = 8.0
        hb = (h.view(np.uint32) >> 16).astype(np.uint16)
        Wb = (Wf.view(np.uint32) >> 16).astype(np.uint16)
        head = L.LMHead(_dev(Wb), max_rows=256)
        conf, am, st = head(_dev(hb))
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        assert am.cpu().numpy().tolist() == c.tolist()
        want = 1.0 / (1.0 + (V - 1) * np.exp(-8.0))
        assert np.allclose(conf.cpu().numpy(), want, rtol=1e-5)


@pytest.mark.parametrize("p2p", [False, True])
@pytest.mark.parametrize("seed,V,K,W,k", [(0, 5000, 128, 32, 7), (1, 20000, 256, 16, 3),
                                          (5, 8000, 128, 32, 14)])
def test_bp_step_lmhead_matches_one_gpu(L, p2p, seed, V, K, W, k):
    """lopa_bp_step_lmhead (one rank: the LM head on the shard's rows, then the NCCL or the
    fused peer-memory exchange with the decisions reading the LM head's conf) gives the same bits
    as lopa_step_lmhead (oracle-checked in test_step_lmhead): winner, scores, spawned tables,
    the rows' conf / argmax — including an absent last branch."""
    rng = np.random.default_rng(seed)
    nbr = k + 1
    h, Wt, _ = syngen.lmhead_inputs(seed, nbr * W, K, V)
    tok = torch.from_numpy(rng.integers(0, V, size=(nbr, W)).astype(np.int32)).to(DEV)
    m_np = (rng.random((nbr, W)) < 0.7).astype(np.uint8)
    m_np[:, 0] = 1
    msk = torch.from_numpy(m_np).to(DEV)
    n = nbr - 1 if seed % 2 else nbr
    nb = torch.tensor([n], dtype=torch.int32, device=DEV)
    hd, wd = _dev(h), _dev(Wt)
    st1 = L.Stepper(V, W, nbr, k, 0.9, DEV)
    o1 = L.LMHead(wd).step(st1, hd, nb, tok, msk)
    torch.cuda.synchronize()
    ref = {key: getattr(o1, key).clone() for key in ("winner", "n_next", "next_tokens", "next_mask", "scores", "status")}
    ref_conf, ref_amax = o1.conf.clone(), o1.argmax.clone()
    st2 = L.Stepper(V, W, nbr, k, 0.9, DEV)
    bp = L.BranchParallel(st2, 0, 1, p2p=p2p)
    try:
        o2 = bp.step_lmhead(hd, wd, nb, tok, msk)
        torch.cuda.synchronize()
        assert int(o2.status.item()) == int(ref["status"].item()) == 0
        assert int(o2.winner.item()) == int(ref["winner"].item())
        nn = int(o2.n_next.item())
        assert nn == int(ref["n_next"].item())
        assert torch.equal(o2.next_tokens[:nn], ref["next_tokens"][:nn])
        assert torch.equal(o2.next_mask[:nn], ref["next_mask"][:nn])
        assert torch.equal(bp.scores[:nbr].view(torch.int32), ref["scores"][:nbr].view(torch.int32))
        sel = torch.from_numpy(m_np.astype(bool)).to(DEV)
        sel[n:] = False
        assert torch.equal(bp.conf[sel].view(torch.int32), ref_conf[sel].view(torch.int32))
        assert torch.equal(bp.argmax[sel], ref_amax[sel])
    finally:
        bp.close()
