"""The workspace's partial-epoch protocol ("Group partials"): one workspace shared
by every kind of call -- lopa_confidence (K1 + fold kernel), lopa_debug_reduce_only (K1 alone,
no consumer) and lopa_step (K1 + the polling K2) -- in any interleaving, and replays of a
captured loop, must give exactly the results of fresh workspaces: a stale partial of an earlier
call is never folded as if it were fresh."""
import ctypes

import pytest
import torch

import _gpu as G

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def L():
    from paper_2512_16229_b200 import lopa
    lopa.lib()
    return lopa


@pytest.mark.parametrize("V,W,k", [(151936, 32, 7), (1000, 16, 3), (300000, 8, 2)])
def test_shared_workspace_interleaved_calls(L, V, W, k):
    tau = 0.9
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    ref = L.Stepper(V, W, k + 1, k, tau, DEV)
    tok, msk, nb = G.fresh_tables(k, W, DEV)
    logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
    L.syn_generate(3, 0, V, tok, msk, n_branches=1, out=logits[:1])
    o = ref.step(logits, nb, tok, msk)
    tok, msk, nb = o.next_tokens.clone(), o.next_mask.clone(), o.n_next.clone()
    n = int(nb.item())
    bufs = []
    for s in range(3):
        b = torch.zeros_like(logits)
        L.syn_generate(10 + s, 0, V, tok, msk, n_branches=n, out=b[:n])
        bufs.append(b)
    rows = (k + 1) * W
    status = L.new_status(DEV)
    lib, P = L.lib(), L._p
    stream = L._stream(torch.device(DEV))
    for it in range(9):
        b = bufs[it % 3]
        flat = b.view(rows, st.ld)
        kind = it % 3
        if kind == 0:   # a1 alone through lopa_confidence on the shared workspace
            c, a, s_ = L.confidence(flat, vocab=V, row_mask=msk.reshape(-1), workspace=st.ws)
            c2, a2, _ = L.confidence(flat, vocab=V, row_mask=msk.reshape(-1))
            torch.cuda.synchronize()
            m = msk.reshape(-1).bool()
            assert torch.equal(c[m].view(torch.int32), c2[m].view(torch.int32))
            assert torch.equal(a[m], a2[m])
        elif kind == 1:  # K1 alone (no consumer) leaves stamped partials behind
            st_ = lib.lopa_debug_reduce_only(P(flat), st.ld, rows, V, P(msk.reshape(-1).contiguous()),
                                             P(status), P(st.ws), st.ws.numel(), stream)
            assert st_ == 0
        # a fused step on the same workspace equals a fresh stepper's step
        o1 = st.step(b, nb, tok, msk)
        o2 = L.Stepper(V, W, k + 1, k, tau, DEV).step(b, nb, tok, msk)
        torch.cuda.synchronize()
        assert int(o1.status.item()) == 0 and int(status.item()) == 0
        sel = msk[:n].bool()
        assert torch.equal(o1.conf[:n][sel].view(torch.int32), o2.conf[:n][sel].view(torch.int32))
        assert int(o1.winner.item()) == int(o2.winner.item())
        nn = int(o1.n_next.item())
        assert nn == int(o2.n_next.item())
        assert torch.equal(o1.next_tokens[:nn], o2.next_tokens[:nn])
        assert torch.equal(o1.next_mask[:nn], o2.next_mask[:nn])


def test_graph_replays_keep_fresh_epochs(L):
    """A captured 6-iteration loop replayed 4 times from the same start: every replay equals the
    eager loop (the epoch lives in device memory, so replayed kernels with frozen parameters
    still stamp fresh epochs)."""
    V, W, k, tau = 1000, 16, 3, 0.9
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    tok, msk, nb = G.fresh_tables(k, W, DEV)
    bufs = []
    for s in range(2):
        b = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
        b.normal_(generator=torch.Generator(device=DEV).manual_seed(s))
        bufs.append(b.mul_(3))
    t0, m0, n0 = tok.clone(), msk.clone(), nb.clone()
    eager = L.Stepper(V, W, k + 1, k, tau, DEV)
    et, em, en = tok.clone(), msk.clone(), nb.clone()
    for i in range(6):
        o = eager.step(bufs[i % 2], en, et, em)
        et[:k + 1].copy_(o.next_tokens)
        em[:k + 1].copy_(o.next_mask)
        en.copy_(o.n_next)
    g = L.StepLoopGraph(st, bufs, nb, tok, msk, 6)
    for _ in range(4):
        tok.copy_(t0), msk.copy_(m0), nb.copy_(n0)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(tok, et) and torch.equal(msk, em) and torch.equal(nb, en)
