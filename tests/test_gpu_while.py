"""Device-terminated loops (lopa_while_*: a CUDA graph with a conditional WHILE node): the Alg. 1
loop of one window and the whole D2F decode run as ONE graph launch that stops on the device --
when the selected branch is complete (R21) / every block is committed -- with results equal to
the host-driven loops, which the other GPU tests check against the oracle."""
import numpy as np
import pytest
import torch

import syngen
from oracle import lopa_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def L():
    from paper_2512_16229_b200 import lopa
    lopa.lib()
    return lopa


@pytest.mark.parametrize("V,W,k,tau,extras,seeds", [(64, 8, 2, 0.9, 1, range(8)),
                                                    (151936, 32, 7, 0.9, 0, range(2)),
                                                    (151936, 32, 15, 0.9, 0, range(1)),
                                                    (1000, 64, 31, 0.95, 0, range(1))])
def test_decode_block_graph_vs_oracle(L, V, W, k, tau, extras, seeds):
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    for seed in seeds:
        g = L.DecodeBlockGraph(st, seed, 0, extras=extras)
        t0 = torch.zeros(W, dtype=torch.int32, device=DEV)
        m0 = torch.ones(W, dtype=torch.uint8, device=DEV)
        for _ in range(2):   # the same graph launched twice from the same start
            tok = g.run(t0, m0).clone()
            torch.cuda.synchronize()
            fw = g.forwards()
            fwd = lambda t, m: syngen.gen_logits(seed, 0, V, t, m, extras=extras)
            tok0, msk0 = syngen.fresh_block(W)
            ref = O.decode_block(fwd, tok0, msk0, k, tau)
            assert fw == ref.forwards
            assert np.array_equal(tok.cpu().numpy(), ref.tokens)
            assert int(st.out.status.item()) == 0
        g.graph.close()


def test_d2f_while_graph(L):
    """The whole D2F decode (256 tokens, k = 15, windows up to 256) as one self-terminating graph
    launch equals the host pipeline, launched twice."""
    from paper_2512_16229_b200 import d2f
    V, Lg, k, seed = 151936, 256, 15, 11
    cfg = d2f.BlockConfig(32, 0.1, 0.95, 0.9, 256)
    h = d2f.decode_d2f(lambda b, t, m: L.syn_generate(seed, b, V, t, m), Lg, k, cfg, V, DEV)
    loop = d2f.D2FDeviceLoop(Lg, k, cfg, V, DEV, seed)
    wg = loop.capture_while()
    for _ in range(2):
        loop.reset()
        loop.launch_while()
        torch.cuda.synchronize()
        g = loop.trace()
        assert wg.iterations() == h.forwards == g.forwards
        assert g.windows == h.windows and g.winners == h.winners and g.commits == h.commits
        assert torch.equal(g.tokens, h.tokens)
    wg.close()


def test_bp_decode_block_graph_nccl_single_rank(L):
    """The branch-parallel block loop (harness forward of the rank's branches, lopa_bp_step with
    its NCCL all-gather, table copies) as one device-terminated graph, one rank: the configs[2]
    blocks' tokens and forward counts equal the oracle's stored decode."""
    import json
    import os
    c = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_decode_configs.json")))["dream_k15_256"]
    st = L.Stepper(c["V"], c["W"], c["k"] + 1, c["k"], c["tau"], DEV)
    bp = L.BranchParallel(st, 0, 1)
    try:
        toks, fws = [], []
        for blk in range(3):
            g = L.DecodeBlockGraphBP(bp, c["seed"], blk)
            t = g.run(torch.zeros(c["W"], dtype=torch.int32, device=DEV),
                      torch.ones(c["W"], dtype=torch.uint8, device=DEV)).clone()
            torch.cuda.synchronize()
            toks.extend(t.cpu().tolist())
            fws.append(g.forwards())
            g.graph.close()
        bp.check()
    finally:
        bp.close()
    assert fws == c["forwards_per_block"][:3]
    assert toks == c["tokens"][: 3 * c["W"]]


def test_bp_decode_block_graph_p2p_single_rank(L):
    """The same BP block graph with the fused peer-memory exchange (epoch on the device), each
    block's graph launched twice: tokens and forwards equal the oracle's stored decode."""
    import json
    import os
    c = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_decode_configs.json")))["dream_k15_256"]
    st = L.Stepper(c["V"], c["W"], c["k"] + 1, c["k"], c["tau"], DEV)
    bp = L.BranchParallel(st, 0, 1, p2p=True)
    try:
        for blk in range(3):
            g = L.DecodeBlockGraphBP(bp, c["seed"], blk)
            for _ in range(2):
                t = g.run(torch.zeros(c["W"], dtype=torch.int32, device=DEV),
                          torch.ones(c["W"], dtype=torch.uint8, device=DEV)).clone()
                torch.cuda.synchronize()
                assert int(st.out.status.item()) == 0
                assert g.forwards() == c["forwards_per_block"][blk]
                assert t.cpu().tolist() == c["tokens"][blk * c["W"]:(blk + 1) * c["W"]]
            g.graph.close()
    finally:
        bp.close()
