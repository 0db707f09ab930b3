"""The device-resident D2F scheduler (lopa_d2f_*, NEXT-1 on the device, R25 / R26):
the whole multi-block decode -- harness forward of the device window, lopa_step with the window
read on the device, lopa_d2f_update -- issued with no host read, and captured in one CUDA graph.
Its trace (windows, branch counts, winners, commit order, forwards, final tokens) must equal the
oracle's D2F loop (oracle/d2f_oracle.py) on the same SYN-D2F forward."""
import numpy as np
import pytest
import torch

import syngen
from oracle import d2f_oracle as D

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def mods():
    from paper_2512_16229_b200 import d2f, lopa
    return d2f, lopa


def _oracle(seed, V, L, B, k, tau_add, tau_act, tau_conf, mw, extras):
    return D.decode_d2f(lambda b, t, m: syngen.gen_logits(seed, b, V, t, m, extras=extras),
                        L, B, k, tau_add, tau_act, tau_conf, max_window=mw)


def _assert_same(g, r):
    assert g.forwards == r.forwards
    assert g.windows == [tuple(w) for w in r.windows]
    assert g.branch_counts == r.branch_counts
    assert g.winners == r.winners
    assert g.commits == r.commits
    assert np.array_equal(g.tokens.cpu().numpy(), r.tokens)


CASES = [
    (0, 64, 48, 8, 3, 0.1, 256, 1), (1, 64, 48, 8, 3, 0.3, 24, 1), (2, 64, 32, 8, 2, 1.0, 256, 1),
    (3, 64, 32, 4, 5, 0.5, 12, 1), (4, 64, 64, 16, 7, 0.1, 256, 1), (5, 64, 256, 32, 3, 0.1, 256, 1),
    (6, 64, 40, 10, 2, 0.1, 30, 1),   # B = 10: fill ratio 1/10 == tau_add exactly (R26, double)
    (7, 151936, 96, 32, 7, 0.1, 256, 0),
]


@pytest.mark.parametrize("seed,V,L,B,k,tau_add,mw,extras", CASES)
def test_d2f_device_loop_vs_oracle(mods, seed, V, L, B, k, tau_add, mw, extras):
    d2f, lopa = mods
    cfg = d2f.BlockConfig(B, tau_add, 0.95, 0.9, mw)
    r = _oracle(seed, V, L, B, k, tau_add, 0.95, 0.9, mw, extras)
    loop = d2f.D2FDeviceLoop(L, k, cfg, V, DEV, seed, extras=extras)
    loop.reset()
    loop.run(r.forwards + 3)            # blind: the extra iterations must be no-ops
    torch.cuda.synchronize()
    assert loop.done() and int(loop.st.out.status.item()) == 0
    _assert_same(loop.trace(), r)


@pytest.mark.parametrize("seed,V,L,B,k,tau_add,mw,extras", [CASES[0], CASES[4], CASES[7]])
def test_d2f_device_loop_graph(mods, seed, V, L, B, k, tau_add, mw, extras):
    """The same decode captured in ONE CUDA graph (no host read between iterations), replayed
    twice from a reset: both replays reproduce the oracle's trace."""
    d2f, lopa = mods
    cfg = d2f.BlockConfig(B, tau_add, 0.95, 0.9, mw)
    r = _oracle(seed, V, L, B, k, tau_add, 0.95, 0.9, mw, extras)
    loop = d2f.D2FDeviceLoop(L, k, cfg, V, DEV, seed, extras=extras)
    loop.capture(r.forwards + 2)
    for _ in range(2):
        loop.reset()
        loop.replay()
        torch.cuda.synchronize()
        assert loop.done()
        _assert_same(loop.trace(), r)


def test_d2f_device_matches_host_pipeline_k15(mods):
    """configs[2] shape through the D2F pipeline (256 tokens, k = 15, windows up to 256): the
    device scheduler reproduces the host pipeline's trace (itself checked against the oracle in
    test_gpu_d2f.py)."""
    d2f, lopa = mods
    V, L, k, seed = 151936, 256, 15, 11
    cfg = d2f.BlockConfig(32, 0.1, 0.95, 0.9, 256)
    h = d2f.decode_d2f(lambda b, t, m: lopa.syn_generate(seed, b, V, t, m), L, k, cfg, V, DEV)
    loop = d2f.D2FDeviceLoop(L, k, cfg, V, DEV, seed)
    loop.reset()
    loop.run(h.forwards + 2)
    torch.cuda.synchronize()
    g = loop.trace()
    assert g.forwards == h.forwards and g.windows == h.windows and g.winners == h.winners
    assert g.branch_counts == h.branch_counts and g.commits == h.commits
    assert torch.equal(g.tokens, h.tokens)


@pytest.mark.parametrize("seed,V,L,B,k,tau_add,mw,extras,metric,param", [
    (20, 64, 32, 32, 0, 0.1, 256, 1, 0, 0.0),      # k = 0: the Eq. 1 baseline through the pipeline
    (21, 64, 256, 256, 3, 0.1, 256, 1, 0, 0.0),    # one block of 256 = the largest window
    (22, 64, 64, 8, 5, 0.1, 256, 1, 1, 3.0),       # Eq. 2 sliding-window minimum
    (23, 64, 64, 8, 5, 0.1, 256, 1, 2, 0.5),       # Eq. 2 least-confident half
    (24, 1000, 48, 16, 31, 0.1, 48, 0, 0, 0.0),    # k = 31 with windows capped at 48
])
def test_d2f_device_loop_edges(mods, seed, V, L, B, k, tau_add, mw, extras, metric, param):
    """Edge configurations of the device scheduler against the host pipeline (itself checked
    against the oracle), run as one self-terminating graph launch."""
    d2f, lopa = mods
    cfg = d2f.BlockConfig(B, tau_add, 0.95, 0.9, mw)
    h = d2f.decode_d2f(lambda b, t, m: lopa.syn_generate(seed, b, V, t, m, extras=extras), L, k, cfg, V, DEV,
                       metric=metric, metric_param=param)
    loop = d2f.D2FDeviceLoop(L, k, cfg, V, DEV, seed, extras=extras, metric=metric, metric_param=param)
    wg = loop.capture_while()
    loop.reset()
    loop.launch_while()
    torch.cuda.synchronize()
    g = loop.trace()
    assert wg.iterations() == h.forwards == g.forwards
    assert g.windows == h.windows and g.winners == h.winners and g.branch_counts == h.branch_counts
    assert g.commits == h.commits and torch.equal(g.tokens, h.tokens)
    wg.close()


def test_d2f_device_loop_matches_oracle_metric(mods):
    """An Eq. 2 variant through the device scheduler against the oracle's D2F loop directly."""
    d2f, lopa = mods
    V, L, B, k = 64, 48, 8, 4
    cfg = d2f.BlockConfig(B, 0.25, 0.95, 0.9, 256)
    r = D.decode_d2f(lambda b, t, m: syngen.gen_logits(30, b, V, t, m, extras=1), L, B, k, 0.25,
                     0.95, 0.9, max_window=256)
    loop = d2f.D2FDeviceLoop(L, k, cfg, V, DEV, 30, extras=1)
    loop.reset()
    loop.run(r.forwards + 2)
    torch.cuda.synchronize()
    _assert_same(loop.trace(), r)
