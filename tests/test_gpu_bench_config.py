"""Parity in the exact launch configuration bench.py times (BASELINE configs[1]): the same
workload builder, rotating buffers and prebuilt C-ABI argument structs, checked against the
oracle on the full step (241 masked rows x V = 151936)."""
import ctypes

import numpy as np
import pytest
import torch

import _gpu as G

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    from paper_2512_16229_b200 import lopa
    return bench, lopa


def test_bench_dream_step_matches_oracle(mods):
    bench, lopa = mods
    V, W, k, tau = 151936, 32, 7, 0.9
    st, tok, msk, nb, full, bufs, rows, _ = bench.build_workload(lopa, torch.device(DEV), V, W, k, tau, 1, 2)
    assert rows == 241
    L = lopa.lib()
    sptr = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = [st.args(b, nb, tok, msk) for b in bufs]
    for i in range(6):                       # the timed loop's launch pattern
        assert L.lopa_step(ctypes.byref(args[i % 2]), sptr) == 0
    torch.cuda.synchronize()
    n = int(nb.item())
    G.check_step(st.out, G.to_np_u16(bufs[1]), tok.cpu().numpy(), msk.cpu().numpy(), n, k, tau, vocab=V)


def test_bench_lmhead_rows_match_oracle(mods):
    """The lmhead-dream configuration (random-init projection from the torch generator, as in
    bench.run_lmhead): 6 sampled rows of the fused LM head + Conf against the fp64 oracle."""
    bench, lopa = mods
    from oracle import lmhead_oracle as LO
    V, Kd, rows = 151936, 3584, 256
    g = torch.Generator(device=DEV).manual_seed(1)
    Wt = (torch.randn(V, Kd, device=DEV, generator=g) / Kd ** 0.5).to(torch.bfloat16)
    H = (torch.randn(rows, Kd, device=DEV, generator=g) * 1.5).to(torch.bfloat16)
    c, a, st = lopa.LMHead(Wt)(H)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    h16 = H.view(torch.int16).cpu().numpy().view(np.uint16)
    w16 = Wt.view(torch.int16).cpu().numpy().view(np.uint16)
    sel = [0, 37, 128, 129, 200, 255]
    rc, ra, ok, Lg = LO.lmhead_confidence(h16, w16, sel)
    E = LO.logit_error_bound(h16, w16, sel)
    gc, ga = c.cpu().numpy(), a.cpu().numpy()
    for i, r in enumerate(sel):
        assert abs(gc[r] - rc[i]) <= rc[i] * np.expm1(2 * E[i]) + 2e-6
        srt = np.sort(Lg[i])[::-1]
        if srt[0] - srt[1] >= 2 * E[i]:
            assert ga[r] == ra[i]
