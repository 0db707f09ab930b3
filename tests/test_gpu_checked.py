"""The checked build's own checks fire (negative control for the LOPA_CHECKED tier, which stands
in for compute-sanitizer on this pool).  Runs only with LOPA_LIB_VARIANT=checked."""
import ctypes
import os

import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _read(lopa):
    out = (ctypes.c_uint32 * 3)()
    st = lopa.lib().lopa_debug_check_read(ctypes.cast(out, ctypes.c_void_p))
    return st, list(out)


@pytest.mark.expect_violations
@pytest.mark.skipif(os.environ.get("LOPA_LIB_VARIANT") != "checked", reason="checked build only")
def test_checked_build_detects_contract_violation():
    from paper_2512_16229_b200 import lopa
    _read(lopa)  # reset
    V, W, k = 1000, 16, 2  # 3 branches over 2 ranks: b_loc = 2, rank 1 owns global rows 2..3
    st = lopa.Stepper(V, W, k + 1, k, 0.9, DEV)
    # tables allocated with spare rows (no real fault), but n_branches > max_branches breaks the
    # contract: the mask rows past the declared table must be reported (sites 2 / 5)
    tok = torch.zeros((2 * (k + 1), W), dtype=torch.int32, device=DEV)
    msk = torch.ones((2 * (k + 1), W), dtype=torch.uint8, device=DEV)
    logits = torch.zeros((2 * (k + 1), W, st.ld), dtype=torch.bfloat16, device=DEV)
    nb = torch.full((1,), k + 2, dtype=torch.int32, device=DEV)  # 4 > max_branches = 3
    emu = lopa.BPEmulator(st, 2)
    emu.step(nb, tok[: k + 1], msk[: k + 1])
    torch.cuda.synchronize()
    s, (count, first, sites) = _read(lopa)
    assert s == 0 and count > 0 and (sites & ((1 << 2) | (1 << 5))), (count, first, sites)
    # a clean call afterwards leaves no violation
    nb.fill_(1)
    lopa.syn_generate(1, 0, V, tok[: k + 1], msk[: k + 1], n_branches=1, out=logits[:1])
    st.step(logits[: k + 1], nb, tok[: k + 1], msk[: k + 1])
    torch.cuda.synchronize()
    assert _read(lopa)[1][0] == 0
