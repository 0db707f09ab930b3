"""Host logic of the D2F block pipeline (paper_2512_16229_b200/d2f.BlockPipeline; R26) against
the oracle's scheduler on random block states.  CPU only: no kernel is called."""
import numpy as np
import pytest

from oracle import d2f_oracle as D
from paper_2512_16229_b200 import d2f


@pytest.mark.parametrize("seed", range(20))
def test_block_pipeline_matches_oracle_scheduler(seed):
    rng = np.random.default_rng(seed)
    B = int(rng.choice([1, 4, 8, 32]))
    nblk = int(rng.integers(1, 9))
    tau_add = float(rng.choice([0.1, 0.3, 0.5, 1.0]))
    mw = int(rng.choice([B, 2 * B, 3 * B, 256 // B * B]))
    cfg = d2f.BlockConfig(B, tau_add, 0.95, 0.9, mw)
    pipe = d2f.BlockPipeline(nblk, cfg)
    status = [D.ACTIVE] + [D.INACTIVE] * (nblk - 1)
    mask = np.ones(nblk * B, np.uint8)
    for _ in range(200):
        win = D.active_window(status, B)
        assert pipe.window() == ((win[0], len(win)) if win else (0, 0))
        assert np.array_equal(np.float32(pipe.thresholds()), D.threshold_map(status, B, 0.95, 0.9))
        # fill a random subset of the window
        for p in win:
            if rng.random() < 0.3:
                mask[p] = 0
        new = D.schedule_blocks(status, mask, B, tau_add, mw)
        committed = pipe.update(mask.reshape(nblk, B).sum(axis=1).tolist())
        assert pipe.status == new
        assert committed == [b for b in range(nblk) if status[b] != D.COMMITTED and new[b] == D.COMMITTED]
        status = new
        if pipe.done():
            assert all(s == D.COMMITTED for s in status)
            break
