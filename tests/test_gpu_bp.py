"""Branch parallelism (a5) against the CPU oracle.

Every BP step -- each rank's local reduction + local Eq. 2 + record, the record exchange, and
the replicated global select / anchor / spawn -- is checked element by element against
oracle.step (tests/_gpu.check_step) on the step's own inputs, iterating to the end of the block,
for G = 1, 2, 4, 8 ranks (emulated on one GPU: the same kernels, the all-gather replaced by the
contiguous record array it produces).  Whole BP decode loops (Alg. 1) are compared
with the oracle's decode of BASELINE configs[2] (256 tokens, k = 15) and configs[3]
(DiffuCoder, k = 10, tau = 0.95), stored by scripts/make_golden_decode.py (oracle only).  The
real NCCL / peer-memory paths run with one rank (this environment has one GPU)."""
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest
import torch

import _gpu as G

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_decode_configs.json")))


@pytest.fixture(scope="module")
def L():
    from paper_2512_16229_b200 import lopa
    lopa.lib()
    return lopa


def _fwd(L, seed, blk, V, extras=0):
    return lambda t, m, out: L.syn_generate(seed, blk, V, t, m, extras=extras, out=out)


def _checked_bp_block(L, world, V, W, k, tau, seed, extras=0, blk=0):
    """One block decoded by BP over `world` emulated ranks; every step checked vs oracle.step."""
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    emu = L.BPEmulator(st, world)
    steps = [0]
    exempt = {}

    def on_step(out, n, tok, msk):
        torch.cuda.synchronize()
        logits = np.zeros((n, W, st.ld), dtype=np.uint16)
        for _, lo, hi, buf in emu.ranks():
            m = max(0, min(hi, n) - lo)
            if m:
                logits[lo:lo + m] = G.to_np_u16(buf[:m])
        conf, amax = emu.gathered()
        o = SimpleNamespace(conf=conf, argmax=amax, scores=emu.scores, winner=out.winner,
                            n_next=out.n_next, next_tokens=out.next_tokens, next_mask=out.next_mask,
                            lookahead=out.lookahead, status=out.status)
        G.check_step(o, logits, tok.cpu().numpy(), msk.cpu().numpy(), n, k, tau, exempt, vocab=V)
        steps[0] += 1

    tok0 = torch.zeros(W, dtype=torch.int32, device=DEV)
    msk0 = torch.ones(W, dtype=torch.uint8, device=DEV)
    tokens, fw = L.decode_block_bp(emu, _fwd(L, seed, blk, V, extras), tok0, msk0, on_step=on_step)
    assert fw == steps[0] and int(out_status(emu)) == 0
    return tokens.cpu().numpy(), fw


def out_status(emu):
    return emu.s.out.status.item()


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("V,W,k,tau,extras,seeds", [
    (64, 8, 2, 0.9, 1, range(6)),        # toy (configs[0]) with tied / flat rows
    (1000, 16, 10, 0.9, 0, range(2)),    # 11 branches: ragged shards (6+5, 3+3+3+2, 2x5+1, ...)
    (4096, 64, 31, 0.9, 0, range(1)),    # 32 branches, W = 64: shards with absent branches
])
def test_bp_steps_vs_oracle_small(L, world, V, W, k, tau, extras, seeds):
    for seed in seeds:
        _checked_bp_block(L, world, V, W, k, tau, seed, extras)


@pytest.mark.parametrize("world", [2, 8])
@pytest.mark.parametrize("k,tau,seed", [(7, 0.9, 1), (15, 0.9, 2), (10, 0.95, 3)])
def test_bp_steps_vs_oracle_dream(L, world, k, tau, seed):
    """Dream / DiffuCoder shapes (V = 151936, W = 32), every step of a block vs the oracle."""
    _checked_bp_block(L, world, 151936, 32, k, tau, seed)


def _bp_decode(L, bp, case):
    c = GOLDEN[case]
    toks, fws = [], []
    for blk in range(c["blocks"]):
        tok0 = torch.zeros(c["W"], dtype=torch.int32, device=DEV)
        msk0 = torch.ones(c["W"], dtype=torch.uint8, device=DEV)
        t, f = L.decode_block_bp(bp, _fwd(L, c["seed"], blk, c["V"]), tok0, msk0)
        toks.extend(t.cpu().numpy().tolist())
        fws.append(f)
    return toks, fws


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bp_decode_configs2_vs_oracle(L, world):
    """configs[2]: 256-token generation (8 blocks), k = 15, branch-parallel over `world` ranks:
    every generated token and every block's forward count equal the oracle's."""
    c = GOLDEN["dream_k15_256"]
    st = L.Stepper(c["V"], c["W"], c["k"] + 1, c["k"], c["tau"], DEV)
    toks, fws = _bp_decode(L, L.BPEmulator(st, world), "dream_k15_256")
    assert fws == c["forwards_per_block"]
    assert toks == c["tokens"]


@pytest.mark.parametrize("world", [1, 2, 4])
def test_bp_decode_configs3_vs_oracle(L, world):
    """configs[3]: D2F-DiffuCoder shape (k = 10, tau = 0.95), 4 blocks at 1 / 2 / 4 ranks."""
    c = GOLDEN["diffucoder_k10_128"]
    st = L.Stepper(c["V"], c["W"], c["k"] + 1, c["k"], c["tau"], DEV)
    toks, fws = _bp_decode(L, L.BPEmulator(st, world), "diffucoder_k10_128")
    assert fws == c["forwards_per_block"]
    assert toks == c["tokens"]


@pytest.mark.parametrize("p2p", [False, True])
def test_bp_decode_real_exchange_single_rank(L, p2p):
    """The real exchange (NCCL all-gather, or the peer-memory records + epoch flags) with one
    rank, driving the whole configs[2] decode: tokens and forwards equal the oracle's."""
    c = GOLDEN["dream_k15_256"]
    st = L.Stepper(c["V"], c["W"], c["k"] + 1, c["k"], c["tau"], DEV)
    bp = L.BranchParallel(st, 0, 1, p2p=p2p)
    try:
        toks, fws = _bp_decode(L, bp, "dream_k15_256")
        torch.cuda.synchronize()
        bp.check()
        assert int(st.out.status.item()) == 0
    finally:
        bp.close()
    assert fws == c["forwards_per_block"]
    assert toks == c["tokens"]


def test_bp_ragged_shards_match_single_gpu(L):
    """Ragged shards whose last ranks own fewer (or no) branches than b_loc (11 branches over
    2 / 4 / 8 ranks): the BP loop equals the single-GPU loop.  (The out-of-bounds mask read of
    ADVICE r1 is checked by compute-sanitizer memcheck on this test with the caching allocator
    off, profiles/r02_sanitizer.md.)"""
    V, W, k, tau = 1000, 16, 10, 0.9
    for world in (2, 4, 8):
        st = L.Stepper(V, W, k + 1, k, tau, DEV)
        emu = L.BPEmulator(st, world)
        tok0 = torch.zeros(W, dtype=torch.int32, device=DEV)
        msk0 = torch.ones(W, dtype=torch.uint8, device=DEV)
        t_bp, f_bp = L.decode_block_bp(emu, _fwd(L, 5, 0, V), tok0, msk0)
        t_1, f_1 = L.decode_block(_fwd(L, 5, 0, V), tok0, msk0, k, tau, V)
        assert f_bp == f_1 and torch.equal(t_bp, t_1)
