"""Small driver that exercises every liblopa kernel once, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck).  Run with PYTORCH_NO_CUDA_MEMORY_CACHING=1 so that every
tensor is its own exact-size cudaMalloc (memcheck then sees out-of-bounds reads that the caching
allocator's rounding would hide).  Sizes are small but span several tiles and ragged tails.

    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck python scripts/sanitize_drive.py
    ... [--part core|bp|lmhead|all]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_16229_b200 import lopa  # noqa: E402

DEV = torch.device("cuda:0")


def fresh(k, W):
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=DEV)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=DEV)
    msk[0] = 1
    nb = torch.ones(1, dtype=torch.int32, device=DEV)
    return tok, msk, nb


def block(V, W, k, tau, seed, steps=3, extras=0, tau_pos=None):
    """K1 + K2 (lopa_step), a few chained steps of one block."""
    st = lopa.Stepper(V, W, k + 1, k, tau, DEV, tau_pos=tau_pos)
    tok, msk, nb = fresh(k, W)
    logits = torch.empty((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
    for _ in range(steps):
        n = int(nb.item())
        lopa.syn_generate(seed, 0, V, tok, msk, n_branches=n, extras=extras, out=logits[:n])
        if n < k + 1:
            logits[n:].fill_(0)
        out = st.step(logits, nb, tok, msk)
        if int(out.n_next.item()) == 0:
            break
        tok, msk, nb = out.next_tokens.clone(), out.next_mask.clone(), out.n_next.clone()
    torch.cuda.synchronize()
    assert int(out.status.item()) == 0, int(out.status.item())
    return st, tok, msk, nb


def part_core():
    # a1 alone: ragged vocabularies, a row mask, -inf / flat rows
    for V, R in ((64, 24), (8193, 37), (151936, 12)):
        ld = (V + 7) // 8 * 8
        x = (torch.randn((R, ld), device=DEV) * 3).to(torch.bfloat16)
        x[1] = float("-inf")
        x[1, 3] = 2.0
        m = (torch.arange(R, device=DEV) % 3 != 0).to(torch.uint8)
        lopa.confidence(x, vocab=V)
        lopa.confidence(x, vocab=V, row_mask=m)
    # fused steps: toy with ties / flat rows, Dream k = 7, D2F window W = 256 with tau_pos
    block(64, 8, 2, 0.9, 0, extras=1)
    block(151936, 32, 7, 0.9, 1, steps=2)
    tp = torch.full((256,), 0.9, dtype=torch.float32, device=DEV)
    tp[224:] = 0.7
    block(4096, 256, 3, 0.9, 2, steps=2, tau_pos=tp)
    # standalone decision kernels (a2 / a3 / a4) and the Eq. 2 variants
    W, k = 32, 7
    conf = torch.rand((k + 1, W), device=DEV)
    amax = torch.randint(0, 1000, (k + 1, W), dtype=torch.int32, device=DEV)
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=DEV)
    msk = (torch.rand((k + 1, W), device=DEV) < 0.7).to(torch.uint8)
    nb = torch.full((1,), k + 1, dtype=torch.int32, device=DEV)
    lopa.anchor_fill(conf[0], amax[0], tok[0], msk[0], 0.9)
    lopa.spawn_branches(conf[0], amax[0], tok[0], msk[0], k)
    for metric, param in ((lopa.METRIC_MEAN, 0.0), (lopa.METRIC_SLIDING_MIN, 4.0),
                          (lopa.METRIC_BOTTOM_FRACTION, 0.25)):
        lopa.verify_select(conf, msk, nb, metric, param)
    # the captured Alg. 1 loop
    st = lopa.Stepper(1000, 16, 4, 3, 0.9, DEV)
    tok, msk, nb = fresh(3, 16)
    bufs = [torch.empty((4, 16, st.ld), dtype=torch.bfloat16, device=DEV) for _ in range(2)]
    for b in bufs:
        lopa.syn_generate(3, 0, 1000, tok, msk, n_branches=1, out=b[:1])
        b[1:].fill_(0)
    g = lopa.StepLoopGraph(st, bufs, nb, tok, msk, 4)
    g.replay()
    torch.cuda.synchronize()


def part_bp():
    # emulated ranks: local kernels (ragged shards, absent branches) + the global half
    for world in (2, 4, 8):
        st = lopa.Stepper(1000, 16, 11, 10, 0.9, DEV)
        emu = lopa.BPEmulator(st, world)
        t0 = torch.zeros(16, dtype=torch.int32, device=DEV)
        m0 = torch.ones(16, dtype=torch.uint8, device=DEV)
        fwd = lambda t, m, out: lopa.syn_generate(5, 0, 1000, t, m, out=out)
        lopa.decode_block_bp(emu, fwd, t0, m0)
    torch.cuda.synchronize()
    # the real exchanges with one rank: NCCL all-gather, peer-memory publish / flags, and the
    # Commit-Winner-Cache payloads (NCCL all-reduce form and the peer-memory pull)
    V, W, k = 151936, 32, 7
    for p2p in (False, True):
        st = lopa.Stepper(V, W, k + 1, k, 0.9, DEV)
        bp = lopa.BranchParallel(st, 0, 1, p2p=p2p, payload_bytes=4096 if p2p else 0)
        t0 = torch.zeros(W, dtype=torch.int32, device=DEV)
        m0 = torch.ones(W, dtype=torch.uint8, device=DEV)
        fwd = lambda t, m, out: lopa.syn_generate(6, 0, V, t, m, out=out)
        lopa.decode_block_bp(bp, fwd, t0, m0, max_forwards=3)
        pay = torch.arange(bp.b_loc * 4096, dtype=torch.int32, device=DEV).to(torch.uint8).view(bp.b_loc, 4096)
        if p2p:
            bp.payload_view(0).copy_(pay)
            bp.payload_view(1).copy_(pay)
            bp.commit_winner_p2p(torch.empty(4096, dtype=torch.uint8, device=DEV))
        else:
            bp.commit_winner(pay)
        torch.cuda.synchronize()
        bp.check()
        bp.close()


def part_lmhead():
    K, V, rows = 128, 1000, 200
    w = (torch.randn((V, K), device=DEV) / K ** 0.5).to(torch.bfloat16)
    h = (torch.randn((rows, K), device=DEV) * 1.5).to(torch.bfloat16)
    head = lopa.LMHead(w, max_rows=256)
    c, a, s = head(h)
    m = (torch.arange(rows, device=DEV) % 4 != 0).to(torch.uint8)
    head(h, row_mask=m)
    k, W = 3, 32
    st = lopa.Stepper(V, W, k + 1, k, 0.9, DEV)
    tok, msk, nb = fresh(k, W)
    hs = (torch.randn(((k + 1) * W, K), device=DEV) * 1.5).to(torch.bfloat16)
    head.step(st, hs, nb, tok, msk)
    torch.cuda.synchronize()
    assert int(s.item()) == 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="all", choices=["core", "bp", "lmhead", "all"])
    a = ap.parse_args()
    if a.part in ("core", "all"):
        part_core()
    if a.part in ("bp", "all"):
        part_bp()
    if a.part in ("lmhead", "all"):
        part_lmhead()
    torch.cuda.synchronize()
    print("sanitize_drive: done", a.part)


if __name__ == "__main__":
    main()
