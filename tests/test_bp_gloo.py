"""Branch-parallel protocol on CPU with torch.distributed gloo, world_size 2 and 4.

Each rank owns the branches `lopa.bp_shard` assigns it, reduces and scores only those (oracle
arithmetic), publishes one record {local scores, local best (score, id), best row} through
all_gather_object (the NCCL all-gather's role), and every rank then runs the same select,
anchor and spawn.  The result must equal the single-process oracle step exactly, on every rank:
this pins the partition and the claim that an all-gather of per-rank bests (ties -> lowest id)
is the global Eq. 2 argmax (R9) that liblopa's lopa_bp_step relies on."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import syngen
from oracle import lopa_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(seed, V, W, k, tau):
    tok0, msk0 = syngen.fresh_block(W)
    L0 = syngen.gen_logits(seed, 0, V, tok0[None], msk0[None], extras=1)
    r0 = O.step(L0, tok0[None].astype(np.int64), msk0[None], k, tau)
    tok, msk = r0.spawn.tokens, r0.spawn.mask
    L = syngen.gen_logits(seed, 0, V, tok, msk, extras=1)
    return L, tok, msk


def _worker(rank, world, port, seeds, V, W, k, tau, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_16229_b200.lopa import bp_shard
    ok = True
    try:
        for seed in seeds:
            L, tok, msk = _case(seed, V, W, k, tau)
            n = len(msk)
            b_loc, lo, hi = bp_shard(k + 1, world, rank)
            hi = min(hi, n)
            lo = min(lo, hi)
            scores, rows = [], []
            for j in range(lo, hi):
                c, a, _ = O.confidence(L[j], msk[j])
                scores.append(O.branch_score(c, msk[j]))
                rows.append((tok[j], msk[j], c, a))
            if scores:
                best = max(scores)
                jl = min(i for i, s in enumerate(scores) if s == best)
                rec = (scores, best, lo + jl, rows[jl])
            else:
                rec = ([], -np.inf, 2**31 - 1, None)
            recs = [None] * world
            dist.all_gather_object(recs, rec)
            gbest = max(r[1] for r in recs)
            wid = min(r[2] for r in recs if r[1] == gbest)
            owner = [r for r in recs if r[2] == wid][0]
            all_scores = [s for r in recs for s in r[0]]
            t_w, m_w, c_w, a_w = owner[3]
            anc = O.anchor_fill(c_w, a_w, t_w, m_w, tau)
            sp = O.spawn_branches(c_w, a_w, anc.tokens, anc.mask, k)
            ref = O.step(L, tok, msk, k, tau)
            ok &= wid == ref.winner
            ok &= np.allclose(all_scores, ref.scores, rtol=0, atol=0)
            ok &= sp.lookahead == ref.spawn.lookahead
            ok &= np.array_equal(sp.tokens, ref.spawn.tokens) and np.array_equal(sp.mask, ref.spawn.mask)
    except Exception as e:  # pragma: no cover
        ok = False
        q.put(repr(e))
    q.put(bool(ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bp_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, list(range(6)), 64, 8, 5, 0.9, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r is True for r in res), res


def _commit_worker(rank, world, port, k, nbytes, q):
    """NEXT-3 Commit-Winner-Cache protocol (lopa_bp_commit_winner): the owner of the winner
    (rank w // b_loc, bp_shard's partition) contributes its payload, every other rank zeros, and
    a sum all-reduce over integers leaves the winner's payload bit-exactly on every rank."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_16229_b200.lopa import bp_shard
    ok = True
    try:
        b_loc, lo, hi = bp_shard(k + 1, world, rank)
        pay = lambda j: torch.from_numpy(np.random.default_rng(1000 + j).integers(0, 2**31, nbytes // 4)).to(torch.int64)
        local = [pay(j) for j in range(lo, lo + b_loc)]
        for w in range(k + 1):
            owner = w // b_loc
            contrib = local[w - lo].clone() if owner == rank else torch.zeros(nbytes // 4, dtype=torch.int64)
            dist.all_reduce(contrib, op=dist.ReduceOp.SUM)
            ok &= bool(torch.equal(contrib, pay(w)))
            ok &= lo <= w < lo + b_loc if owner == rank else not (lo <= w < hi)
    finally:
        dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.parametrize("world,k", [(2, 7), (4, 7), (4, 14), (2, 2)])
def test_commit_winner_protocol(world, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_commit_worker, args=(r, world, port, k, 256, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(res[r] for r in range(world))
