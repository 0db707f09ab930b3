"""GPU (liblopa, sm_100a) vs CPU oracle parity on seeded SYN-D2F inputs.

All calls go through the C ABI (paper_2512_16229_b200.lopa -> liblopa.so)."""
import numpy as np
import pytest
import torch

import syngen
from oracle import lopa_oracle as O
import _gpu as G

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def L():
    from paper_2512_16229_b200 import lopa
    lopa.lib()
    return lopa


# ----------------------------------------------------------------------------- generator
@pytest.mark.parametrize("V,W,extras,ld", [(64, 8, 1, None), (61, 5, 1, 64), (1000, 4, 0, None),
                                           (151936, 2, 0, None)])
def test_syn_generate_matches_numpy(L, V, W, extras, ld):
    rng = np.random.default_rng(V + W)
    tok = rng.integers(0, V, size=(3, W)).astype(np.int32)
    msk = (rng.random((3, W)) < 0.6).astype(np.uint8)
    g = L.syn_generate(11, 2, V, torch.from_numpy(tok).to(DEV), torch.from_numpy(msk).to(DEV),
                       extras=extras, ld=ld)
    ref = syngen.gen_logits(11, 2, V, tok, msk, extras=extras, ld=ld if ld else ((V + 7) // 8) * 8)
    assert np.array_equal(G.to_np_u16(g), ref)


# ----------------------------------------------------------------------------- a1
def _bits(x):
    return (np.asarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def special_rows(V):
    rows = []
    r = np.zeros(V, np.float32); rows.append(r)                                  # flat: 1/V, argmax 0
    r = np.full(V, -3.0, np.float32); r[V - 1] = 5.0; rows.append(r)             # spike at the end
    r = np.full(V, -3.0, np.float32); r[0] = 5.0; rows.append(r)                 # spike at 0
    r = np.full(V, -np.inf, np.float32); r[V // 2] = 1.0; rows.append(r)         # spike over -inf: 1
    r = np.full(V, 1.0, np.float32); r[3] = 2.0; r[V - 2] = 2.0; rows.append(r)  # tie: lowest id
    r = np.linspace(-4, 4, V).astype(np.float32); rows.append(r)                 # ramp
    return np.stack([_bits(x) for x in rows])


@pytest.mark.parametrize("V", [1, 7, 61, 64, 1000, 8192, 8193, 16391, 151936])
def test_confidence_rows(L, V):
    rng = np.random.default_rng(V)
    ld = ((V + 7) // 8) * 8
    rnd = _bits(rng.normal(0, 2, size=(20, V)).astype(np.float32))
    rows = np.concatenate([special_rows(V), rnd]) if V >= 8 else rnd
    buf = np.zeros((rows.shape[0], ld), np.uint16)
    buf[:, :V] = rows
    buf[:, V:] = 0x7FC0  # NaN padding must never be read
    t = torch.from_numpy(buf.view(np.int16)).to(DEV).view(torch.bfloat16)
    conf, amax, st = L.confidence(t, vocab=V)
    rc, ra, rst = O.confidence(rows)
    assert int(st.item()) == rst == 0
    c = conf.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(c - rc)) <= G.CONF_TOL
    assert np.max(np.abs(c - rc)) <= 2e-6          # the fp32 budget, tighter than the contract
    assert np.array_equal(amax.cpu().numpy(), ra)


@pytest.mark.parametrize("n_rows,V", [(3, 1000), (300, 151936), (40, 8193)])
def test_reduce_only_leaves_workspace_zeroed(L, n_rows, V):
    """K1 alone (lopa_debug_reduce_only, bench.py's roofline launches) resets its own work
    counter: after several back-to-back K1-only launches the workspace counters are zero and a
    lopa_confidence call on the same workspace is still exact."""
    rng = np.random.default_rng(n_rows)
    ld = ((V + 7) // 8) * 8
    rows = _bits(rng.normal(0, 2, size=(n_rows, V)).astype(np.float32))
    buf = np.zeros((n_rows, ld), np.uint16)
    buf[:, :V] = rows
    t = torch.from_numpy(buf.view(np.int16)).to(DEV).view(torch.bfloat16)
    rm = torch.from_numpy((rng.random(n_rows) < 0.8).astype(np.uint8)).to(DEV)
    ws = L.new_workspace(n_rows, V, DEV)
    st = L.new_status(DEV)
    import ctypes
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(5):
        assert L.lib().lopa_debug_reduce_only(L._p(t), ld, n_rows, V, L._p(rm), L._p(st), L._p(ws),
                                              ws.numel(), sp) == 0
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert ws[:8].view(torch.int32).cpu().tolist() == [0, 0]
    conf, amax, st2 = L.confidence(t, vocab=V, row_mask=rm, workspace=ws)
    rc, ra, _ = O.confidence(rows)
    sel = rm.cpu().numpy().astype(bool)
    assert int(st2.item()) == 0
    assert np.max(np.abs(conf.cpu().numpy().astype(np.float64)[sel] - rc[sel])) <= G.CONF_TOL
    assert np.array_equal(amax.cpu().numpy()[sel], ra[sel])
    assert ws[:8].view(torch.int32).cpu().tolist() == [0, 0]


@pytest.mark.parametrize("n_rows,V,n_valid", [(256, 8193, n) for n in (0, 1, 100, 223, 224, 225, 256)]
                         + [(30, 16391, 10), (30, 16391, 30), (100, 151936, 60), (100, 151936, 99),
                            (147, 151936, 120), (149, 16391, 120), (5, 151936, 2)])
def test_confidence_item_spaces(L, n_rows, V, n_valid):
    """K1 numbers its work items over the raw rows when >= 7/8 of them are valid, else over the
    valid rows only, after the speculative copies of the raw items [0, G): both
    sides of the switch, fewer rows than CTAs, and the degenerate row sets give the oracle's
    conf / argmax on exactly the masked rows."""
    rng = np.random.default_rng(n_valid)
    ld = ((V + 7) // 8) * 8
    rows = _bits(rng.normal(0, 2, size=(n_rows, V)).astype(np.float32))
    buf = np.zeros((n_rows, ld), np.uint16)
    buf[:, :V] = rows
    t = torch.from_numpy(buf.view(np.int16)).to(DEV).view(torch.bfloat16)
    m = np.zeros(n_rows, np.uint8)
    m[rng.permutation(n_rows)[:n_valid]] = 1
    conf, amax, st = L.confidence(t, vocab=V, row_mask=torch.from_numpy(m).to(DEV))
    rc, ra, _ = O.confidence(rows)
    sel = m.astype(bool)
    assert int(st.item()) == 0
    c, a = conf.cpu().numpy().astype(np.float64), amax.cpu().numpy()
    assert np.max(np.abs(c[sel] - rc[sel]), initial=0.0) <= G.CONF_TOL
    assert np.array_equal(a[sel], ra[sel])
    assert np.all(np.isnan(c[~sel])) and np.all(a[~sel] == -1)


@pytest.mark.parametrize("V", [(1 << 20) + 3, 1 << 23])
def test_confidence_huge_vocab(L, V):
    """Up to LOPA_MAX_VOCAB = 2^23: 512 groups per row, so the fold takes its sequential
    (> 16 groups) path; ragged tail at 2^20 + 3."""
    rng = np.random.default_rng(V)
    ld = ((V + 7) // 8) * 8
    rnd = _bits(rng.standard_normal((3, V), dtype=np.float32) * np.float32(2))
    rows = np.concatenate([special_rows(V), rnd])
    buf = np.zeros((rows.shape[0], ld), np.uint16)
    buf[:, :V] = rows
    buf[:, V:] = 0x7FC0
    t = torch.from_numpy(buf.view(np.int16)).to(DEV).view(torch.bfloat16)
    conf, amax, st = L.confidence(t, vocab=V)
    rc, ra, rst = O.confidence(rows)
    assert int(st.item()) == rst == 0
    c = conf.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(c - rc)) <= G.CONF_TOL
    assert np.array_equal(amax.cpu().numpy(), ra)


def test_confidence_row_mask_and_nonfinite(L):
    V = 3000
    rows = np.zeros((6, V), np.float32)
    rows[1, 5] = np.nan
    rows[2, 7] = np.inf
    rows[3, :] = -np.inf
    rows[4, 9] = 4.0
    u = np.stack([_bits(r) for r in rows])
    t = torch.from_numpy(u.view(np.int16)).to(DEV).view(torch.bfloat16)
    for sel in ([1, 1, 1, 1, 1, 1], [1, 0, 0, 0, 1, 1], [0, 1, 0, 0, 0, 0], [0, 0, 0, 1, 0, 0]):
        m = torch.tensor(sel, dtype=torch.uint8, device=DEV)
        conf, amax, st = L.confidence(t, row_mask=m)
        rc, ra, rst = O.confidence(u, np.array(sel))
        assert int(st.item()) == rst
        c, a = conf.cpu().numpy(), amax.cpu().numpy()
        for r in range(6):
            if not sel[r]:
                assert np.isnan(c[r]) and a[r] == -1          # untouched
            elif r in (0, 4, 5):
                assert abs(c[r] - rc[r]) <= 1e-6 and a[r] == ra[r]


def test_confidence_shift_metamorphic(L):
    """+1.0 on every logit is bf16-exact for SYN rows; (x - m) is formed exactly, so conf and
    argmax bits must be identical (SURVEY §8(c) pin iii)."""
    V, W = 151936, 4
    tok = torch.zeros((1, W), dtype=torch.int32, device=DEV)
    msk = torch.ones((1, W), dtype=torch.uint8, device=DEV)
    x = L.syn_generate(5, 0, V, tok, msk).view(W, -1)
    y = (x.float() + 1.0).to(torch.bfloat16)
    assert torch.equal(y.float() - 1.0, x.float())
    c1, a1, _ = L.confidence(x)
    c2, a2, _ = L.confidence(y)
    assert torch.equal(c1.view(torch.int32), c2.view(torch.int32)) and torch.equal(a1, a2)


def test_confidence_invariant_to_row_set(L):
    """Segment-canonical reduction: a row's conf bits do not depend on which or how many other
    rows are reduced in the same launch (hence on k, the launch split, or the BP world size)."""
    V, W = 151936, 32
    tok = torch.zeros((4, W), dtype=torch.int32, device=DEV)
    msk = torch.ones((4, W), dtype=torch.uint8, device=DEV)
    x = L.syn_generate(9, 0, V, tok, msk).view(4 * W, -1)
    c_all, a_all, _ = L.confidence(x)
    for sub in (slice(0, 1), slice(5, 37), slice(100, 128)):
        c, a, _ = L.confidence(x[sub].contiguous())
        assert torch.equal(c.view(torch.int32), c_all[sub].view(torch.int32))
        assert torch.equal(a, a_all[sub])


# ----------------------------------------------------------------------------- a2-a4 (SPEC)
GOLD = None


def _gold():
    import json, os
    global GOLD
    if GOLD is None:
        GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_decode_examples.json")))
    return GOLD


def _dense(case):
    W = case["window"]
    conf = np.zeros(W, np.float32)
    mask = np.zeros(W, np.uint8)
    for k, v in case["conf"].items():
        conf[int(k)] = np.float32(v)
        mask[int(k)] = 1
    return conf, mask


def test_spec_anchor_examples_on_gpu(L):
    for case in _gold()["select_fill_set"] + _gold()["anchor_step"]:
        conf, mask = _dense(case)
        W = case["window"]
        amax = np.arange(100, 100 + W, dtype=np.int32)
        tok = np.full(W, 7, np.int32)
        t, m, st = L.anchor_fill(*(torch.from_numpy(a).to(DEV) for a in (conf, amax, tok, mask)), case["tau"])
        filled = [i for i in range(W) if mask[i] and not m[i].item()]
        expect = case.get("i_fill", case.get("filled"))
        assert filled == expect, case["cite"]
        assert int(st.item()) == 0


def test_spec_spawn_examples_on_gpu(L):
    for case in _gold()["spawn_lookahead"]:
        conf, mask = _dense(case)
        W = case["window"]
        amax = np.arange(100, 100 + W, dtype=np.int32)
        tok = np.full(W, 7, np.int32)
        bt, bm, look, nb = L.spawn_branches(*(torch.from_numpy(a).to(DEV) for a in (conf, amax, tok, mask)), case["k"])
        n = len(case["lookahead"])
        assert look.cpu().tolist()[:n] == case["lookahead"], case["cite"]
        assert all(x == -1 for x in look.cpu().tolist()[n:])
        assert int(nb.item()) == n + 1


def test_spec_verify_examples_on_gpu(L):
    for case in _gold()["branch_confidence"]:
        conf, mask = _dense(case)
        s, w = L.verify_select(torch.from_numpy(conf[None]).to(DEV), torch.from_numpy(mask[None]).to(DEV),
                               torch.ones(1, dtype=torch.int32, device=DEV))
        assert abs(s.item() - case["score"]) <= 1e-7, case["cite"]
    for case in _gold()["verify_branches"]:
        sc = case["scores"]
        n = len(sc)
        # a branch with one masked position of conf c has score c exactly
        conf = np.zeros((n, 1), np.float32)
        conf[:, 0] = sc
        mask = np.ones((n, 1), np.uint8)
        s, w = L.verify_select(torch.from_numpy(conf).to(DEV), torch.from_numpy(mask).to(DEV),
                               torch.tensor([n], dtype=torch.int32, device=DEV))
        assert int(w.item()) == case["winner"], case["cite"]


def test_anchor_empty_mask_flag(L):
    W = 8
    z = torch.zeros(W, device=DEV)
    t, m, st = L.anchor_fill(z, torch.zeros(W, dtype=torch.int32, device=DEV),
                             torch.arange(W, dtype=torch.int32, device=DEV),
                             torch.zeros(W, dtype=torch.uint8, device=DEV), 0.9)
    assert int(st.item()) == O.DEV_EMPTY_MASK
    assert t.cpu().tolist() == list(range(W))


@pytest.mark.parametrize("W", [1, 5, 8, 31, 32, 33, 64])
def test_decisions_random_maps(L, W):
    """Eq. 1 / top-k / Eq. 2 kernels vs the oracle on random fp32 conf maps with forced ties."""
    rng = np.random.default_rng(W)
    for it in range(60):
        conf = rng.choice(np.float32([0.1, 0.5, 0.9, 0.95, 0.3]), size=W) if it % 3 == 0 \
            else rng.random(W).astype(np.float32)
        mask = (rng.random(W) < 0.7).astype(np.uint8)
        if not mask.any():
            mask[rng.integers(W)] = 1
        amax = rng.integers(0, 151936, size=W).astype(np.int32)
        tok = rng.integers(0, 151936, size=W).astype(np.int32)
        tau = float(rng.choice([0.3, 0.9, 0.95, 1.0]))
        k = int(rng.integers(0, min(W, 31) + 1))
        d = [torch.from_numpy(a).to(DEV) for a in (conf, amax, tok, mask)]
        t, m, st = L.anchor_fill(*d, tau)
        ref = O.anchor_fill(conf.astype(np.float64), amax, tok, mask, tau)
        assert np.array_equal(t.cpu().numpy(), ref.tokens) and np.array_equal(m.cpu().numpy(), ref.mask)
        bt, bm, look, nb = L.spawn_branches(d[0], d[1], t, m, k)
        sp = O.spawn_branches(conf.astype(np.float64), amax, ref.tokens, ref.mask, k)
        n = len(sp.lookahead)
        assert int(nb.item()) == n + 1
        assert look.cpu().tolist()[:n] == sp.lookahead
        assert np.array_equal(bt.cpu().numpy()[: n + 1], sp.tokens)
        assert np.array_equal(bm.cpu().numpy()[: n + 1], sp.mask)
        # verify over random branch confs
        nbr = int(rng.integers(1, 33))
        bc = rng.random((nbr, W)).astype(np.float32)
        if it % 4 == 0:
            bc[:] = bc[0]
        bmask = (rng.random((nbr, W)) < 0.5).astype(np.uint8)
        s, w = L.verify_select(torch.from_numpy(bc).to(DEV), torch.from_numpy(bmask).to(DEV),
                               torch.tensor([nbr], dtype=torch.int32, device=DEV))
        rs = [O.branch_score(bc[j].astype(np.float64), bmask[j]) for j in range(nbr)]
        assert np.max(np.abs(s.cpu().numpy().astype(np.float64) - rs)) <= 1e-7
        assert int(w.item()) == O.verify_select([float(np.float32(x)) for x in rs])


# ----------------------------------------------------------------------------- fused step
def _run_steps(L, seed, V, W, k, tau, iters, extras, blk=0, counter=None, metric=0, param=0.0):
    st = L.Stepper(V, W, k + 1, k, tau, DEV, metric=metric, metric_param=param)
    tok, msk, nb = G.fresh_tables(k, W, DEV)
    fills = 0
    for it in range(iters):
        n = int(nb.item())
        logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
        L.syn_generate(seed, blk, V, tok, msk, n_branches=n, extras=extras, out=logits[:n])
        out = st.step(logits, nb, tok, msk)
        torch.cuda.synchronize()
        G.check_step(out, G.to_np_u16(logits), tok.cpu().numpy(), msk.cpu().numpy(), n, k, tau, counter,
                     vocab=V, metric=metric, param=param)
        if int(out.n_next.item()) == 0:
            return it + 1
        tok, msk, nb = out.next_tokens.clone(), out.next_mask.clone(), out.n_next.clone()
        fills += 1
    return iters


@pytest.mark.parametrize("V,W,k", [(300000, 8, 2), (1 << 21, 4, 1)])
def test_step_many_groups(L, V, W, k):
    """Vocabularies with more than 16 groups per row (19 and 128 groups): the decision kernel
    folds them without staging, through the sequential fold."""
    _run_steps(L, 5, V, W, k, 0.9, 3, extras=0)


@pytest.mark.parametrize("seed", range(0, 120))
def test_step_toy(L, seed):
    """Toy config (BASELINE configs[0]): V=64, W=8, k=2, tau=0.9, with tie / flat rows, iterated
    to the end of the block (every iteration compared)."""
    _run_steps(L, seed, 64, 8, 2, 0.9, 20, extras=1)


@pytest.mark.parametrize("V,W,k,tau", [(64, 64, 31, 0.9), (61, 33, 5, 0.5), (1000, 16, 3, 0.95),
                                       (8193, 12, 11, 1.0), (64, 1, 0, 0.9), (64, 8, 0, 0.9)])
def test_step_shapes(L, V, W, k, tau):
    for seed in range(3):
        _run_steps(L, seed, V, W, k, tau, 80, extras=1)


@pytest.mark.parametrize("seed", [1, 2])
def test_step_dream(L, seed):
    """D2F-Dream shape (configs[1]): V=151936, W=32, k=7, tau=0.9, three iterations."""
    cnt = {}
    _run_steps(L, seed, 151936, 32, 7, 0.9, 3, extras=0, counter=cnt)


def test_step_diffucoder_one_iter(L):
    """D2F-DiffuCoder shape (configs[3]): V=151936, W=32, k=10, tau=0.95."""
    _run_steps(L, 3, 151936, 32, 10, 0.95, 2, extras=0)


def test_step_all_unmasked_block_is_done(L):
    V, W, k = 64, 8, 2
    st = L.Stepper(V, W, k + 1, k, 0.9, DEV)
    tok = torch.arange((k + 1) * W, dtype=torch.int32, device=DEV).view(k + 1, W)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=DEV)
    nb = torch.tensor([2], dtype=torch.int32, device=DEV)
    logits = torch.zeros((k + 1, W, 64), dtype=torch.bfloat16, device=DEV)
    out = st.step(logits, nb, tok, msk)
    assert int(out.n_next.item()) == 0 and int(out.winner.item()) == 0
    assert out.scores[:2].cpu().tolist() == [1.0, 1.0]
    assert torch.equal(out.next_tokens[0], tok[0])


# ----------------------------------------------------------------------------- loop
def _gpu_decode_block(L, seed, V, W, k, tau, extras, blk=0):
    """The package's Alg. 1 loop (lopa.decode_block) on the SYN-D2F forward."""
    fwd = lambda t, m, out: L.syn_generate(seed, blk, V, t, m, extras=extras, out=out)
    tok0 = torch.zeros(W, dtype=torch.int32, device=DEV)
    msk0 = torch.ones(W, dtype=torch.uint8, device=DEV)
    tokens, forwards = L.decode_block(fwd, tok0, msk0, k, tau, V)
    return tokens.cpu().numpy(), forwards


@pytest.mark.parametrize("seed", range(20))
def test_decode_loop_toy(L, seed):
    """Alg. 1 loop: final block tokens and forward count equal the oracle's."""
    V, W, k, tau = 64, 8, 2, 0.9
    fwd = lambda t, m: syngen.gen_logits(seed, 0, V, t, m, extras=1)
    tok0, msk0 = syngen.fresh_block(W)
    ref = O.decode_block(fwd, tok0, msk0, k, tau)
    g_tok, g_fw = _gpu_decode_block(L, seed, V, W, k, tau, 1)
    assert g_fw == ref.forwards and np.array_equal(g_tok, ref.tokens)


def test_decode_loop_dream_k7(L):
    V, W, k, tau, seed = 151936, 32, 7, 0.9, 1
    fwd = lambda t, m: syngen.gen_logits(seed, 0, V, t, m)
    tok0, msk0 = syngen.fresh_block(W)
    ref = O.decode_block(fwd, tok0, msk0, k, tau)
    g_tok, g_fw = _gpu_decode_block(L, seed, V, W, k, tau, 0)
    assert g_fw == ref.forwards and np.array_equal(g_tok, ref.tokens)


# ----------------------------------------------------------------------------- BP (emulated ranks)
@pytest.mark.parametrize("V,W,k", [(64, 8, 2), (151936, 32, 7), (151936, 32, 15), (1000, 16, 10)])
def test_bp_world_invariance(L, V, W, k):
    """Branch-parallel step with G in {1, 2, 4, 8} emulated ranks (local kernels + record
    exchange + global select) gives bit-identical outputs to the fused single-GPU step."""
    tau = 0.9
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    tok, msk, nb = G.fresh_tables(k, W, DEV)
    logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
    L.syn_generate(4, 0, V, tok, msk, n_branches=1, out=logits[:1])
    out = st.step(logits, nb, tok, msk)
    tok, msk, nb = out.next_tokens.clone(), out.next_mask.clone(), out.n_next.clone()
    n = int(nb.item())
    L.syn_generate(4, 0, V, tok, msk, n_branches=n, out=logits[:n])
    out = st.step(logits, nb, tok, msk)
    torch.cuda.synchronize()
    ref = {f: getattr(out, f).clone() for f in ("scores", "winner", "next_tokens", "next_mask", "lookahead", "n_next")}
    ref_conf = out.conf.clone()
    for world in (1, 2, 4, 8):
        st2 = L.Stepper(V, W, k + 1, k, tau, DEV)
        o2, confs, scores = L.bp_emulate_step(st2, world, logits, nb, tok, msk)
        torch.cuda.synchronize()
        b_loc = L.bp_shard(k + 1, world, 0)[0]
        for r, (c, a) in enumerate(confs):
            lo = r * b_loc
            hi = min(lo + b_loc, n)
            if hi > lo:
                m = msk[lo:hi].bool()
                assert torch.equal(c[: hi - lo][m].view(torch.int32), ref_conf[lo:hi][m].view(torch.int32))
        assert torch.equal(scores[:n].view(torch.int32), ref["scores"][:n].view(torch.int32))
        assert int(o2.winner.item()) == int(ref["winner"].item())
        nn = int(o2.n_next.item())
        assert nn == int(ref["n_next"].item())
        assert torch.equal(o2.next_tokens[:nn], ref["next_tokens"][:nn])
        assert torch.equal(o2.next_mask[:nn], ref["next_mask"][:nn])


def test_bp_nccl_single_rank(L):
    """The real NCCL path with one rank (communicator of size 1): same result as lopa_step."""
    V, W, k, tau = 151936, 32, 7, 0.9
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    tok, msk, nb = G.fresh_tables(k, W, DEV)
    logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
    L.syn_generate(8, 0, V, tok, msk, n_branches=1, out=logits[:1])
    out = st.step(logits, nb, tok, msk)
    tok, msk, nb = out.next_tokens.clone(), out.next_mask.clone(), out.n_next.clone()
    L.syn_generate(8, 0, V, tok, msk, n_branches=int(nb.item()), out=logits[: int(nb.item())])
    out = st.step(logits, nb, tok, msk)
    torch.cuda.synchronize()
    ref = (out.winner.item(), out.n_next.item(), out.next_tokens.clone(), out.next_mask.clone())
    st2 = L.Stepper(V, W, k + 1, k, tau, DEV)
    bp = L.BranchParallel(st2, 0, 1)
    try:
        o2 = bp.step(logits, nb, tok, msk)
        torch.cuda.synchronize()
        bp.check()
        assert (o2.winner.item(), o2.n_next.item()) == ref[:2]
        assert torch.equal(o2.next_tokens[: ref[1]], ref[2][: ref[1]])
        assert torch.equal(o2.next_mask[: ref[1]], ref[3][: ref[1]])
    finally:
        bp.close()


def test_bp_p2p_single_rank(L):
    """The peer-memory exchange (lopa_bp_step_p2p: records written into every rank's mapped
    buffer, epoch flags released at system scope, double-buffered by parity) with one rank:
    five consecutive steps identical to lopa_step, no peer timeout."""
    V, W, k, tau = 151936, 32, 7, 0.9
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    st2 = L.Stepper(V, W, k + 1, k, tau, DEV)
    bp = L.BranchParallel(st2, 0, 1, p2p=True)
    try:
        tok, msk, nb = G.fresh_tables(k, W, DEV)
        logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
        for it in range(5):
            n = int(nb.item())
            L.syn_generate(9, 0, V, tok, msk, n_branches=n, out=logits[:n])
            ref = st.step(logits, nb, tok, msk)
            o2 = bp.step(logits, nb, tok, msk)
            torch.cuda.synchronize()
            assert int(o2.status.item()) == 0
            assert (o2.winner.item(), o2.n_next.item()) == (ref.winner.item(), ref.n_next.item())
            m = int(ref.n_next.item())
            assert torch.equal(o2.next_tokens[:m], ref.next_tokens[:m])
            assert torch.equal(o2.next_mask[:m], ref.next_mask[:m])
            if m == 0:
                break
            tok, msk, nb = ref.next_tokens.clone(), ref.next_mask.clone(), ref.n_next.clone()
        bp.check()
    finally:
        bp.close()


def test_bp_commit_winner_p2p_single_rank(L):
    """NEXT-3 over peer memory with one rank: each step's payloads are written into the slots of
    the step's parity before the step; afterwards the winner's payload is pulled bit-exactly."""
    V, W, k, tau, nbytes = 1000, 16, 3, 0.9, 4096
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    bp = L.BranchParallel(st, 0, 1, p2p=True, payload_bytes=nbytes)
    try:
        tok, msk, nb = G.fresh_tables(k, W, DEV)
        logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
        out = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
        for e in range(1, 5):
            pay = torch.randint(0, 256, (bp.b_loc, nbytes), dtype=torch.uint8, device=DEV)
            bp.payload_view(e & 1).copy_(pay)   # the owner writes step e's payloads (parity e & 1)
            n = int(nb.item())
            L.syn_generate(3, 0, V, tok, msk, n_branches=n, out=logits[:n])
            o = bp.step(logits, nb, tok, msk)
            bp.commit_winner_p2p(out)
            torch.cuda.synchronize()
            assert int(o.status.item()) == 0
            w = int(o.winner.item())
            assert torch.equal(out, pay[w])
            if int(o.n_next.item()) == 0:
                break
            tok, msk, nb = o.next_tokens.clone(), o.next_mask.clone(), o.n_next.clone()
        bp.check()
    finally:
        bp.close()


@pytest.mark.parametrize("nbytes", [16, 4096, 1835008])
def test_bp_commit_winner_single_rank(L, nbytes):
    """NEXT-3 Commit-Winner-Cache over the real NCCL path (one rank): the winner's payload
    (KV-sized for the largest case: 28 layers x 2 x 4 KV heads x 128 x 32 positions x 2 B)
    arrives bit-exactly, for every possible winner; invalid sizes are rejected."""
    V, W, k, tau = 64, 8, 3, 0.9
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    bp = L.BranchParallel(st, 0, 1)
    try:
        g = torch.Generator(device=DEV).manual_seed(nbytes)
        pay = torch.randint(0, 256, (bp.b_loc, nbytes), dtype=torch.uint8, device=DEV, generator=g)
        for w in range(bp.b_loc):
            win = torch.tensor([w], dtype=torch.int32, device=DEV)
            out = bp.commit_winner(pay, winner=win)
            torch.cuda.synchronize()
            assert torch.equal(out, pay[w])
        bp.check()
        with pytest.raises(L.LopaError):
            bp.commit_winner(torch.zeros((bp.b_loc, 12), dtype=torch.uint8, device=DEV))
    finally:
        bp.close()


# ----------------------------------------------------------------------------- errors
def test_invalid_args_raise(L):
    t = torch.zeros((2, 60), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(L.LopaError):
        L.confidence(t[:, 1:])            # misaligned base
    with pytest.raises(L.LopaError):
        L.Stepper(64, 257, 2, 1, 0.9, DEV).step(torch.zeros((2, 257, 64), dtype=torch.bfloat16, device=DEV),
                                                 torch.ones(1, dtype=torch.int32, device=DEV),
                                                 torch.zeros((2, 257), dtype=torch.int32, device=DEV),
                                                 torch.ones((2, 257), dtype=torch.uint8, device=DEV))
    with pytest.raises(L.LopaError):      # W > 64 needs V <= 2^22 (R24)
        L.Stepper((1 << 22) + 8, 65, 1, 1, 0.9, DEV).step(
            torch.zeros((1, 65, (1 << 22) + 8), dtype=torch.bfloat16, device=DEV),
            torch.ones(1, dtype=torch.int32, device=DEV), torch.zeros((1, 65), dtype=torch.int32, device=DEV),
            torch.ones((1, 65), dtype=torch.uint8, device=DEV))
    with pytest.raises(L.LopaError):
        L.confidence(torch.zeros((2, 64)))  # CPU tensor: no fallback


# ----------------------------------------------------------------------------- multi-block loops
def _gpu_decode_blocks(L, seed, V, W, k, tau, n_blocks, extras=0):
    toks, fw = [], 0
    for blk in range(n_blocks):
        t, f = _gpu_decode_block(L, seed, V, W, k, tau, extras, blk=blk)
        toks.append(t)
        fw += f
    return np.concatenate(toks), fw


@pytest.mark.parametrize("seed", [0, 1])
def test_multiblock_decode_toy(L, seed):
    """Sequential blocks (R18/R22: each block starts from its own initial forward)."""
    V, W, k, tau = 64, 8, 2, 0.9
    ref_tok, ref_fw = [], 0
    for blk in range(4):
        fwd = lambda t, m, blk=blk: syngen.gen_logits(seed, blk, V, t, m, extras=1)
        tok0, msk0 = syngen.fresh_block(W)
        tr = O.decode_block(fwd, tok0, msk0, k, tau)
        ref_tok.append(tr.tokens)
        ref_fw += tr.forwards
    g_tok, g_fw = _gpu_decode_blocks(L, seed, V, W, k, tau, 4, extras=1)
    assert g_fw == ref_fw and np.array_equal(g_tok, np.concatenate(ref_tok))


def test_multiblock_decode_diffucoder(L):
    """D2F-DiffuCoder shape (configs[3]): V=151936, W=32, k=10, tau=0.95, 2 sequential blocks
    (64 tokens), final tokens and forward counts equal to the oracle's."""
    V, W, k, tau, seed = 151936, 32, 10, 0.95, 3
    ref_tok, ref_fw = [], 0
    for blk in range(2):
        fwd = lambda t, m, blk=blk: syngen.gen_logits(seed, blk, V, t, m)
        tok0, msk0 = syngen.fresh_block(W)
        tr = O.decode_block(fwd, tok0, msk0, k, tau)
        ref_tok.append(tr.tokens)
        ref_fw += tr.forwards
    g_tok, g_fw = _gpu_decode_blocks(L, seed, V, W, k, tau, 2)
    assert g_fw == ref_fw and np.array_equal(g_tok, np.concatenate(ref_tok))


@pytest.mark.parametrize("k,W", [(1, 16), (3, 16), (15, 32), (31, 64), (31, 16)])
def test_sweep_shapes_one_step(L, k, W):
    """BASELINE configs[4] sweep shapes (k in {1,3,15,31} x W in {16,32,64}) at V=151936: one
    verify step after the initial anchor, compared with the oracle."""
    _run_steps(L, 7, 151936, W, k, 0.9, 2, extras=0)


def test_dense_rows_roofline_mode(L):
    """Dense mode of the bench roofline (every (branch, position) row masked): a1 over 256 rows
    equals the oracle on sampled rows."""
    V, W, k = 151936, 32, 7
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=DEV)
    msk = torch.ones((k + 1, W), dtype=torch.uint8, device=DEV)
    x = L.syn_generate(21, 0, V, tok, msk).view((k + 1) * W, -1)
    c, a, st = L.confidence(x)
    assert int(st.item()) == 0
    xs = G.to_np_u16(x)
    for r in (0, 77, 128, 255):
        rc, ra, _ = O.row_confidence(xs[r])
        assert abs(c[r].item() - rc) <= 2e-6 and a[r].item() == ra


# ----------------------------------------------------------------------------- Eq. 2 variants
def test_spec_sliding_window_on_gpu(L):
    """[.9,.2,.8] in position order, sliding_window(2) -> 0.5."""
    conf = torch.tensor([[0.9, 0.2, 0.8]], dtype=torch.float32, device=DEV)
    mask = torch.ones((1, 3), dtype=torch.uint8, device=DEV)
    s, w = L.verify_select(conf, mask, torch.ones(1, dtype=torch.int32, device=DEV),
                           metric=L.METRIC_SLIDING_MIN, param=2.0)
    assert s.item() == float(np.float32(O.branch_score(conf.cpu().numpy()[0].astype(np.float64), [1, 1, 1],
                                                       O.METRIC_SLIDING_MIN, 2)))
    assert abs(s.item() - 0.5) < 1e-7


@pytest.mark.parametrize("metric,param", [(1, 1.0), (1, 3.0), (1, 64.0), (2, 0.25), (2, 0.5), (2, 1.0),
                                          (2, 0.1)])
def test_metric_variants_random_maps(L, metric, param):
    """The P:204 variants on random confidence maps with forced ties: scores bit-equal to the
    oracle's fp64 value rounded to fp32 (exact sums on both sides); winner by the oracle's rule."""
    rng = np.random.default_rng(int(metric * 100 + param * 10))
    for it in range(40):
        W = int(rng.integers(1, 65))
        nbr = int(rng.integers(1, 33))
        bc = rng.random((nbr, W)).astype(np.float32)
        if it % 3 == 0:
            bc = rng.choice(np.float32([0.25, 0.5, 0.75]), size=(nbr, W))
        bm = (rng.random((nbr, W)) < 0.6).astype(np.uint8)
        s, w = L.verify_select(torch.from_numpy(bc).to(DEV), torch.from_numpy(bm).to(DEV),
                               torch.tensor([nbr], dtype=torch.int32, device=DEV), metric=metric, param=param)
        rs = [O.branch_score(bc[j].astype(np.float64), bm[j], metric, param) for j in range(nbr)]
        rs32 = [float(np.float32(x)) for x in rs]
        assert s.cpu().tolist() == rs32
        assert int(w.item()) == O.verify_select(rs32)


@pytest.mark.parametrize("metric,param", [(1, 4.0), (2, 0.3)])
def test_step_with_metric_variants(L, metric, param):
    """Full fused steps with a P:204 branch-confidence variant: toy (iterated) and Dream shape."""
    for seed in range(20):
        _run_steps(L, seed, 64, 8, 2, 0.9, 20, extras=1, metric=metric, param=param)
    _run_steps(L, 1, 151936, 32, 7, 0.9, 2, extras=0, metric=metric, param=param)


# ----------------------------------------------------------------------------- wide windows (D2F)
@pytest.mark.parametrize("W", [65, 96, 128, 200, 256])
def test_decisions_wide_windows(L, W):
    """W > 64 (the D2F multi-block window, 8 positions per lane): Eq. 1 with per-position tau,
    top-k spawn and Eq. 2 (all metrics) vs the oracle on random maps with forced ties."""
    rng = np.random.default_rng(W)
    for it in range(20):
        conf = rng.choice(np.float32([0.1, 0.5, 0.9, 0.95]), size=W) if it % 3 == 0 \
            else rng.random(W).astype(np.float32)
        mask = (rng.random(W) < 0.7).astype(np.uint8)
        if not mask.any():
            mask[0] = 1
        amax = rng.integers(0, 151936, size=W).astype(np.int32)
        tok = rng.integers(0, 151936, size=W).astype(np.int32)
        taus = rng.choice(np.float32([0.9, 0.95, 0.5]), size=W).astype(np.float32)
        k = int(rng.integers(0, 32))
        d = [torch.from_numpy(a).to(DEV) for a in (conf, amax, tok, mask)]
        t, m, st = L.anchor_fill(*d, 0.9, tau_pos=torch.from_numpy(taus).to(DEV))
        ref = O.anchor_fill(conf.astype(np.float64), amax, tok, mask, taus)
        assert np.array_equal(t.cpu().numpy(), ref.tokens) and np.array_equal(m.cpu().numpy(), ref.mask)
        bt, bm, look, nb = L.spawn_branches(d[0], d[1], t, m, k)
        sp = O.spawn_branches(conf.astype(np.float64), amax, ref.tokens, ref.mask, k)
        n = len(sp.lookahead)
        assert int(nb.item()) == n + 1 and look.cpu().tolist()[:n] == sp.lookahead
        assert np.array_equal(bt.cpu().numpy()[: n + 1], sp.tokens)
        assert np.array_equal(bm.cpu().numpy()[: n + 1], sp.mask)
        nbr = int(rng.integers(1, 17))
        bc = rng.random((nbr, W)).astype(np.float32)
        bmask = (rng.random((nbr, W)) < 0.5).astype(np.uint8)
        for metric, param in ((0, 0.0), (1, 5.0), (2, 0.3)):
            s, w = L.verify_select(torch.from_numpy(bc).to(DEV), torch.from_numpy(bmask).to(DEV),
                                   torch.tensor([nbr], dtype=torch.int32, device=DEV), metric=metric, param=param)
            rs = [float(np.float32(O.branch_score(bc[j].astype(np.float64), bmask[j], metric, param))) for j in range(nbr)]
            assert s.cpu().tolist() == rs and int(w.item()) == O.verify_select(rs)


@pytest.mark.parametrize("V,W,k", [(64, 96, 5), (1000, 128, 7), (151936, 128, 7), (64, 256, 15)])
def test_step_wide_windows(L, V, W, k):
    """Fused steps on W > 64 windows with per-position thresholds (tau_act on the newest block,
    tau_conf elsewhere), iterated, against the oracle."""
    taus = np.full(W, 0.9, np.float32)
    taus[-32:] = 0.95
    tp = torch.from_numpy(taus).to(DEV)
    st = L.Stepper(V, W, k + 1, k, 0.9, DEV, tau_pos=tp)
    tok, msk, nb = G.fresh_tables(k, W, DEV)
    for it in range(3 if V > 10000 else 12):
        n = int(nb.item())
        logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
        L.syn_generate(2, 0, V, tok, msk, n_branches=n, extras=1 if V < 10000 else 0, out=logits[:n])
        out = st.step(logits, nb, tok, msk)
        torch.cuda.synchronize()
        G.check_step(out, G.to_np_u16(logits), tok.cpu().numpy(), msk.cpu().numpy(), n, k, taus,
                     vocab=V)
        if int(out.n_next.item()) == 0:
            break
        tok, msk, nb = out.next_tokens.clone(), out.next_mask.clone(), out.n_next.clone()


# ----------------------------------------------------------------------------- CUDA graph loop
def test_step_loop_graph_matches_eager(L):
    """A 10-iteration Alg. 1 loop captured in one CUDA graph (lopa.StepLoopGraph) visits the
    same states as the same loop run eagerly step by step (fixed logits buffers per iteration;
    the tables feed back on the device)."""
    V, W, k, tau = 1000, 32, 5, 0.9
    g = torch.Generator(device=DEV).manual_seed(3)
    bufs = [(torch.randn((k + 1, W, 1000), generator=g, device=DEV) * 3).to(torch.bfloat16) for _ in range(3)]

    def fresh():
        tok, msk, nb = G.fresh_tables(k, W, DEV)
        return tok, msk, nb

    st_e = L.Stepper(V, W, k + 1, k, tau, DEV)
    tok, msk, nb = fresh()
    trace_e = []
    for i in range(10):
        o = st_e.step(bufs[i % 3], nb, tok, msk)
        trace_e.append((int(o.winner.item()), int(o.n_next.item())))
        tok[: k + 1].copy_(o.next_tokens)
        msk[: k + 1].copy_(o.next_mask)
        nb.copy_(o.n_next)
    final_e = (tok.clone(), msk.clone())
    st_g = L.Stepper(V, W, k + 1, k, tau, DEV)
    tok, msk, nb = fresh()
    t0, m0 = tok.clone(), msk.clone()
    gl = L.StepLoopGraph(st_g, bufs, nb, tok, msk, 10)
    # the constructor ran one warm-up iteration: restore the initial state, then replay
    tok.copy_(t0), msk.copy_(m0), nb.fill_(1)
    gl.replay()
    torch.cuda.synchronize()
    assert torch.equal(tok, final_e[0]) and torch.equal(msk, final_e[1])
    assert (int(st_g.out.winner.item()), int(st_g.out.n_next.item())) == trace_e[-1]
    # replaying again from the same start gives the same result (the graph is reusable)
    tok.copy_(t0), msk.copy_(m0), nb.fill_(1)
    gl.replay()
    torch.cuda.synchronize()
    assert torch.equal(tok, final_e[0]) and torch.equal(msk, final_e[1])


def test_step_without_branches_passes_through(L):
    """n_branches = 0 (a complete block fed back into the step, R21): row 0 passes through,
    n_branches_next = 0, winner 0 — so a graph-captured loop rests at its fixed point."""
    V, W, k = 64, 8, 2
    st = L.Stepper(V, W, k + 1, k, 0.9, DEV)
    tok = torch.arange((k + 1) * W, dtype=torch.int32, device=DEV).reshape(k + 1, W)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=DEV)
    nb = torch.zeros(1, dtype=torch.int32, device=DEV)
    logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=DEV)
    o = st.step(logits, nb, tok, msk)
    torch.cuda.synchronize()
    assert int(o.n_next.item()) == 0 and int(o.winner.item()) == 0 and int(o.status.item()) == 0
    assert torch.equal(o.next_tokens[0], tok[0]) and torch.equal(o.next_mask[0], msk[0])


def test_logits_prefetch_switch_bit_identical(L):
    """lopa_set_logits_prefetch(0) (K1's first copy after the PDL wait) gives the same bits as the
    default early copy, on the Dream step and through a chained sequence of steps."""
    import numpy as np
    V, W, k, tau = 151936, 32, 7, 0.9
    st = L.Stepper(V, W, k + 1, k, tau, DEV)
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=DEV)
    msk = torch.ones((k + 1, W), dtype=torch.uint8, device=DEV)
    nb = torch.full((1,), k + 1, dtype=torch.int32, device=DEV)
    g = torch.Generator(device=DEV).manual_seed(5)
    logits = [(torch.randn((k + 1, W, st.ld), device=DEV, generator=g) * 2).to(torch.bfloat16)
              for _ in range(3)]
    outs = {}
    for pf in (True, False):
        prev = L.set_logits_prefetch(pf)
        try:
            res = []
            for x in logits:
                o = st.step(x, nb, tok, msk)
                torch.cuda.synchronize()
                res.append((o.conf.clone(), o.argmax.clone(), o.winner.clone(), o.next_tokens.clone()))
        finally:
            L.set_logits_prefetch(prev)
        outs[pf] = res
    for a, b in zip(outs[True], outs[False]):
        for u, v in zip(a, b):
            assert torch.equal(u.view(torch.int32) if u.dtype == torch.float32 else u,
                               v.view(torch.int32) if v.dtype == torch.float32 else v)
