"""Randomised stress of the round-2 paths (not part of the suite): branch-parallel decodes at
random G / k / W / V against the single-GPU loop (bit-identical) with sampled per-step oracle
checks, and device-scheduled D2F decodes against the host pipeline.
Usage: python scripts/stress_r02.py [seconds] [seed]."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch
import _gpu as G
from paper_2512_16229_b200 import d2f, lopa

dev = "cuda:0"


def _checked_violations():
    """Violations counted by a -DLOPA_CHECKED build (LOPA_LIB_VARIANT=checked), else 0."""
    import ctypes
    out = (ctypes.c_uint32 * 3)()
    st = lopa.lib().lopa_debug_check_read(ctypes.cast(out, ctypes.c_void_p))
    if st == 0 and out[0]:
        raise AssertionError(f"checked build: {out[0]} violations, first site {out[1]}, sites {out[2]:#x}")
    return st == 0

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0 = time.time()
n_bp = n_d2f = n_checked = 0
while time.time() - t0 < budget:
    V = int(rng.choice([7, 64, 1000, 8193, 151936]))
    seed = int(rng.integers(0, 1 << 30))
    extras = int(rng.integers(0, 2)) if V >= 8 else 0
    if rng.random() < 0.6:
        W = int(rng.choice([1, 4, 8, 16, 32, 64]))
        k = int(rng.integers(0, min(31, 4096 // W - 1) + 1))
        world = int(rng.integers(1, 9))
        tau = float(rng.choice([0.5, 0.9, 0.95]))
        fwd = lambda t, m, out: lopa.syn_generate(seed, 0, V, t, m, extras=extras, out=out)
        t0_ = torch.zeros(W, dtype=torch.int32, device=dev)
        m0_ = torch.ones(W, dtype=torch.uint8, device=dev)
        st = lopa.Stepper(V, W, k + 1, k, tau, dev)
        emu = lopa.BPEmulator(st, world)
        check = rng.random() < 0.3 and V * W * (k + 1) < 5e7

        def on_step(out, n, tok, msk):
            global n_checked
            if not check:
                return
            torch.cuda.synchronize()
            logits = np.zeros((n, W, st.ld), dtype=np.uint16)
            for _, lo, hi, buf in emu.ranks():
                m = max(0, min(hi, n) - lo)
                if m:
                    logits[lo:lo + m] = G.to_np_u16(buf[:m])
            conf, amax = emu.gathered()
            from types import SimpleNamespace
            o = SimpleNamespace(conf=conf, argmax=amax, scores=emu.scores, winner=out.winner,
                                n_next=out.n_next, next_tokens=out.next_tokens, next_mask=out.next_mask,
                                lookahead=out.lookahead, status=out.status)
            G.check_step(o, logits, tok.cpu().numpy(), msk.cpu().numpy(), n, k, tau, vocab=V)
            n_checked += 1

        tb, fb = lopa.decode_block_bp(emu, fwd, t0_, m0_, on_step=on_step)
        ts, fs = lopa.decode_block(fwd, t0_, m0_, k, tau, V)
        assert fb == fs and torch.equal(tb, ts), ("BP", V, W, k, world, seed)
        assert int(st.out.status.item()) == 0
        n_bp += 1
    else:
        B = int(rng.choice([4, 8, 16, 32]))
        L_ = B * int(rng.integers(1, 9))
        k = int(rng.integers(0, 16))
        mw = B * int(rng.integers(1, max(2, 256 // B) + 1))
        mw = min(mw, 256)
        cfg = d2f.BlockConfig(B, float(rng.choice([0.1, 0.25, 0.5, 1.0])), 0.95, 0.9, mw)
        V = min(V, 20000)
        fwdb = lambda b, t, m: lopa.syn_generate(seed, b, V, t, m, extras=extras)
        h = d2f.decode_d2f(fwdb, L_, k, cfg, V, dev)
        loop = d2f.D2FDeviceLoop(L_, k, cfg, V, dev, seed, extras=extras)
        loop.reset()
        loop.run(h.forwards + 2)
        torch.cuda.synchronize()
        g = loop.trace()
        assert (g.forwards, g.windows, g.winners, g.branch_counts, g.commits) == \
               (h.forwards, h.windows, h.winners, h.branch_counts, h.commits), ("D2F", B, L_, k, mw, seed)
        assert torch.equal(g.tokens, h.tokens)
        n_d2f += 1
    if (n_bp + n_d2f) % 200 == 0:
        _checked_violations()
checked = _checked_violations()
print(("checked build, 0 violations; " if checked else "") + f"stress_r02: {n_bp} BP decodes ({n_checked} steps oracle-checked), {n_d2f} device D2F "
      f"decodes, {time.time() - t0:.0f} s, no failure")
