"""Randomised parity stress of lopa_step against the oracle (not part of the test suite):
random V, W, k, tau / per-position tau, Eq. 2 metric, branch states and SYN-D2F extras, each
step checked with tests/_gpu.check_step.  Usage: python scripts/stress.py [seconds] [seed]."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch
import syngen
import _gpu as G
from paper_2512_16229_b200 import lopa

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
t0, n_cases, n_steps = time.time(), 0, 0
while time.time() - t0 < budget:
    W = int(rng.choice([1, 2, 7, 8, 16, 31, 32, 33, 48, 64, 65, 96, 128, 200, 256]))
    kmax = min(31, 4096 // W - 1)
    k = int(rng.integers(0, kmax + 1))
    V = int(rng.choice([2, 7, 64, 100, 1000, 8192, 8193, 20000, 151936, 300000]))
    if W > 64 and V > (1 << 22):
        V = 151936
    if (k + 1) * W * V * 2 > 2e9:
        continue
    tau = float(rng.choice([0.5, 0.9, 0.95, 0.99]))
    metric = int(rng.choice([0, 0, 1, 2]))
    param = {0: 0.0, 1: float(rng.integers(1, 9)), 2: float(rng.choice([0.1, 0.3, 0.5, 1.0]))}[metric]
    taus = None
    if rng.random() < 0.3:
        taus = rng.choice(np.float32([0.5, 0.9, 0.95]), size=W).astype(np.float32)
    extras = int(rng.integers(0, 2)) if V >= 8 else 0
    seed = int(rng.integers(0, 1 << 30))
    st = lopa.Stepper(V, W, k + 1, k, tau, dev, metric=metric, metric_param=param,
                      tau_pos=None if taus is None else torch.from_numpy(taus).to(dev))
    tok, msk, nb = G.fresh_tables(k, W, dev)
    if rng.random() < 0.3:   # a partially filled start
        m0 = (rng.random(W) < 0.6).astype(np.uint8)
        m0[rng.integers(W)] = 1
        msk[0] = torch.from_numpy(m0).to(dev)
    logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=dev)
    for it in range(int(rng.integers(1, 4))):
        n = int(nb.item())
        lopa.syn_generate(seed, 0, V, tok, msk, n_branches=n, extras=extras, out=logits[:n])
        out = st.step(logits, nb, tok, msk)
        torch.cuda.synchronize()
        try:
            G.check_step(out, G.to_np_u16(logits), tok.cpu().numpy(), msk.cpu().numpy(), n, k,
                         tau if taus is None else taus, vocab=V, metric=metric, param=param)
        except AssertionError as e:
            print("FAIL", dict(V=V, W=W, k=k, tau=tau, metric=metric, param=param, taus=taus is not None,
                               extras=extras, seed=seed, it=it), repr(e)[:300], flush=True)
            raise
        n_steps += 1
        if int(out.n_next.item()) == 0:
            break
        tok, msk, nb = out.next_tokens.clone(), out.next_mask.clone(), out.n_next.clone()
    n_cases += 1
    if n_cases % 50 == 0:
        _checked_violations()
checked = _checked_violations()
print(f"stress ok ({'checked build, 0 violations' if checked else 'product build'}): {n_cases} cases, {n_steps} steps in {time.time() - t0:.0f} s", flush=True)
