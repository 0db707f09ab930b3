"""Debug probe for the CTA-pair LM head: per-row errors against fp64 numpy, split by CTA rank
(rows < 128 / >= 128), and a planted-column probe (logits[r][v] = 8 only at v = c_r)."""
import numpy as np
import torch

import syngen
from paper_2512_16229_b200 import lopa as L

DEV = "cuda:0"


def dev(u16):
    return torch.from_numpy(np.ascontiguousarray(u16).view(np.int16)).to(DEV).view(torch.bfloat16)


def f32(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def run(h, W):
    head = L.LMHead(dev(W), max_rows=256)
    c, a, st = head(dev(h))
    torch.cuda.synchronize()
    return c.cpu().numpy().astype(np.float64), a.cpu().numpy(), int(st.item())


for (M, K, V) in [(256, 64, 18944), (256, 64, 8200), (129, 64, 8200), (256, 128, 151936 // 8)]:
    h, W, _ = syngen.lmhead_inputs(M * 7 + V, M, K, V)
    gc, ga, st = run(h, W)
    Lg = f32(h) @ f32(W).T
    m = Lg.max(1, keepdims=True)
    rc = 1.0 / np.exp(Lg - m).sum(1)
    ra = Lg.argmax(1)
    rel = np.abs(gc - rc) / rc
    print(f"M={M} K={K} V={V} st={st} rel<128 max {rel[:128].max():.3e} med {np.median(rel[:128]):.3e}"
          f" | rel>=128 max {rel[128:].max() if M > 128 else 0:.3e} | argmax mism {int((ga != ra).sum())}"
          f" first {np.nonzero(ga != ra)[0][:8].tolist()} {ga[np.nonzero(ga != ra)[0][:4]].tolist()} vs {ra[np.nonzero(ga != ra)[0][:4]].tolist()}",
          flush=True)

# planted probe
M = K = 256
for V in (18944, 74 * 256 * 2, 8200):
    h = np.zeros((M, K), np.float32)
    h[np.arange(M), np.arange(M)] = 1.0
    Wf = np.zeros((V, K), np.float32)
    c = (np.arange(M) * 7919) % V
    Wf[c, np.arange(M)] = 8.0
    hb = (h.view(np.uint32) >> 16).astype(np.uint16)
    Wb = (Wf.view(np.uint32) >> 16).astype(np.uint16)
    gc, ga, st = run(hb, Wb)
    exp_conf = 1.0 / (1.0 + (V - 1) * np.exp(-8.0))
    bad = np.nonzero(ga != c)[0]
    print(f"planted V={V}: argmax wrong {bad.size}; rows {bad[:10].tolist()} got {ga[bad[:10]].tolist()} want {c[bad[:10]].tolist()}"
          f" (want-v0 mod 256?) ; conf ratio min/max {(gc / exp_conf).min():.4f} {(gc / exp_conf).max():.4f}", flush=True)
