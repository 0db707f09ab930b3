"""Which tile widths N does the CTA-pair MMA get right?  V = 74 N gives every pair one N-column
tile (74 pairs on a B200); rows 0..255 against fp64 numpy."""
import numpy as np
import torch

import syngen
from paper_2512_16229_b200 import lopa as L

DEV = "cuda:0"


def dev(u16):
    return torch.from_numpy(np.ascontiguousarray(u16).view(np.int16)).to(DEV).view(torch.bfloat16)


def f32(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


for N in (16, 32, 48, 64, 80, 96, 112, 128, 144, 160, 192, 224, 240, 256):
    M, K, V = 256, 64, 74 * N
    h, W, _ = syngen.lmhead_inputs(N, M, K, V)
    head = L.LMHead(dev(W), max_rows=256)
    c, a, st = head(dev(h))
    torch.cuda.synchronize()
    gc, ga = c.cpu().numpy().astype(np.float64), a.cpu().numpy()
    Lg = f32(h) @ f32(W).T
    rc = 1.0 / np.exp(Lg - Lg.max(1, keepdims=True)).sum(1)
    rel = np.abs(gc - rc) / rc
    print(f"N={N}: rel max {rel.max():.2e} argmax mism {int((ga != Lg.argmax(1)).sum())}", flush=True)
