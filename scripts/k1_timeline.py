"""Per-item timeline of K1's TMA form (LOPA_K1_TL build): one Dream-step K1 launch alone.
Producer: how long each copy waited for a free stage; consumers: how long each warpgroup waited
for data and how long it computed."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_16229_b200 import lopa

dev = torch.device("cuda:0")
V, W, K = 151936, 32, 7
rows = (K + 1) * W
x = (torch.randn((rows, V), device=dev) * 2).to(torch.bfloat16)
mask = torch.ones(rows, dtype=torch.uint8, device=dev)
mask[241:] = 0
L = lopa.lib()
L.lopa_debug_k1_timeline.restype = ctypes.c_int
L.lopa_debug_k1_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
need = -L.lopa_debug_k1_timeline(None, 0)
ws = lopa.new_workspace(rows, V, dev)
st = lopa.new_status(dev)
for rep in range(3):
    lopa.confidence(x, vocab=V, row_mask=mask, workspace=ws, status=st)
    torch.cuda.synchronize()
buf = np.zeros(need, dtype=np.uint64)
L.lopa_debug_k1_timeline(buf.ctypes.data, need)
a = buf.reshape(160, -1).astype(np.int64)[:148]
valid = a[:, 1] > 0
a = a[valid]
t0 = a[:, 1].min()
us = lambda v: (v - t0) / 1000.0
print("CTAs", len(a))
print("producer: item  wait-begin  issued  blocked(us)   [medians over CTAs]")
for i in range(0, 24):
    wb, iss = a[:, 2 * i], a[:, 2 * i + 1]
    ok = (wb > 0) & (iss > 0)
    if ok.sum() < 10:
        break
    print("  %2d  %6.2f  %6.2f  %5.2f  (n=%d)" % (i, np.median(us(wb[ok])), np.median(us(iss[ok])),
                                                np.median((iss - wb)[ok]) / 1000, ok.sum()))
print("consumer warpgroups: n  full-return  done  compute(us)  wait-before(us)")
for wg in range(6):
    print(" wg", wg)
    prev = None
    for n in range(16):
        f, d = a[:, 96 + 48 * wg + 3 * n], a[:, 96 + 48 * wg + 3 * n + 2]
        ok = (f > 0) & (d > 0)
        if ok.sum() < 10:
            break
        wait = np.median((f - prev)[ok & (prev > 0)]) / 1000 if prev is not None else float("nan")
        print("   %2d %6.2f %6.2f  %5.2f  %5.2f (n=%d)" % (n, np.median(us(f[ok])), np.median(us(d[ok])),
                                                     np.median((d - f)[ok]) / 1000, wait, ok.sum()))
        prev = d
