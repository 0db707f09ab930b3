"""Per-warp timeline of the warp-staged K1 (LOPA_LDG_TL build): one Dream-step K1 launch alone."""
import ctypes
import os
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
L.lopa_debug_ldg_timeline.restype = ctypes.c_int
L.lopa_debug_ldg_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
need = -L.lopa_debug_ldg_timeline(None, 0)
ws = lopa.new_workspace(rows, V, dev)
st = lopa.new_status(dev)
for rep in range(3):
    lopa.confidence(x, vocab=V, row_mask=mask, workspace=ws, status=st)
    torch.cuda.synchronize()
buf = np.zeros(need, dtype=np.uint64)
L.lopa_debug_ldg_timeline(buf.ctypes.data, need)
nw = int(os.environ.get("NWARPS", "16"))
items = 40
a = buf.reshape(160, nw, 2 + 3 * items).astype(np.int64)
G = 148
a = a[:G]
t0 = a[:, :, 0][a[:, :, 0] > 0].min()
def us(v):
    return (v - t0) / 1000.0
print("start  med %.2f max %.2f" % (np.median(us(a[:, :, 0])), us(a[:, :, 0]).max()))
print("masks  med %.2f max %.2f" % (np.median(us(a[:, :, 1])), us(a[:, :, 1]).max()))
for k in range(12):
    s, w, c = a[:, :, 2 + 3 * k], a[:, :, 3 + 3 * k], a[:, :, 4 + 3 * k]
    ok = (c > 0) & (w > 0) & (s > 0)
    if not ok.any():
        break
    print("item %2d: begin med %6.2f  landed med %6.2f  consumed med %6.2f | stage+wait %5.2f us  consume %5.2f us (n=%d)" % (
        k, np.median(us(s[ok])), np.median(us(w[ok])), np.median(us(c[ok])),
        np.median((w - s)[ok]) / 1000, np.median((c - w)[ok]) / 1000, ok.sum()))
# ends
last = np.where(a[:, :, 4::3] > 0, a[:, :, 4::3], 0).max(axis=2)
print("warp end med %.2f max %.2f" % (np.median(us(last[last > 0])), us(last[last > 0]).max()))
# leader warps: waits
