"""Chained Dream steps (as bench.py's timed region) with per-step marks (LOPA_CHAIN_TL build):
where each step's time goes between consecutive K1 launches."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_16229_b200 import lopa  # noqa: E402

dev = torch.device("cuda:0")
st, tok, msk, nb, full, bufs, rows, _ = bench.build_workload(lopa, dev, 151936, 32, 7, 0.9, 1, 8)
L = lopa.lib()
buf = np.zeros(768, dtype=np.uint64)
L.lopa_debug_chain_timeline(buf.ctypes.data, 768)   # clear
argv = [st.args(b, nb, tok, msk) for b in bufs]
s = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
for i in range(10):
    L.lopa_step(ctypes.byref(argv[i % 8]), s)
torch.cuda.synchronize()
L.lopa_debug_chain_timeline(buf.ctypes.data, 768)   # clear again
bench.head_start(torch.cuda.current_stream(dev))
for i in range(40):
    L.lopa_step(ctypes.byref(argv[i % 8]), s)
torch.cuda.synchronize()
L.lopa_debug_chain_timeline(buf.ctypes.data, 768)
a = buf.reshape(64, 12).astype(np.int64)
ok = [e for e in range(64) if a[e, 1] > 0 and a[e, 5] > 0 and a[e, 6] < (1 << 62)]
ok.sort(key=lambda e: a[e, 6])
names = ["K1 start(wait done)", "K1 end", "K2 start", "K2 folded", "scores", "anchor", "ranks", "tables", "K2 decided", "K2 wait ret"]
cols = [6, 1, 2, 3, 7, 8, 9, 10, 4, 5]
base = a[ok[0], 6]
print("step | " + " | ".join(names) + " | period (us)")
prev = None
for e in ok[:30]:
    t = [(a[e, c] - a[e, 6]) / 1000.0 for c in cols]
    per = (a[e, 6] - prev) / 1000.0 if prev is not None else float("nan")
    prev = a[e, 6]
    print(f"{e:3d} | " + " | ".join(f"{x:7.2f}" for x in t) + f" | {per:.2f}")
