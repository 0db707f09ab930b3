"""K2 phase durations in SM cycles (LOPA_K2_CYC build: thread 0 stamps clock64 at each phase
boundary of chained Dream steps; no K1 marks).  Columns are deltas between consecutive marks."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_16229_b200 import lopa  # noqa: E402

dev = torch.device("cuda:0")
W_, K_ = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (32, 7)
st, tok, msk, nb, full, bufs, rows, _ = bench.build_workload(lopa, dev, 151936, W_, K_, 0.9, 1, 8)
L = lopa.lib()
buf = np.zeros(2048, dtype=np.uint64)
nw = L.lopa_debug_chain_timeline(buf.ctypes.data, 2048)
argv = [st.args(b, nb, tok, msk) for b in bufs]
s = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
for i in range(10):
    L.lopa_step(ctypes.byref(argv[i % 8]), s)
torch.cuda.synchronize()
nw = L.lopa_debug_chain_timeline(buf.ctypes.data, 2048)
bench.head_start(torch.cuda.current_stream(dev))
for i in range(40):  # noqa
    L.lopa_step(ctypes.byref(argv[i % 8]), s)
torch.cuda.synchronize()
nw = L.lopa_debug_chain_timeline(buf.ctypes.data, 2048)
a = buf[:nw].reshape(64, nw // 64).astype(np.int64)
order = [2, 3, 12, 13, 14, 0, 7, 1, 6, 11, 8, 9, 10, 4, 5]
names = ["prologue->folded", "folded->loaded", "loaded->reduced", "reduced->divided", "divided->scores(t0)", "scores(t0)->synced", "synced->select",
         "select->anchored", "anchored->keys", "keys->bar", "bar->ranks", "ranks->tables",
         "tables->decided", "decided->wait ret"]
ok = [e for e in range(64) if all(a[e, c] > 0 for c in order)]
d = np.array([[a[e, order[j + 1]] - a[e, order[j]] for j in range(len(order) - 1)] for e in ok])
print(f"{len(ok)} steps; cycles (median / p10 / p90) per phase; 1 us ~ 1965 cycles")
for j, n in enumerate(names):
    print(f"{n:22s} {int(np.median(d[:, j])):7d} {int(np.percentile(d[:, j], 10)):7d} {int(np.percentile(d[:, j], 90)):7d}")
