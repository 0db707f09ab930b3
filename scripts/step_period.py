"""Chained Dream steps (bench.py's workload and launch pattern) timed with CUDA events, no result
checks: for experiment builds (LOPA_LIB_VARIANT=...) whose results are not meant to be right."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2512_16229_b200 import lopa  # noqa: E402

dev = torch.device("cuda:0")
st, tok, msk, nb, full, bufs, rows, _ = bench.build_workload(lopa, dev, 151936, 32, 7, 0.9, 1, 8)
L = lopa.lib()
argv = [st.args(b, nb, tok, msk) for b in bufs]
refs = [ctypes.byref(a) for a in argv]
s = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
for i in range(50):
    L.lopa_step(refs[i % 8], s)
torch.cuda.synchronize()
res = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bench.head_start(torch.cuda.current_stream(dev))
    e0.record()
    for i in range(2000):
        L.lopa_step(refs[i % 8], s)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) * 1000 / 2000)
print(sys.argv[1] if len(sys.argv) > 1 else "", " ".join(f"{x:.3f}" for x in res))
