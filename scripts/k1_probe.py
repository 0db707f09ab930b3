"""Where does the event-timed K1 duration come from?  Compares, on the bench workload:
headline steps (events at the ends), the library's per-K1 event pairs, and confidence-only
loops.  Harness only."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_16229_b200 import lopa

dev = torch.device("cuda", 0)
V, W, k, tau = 151936, 32, 7, 0.9
st, tok, msk, nb, full, bufs, rows, _ = bench.build_workload(lopa, dev, V, W, k, tau, 1, 8)
s = torch.cuda.current_stream()
N = 1000


def timed(fn, n=N):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    bench.head_start(s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n


step = lambda i: st.step(bufs[i % 8], nb, tok, msk, validate=False)
print("headline step (events at ends): %.2f us" % timed(step))
lopa.profile_enable(N)
bench.head_start(s)
for i in range(N):
    step(i)
torch.cuda.synchronize()
per = lopa.profile_read(N)
print("per-K1 event pairs inside steps: mean %.2f med %.2f min %.2f us" % (
    statistics.mean(per) * 1e3, statistics.median(per) * 1e3, min(per) * 1e3))
rm = (msk[: int(nb.item())].reshape(-1) != 0).to(torch.uint8)
rows_all = torch.zeros((k + 1) * W, dtype=torch.uint8, device=dev)
rows_all[: rm.numel()] = rm
ld = bufs[0].shape[-1]
nr = (k + 1) * W
c_out = torch.empty(nr, dtype=torch.float32, device=dev)
a_out = torch.empty(nr, dtype=torch.int32, device=dev)
stt = lopa.new_status(dev)
ws = lopa.new_workspace(nr, V, dev)
L = lopa.lib()
sp = ctypes.c_void_p(s.cuda_stream)
P = lopa._p


def conf(i):
    L.lopa_confidence(P(bufs[i % 8]), ld, nr, V, P(rows_all), P(c_out), P(a_out), P(stt), P(ws),
                      ws.numel(), sp)
print("confidence (K1 + fold kernel) loop: %.2f us" % timed(conf))
lopa.profile_enable(N)
bench.head_start(s)
for i in range(N):
    conf(i)
torch.cuda.synchronize()
per = lopa.profile_read(N)
print("per-K1 event pairs inside confidence: mean %.2f med %.2f min %.2f us" % (
    statistics.mean(per) * 1e3, statistics.median(per) * 1e3, min(per) * 1e3))
