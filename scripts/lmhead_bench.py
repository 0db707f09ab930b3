"""Fused LM-head + Conf (lopa_lmhead_confidence) vs the unfused path (cuBLAS bf16 GEMM writing
the logits, then lopa_confidence reading them), Dream-7B shapes.  Harness only."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2512_16229_b200 import lopa

dev = torch.device("cuda", 0)
M, K, V = int(os.environ.get("M", 241)), 3584, 151936
g = torch.Generator(device=dev).manual_seed(0)
NW = int(os.environ.get("NW", 2))  # rotating weight copies (2 x 1.09 GB > L2)
Ws = [(torch.randn(V, K, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16) for _ in range(NW)]
H = (torch.randn(M, K, device=dev, generator=g) * 1.5).to(torch.bfloat16)
heads = [lopa.LMHead(W) for W in Ws]
s = torch.cuda.current_stream()
N = int(os.environ.get("N", 50))


def timed(fn, n=N):
    for i in range(3):
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


fused = timed(lambda i: heads[i % NW](H))
logits = torch.empty(M, V, dtype=torch.bfloat16, device=dev)
gemm = timed(lambda i: torch.matmul(H, Ws[i % NW].t(), out=logits))
rm = torch.ones(M, dtype=torch.uint8, device=dev)
ws = lopa.new_workspace(M, V, dev)
co = torch.empty(M, dtype=torch.float32, device=dev)
ao = torch.empty(M, dtype=torch.int32, device=dev)
stt = lopa.new_status(dev)
L = lopa.lib()
P = lopa._p
sp = ctypes.c_void_p(s.cuda_stream)


def unfused(i):
    torch.matmul(H, Ws[i % NW].t(), out=logits)
    L.lopa_confidence(P(logits), V, M, V, P(rm), P(co), P(ao), P(stt), P(ws), ws.numel(), sp)


unf = timed(unfused)
wb = V * K * 2
fl = 2.0 * M * K * V
print(f"M={M} K={K} V={V}")
print(f"fused lmhead+conf : {fused:8.1f} us  weight stream {wb / fused / 1e3:7.1f} GB/s  {fl / fused / 1e6:7.1f} TFLOP/s")
print(f"cuBLAS GEMM only  : {gemm:8.1f} us  {fl / gemm / 1e6:7.1f} TFLOP/s")
print(f"cuBLAS + a1 conf  : {unf:8.1f} us")
c1, a1, _ = heads[0](H)
torch.matmul(H, Ws[0].t(), out=logits)
L.lopa_confidence(P(logits), V, M, V, P(rm), P(co), P(ao), P(stt), P(ws), ws.numel(), sp)
torch.cuda.synchronize()
print("argmax agreement fused vs unfused(bf16 logits):", (a1 == ao).float().mean().item(),
      "max conf diff", (c1 - co).abs().max().item())

if hasattr(L, "lopa_debug_lmhead_prof"):
    import numpy as np
    buf = (ctypes.c_ulonglong * (256 * 8))()
    L.lopa_debug_lmhead_prof(buf, 256)          # clear
    heads[0](H)
    torch.cuda.synchronize()
    L.lopa_debug_lmhead_prof(buf, 256)
    a = np.array(buf[:], dtype=np.uint64).reshape(256, 8)[:148].astype(np.float64)
    tot = a[:, 5] - a[:, 6]
    names = ["prod wait empty", "mma wait tempty", "mma wait full", "epi wait tfull", "epi busy"]
    print("one launch, per-CTA cycles (median over CTAs): total %.0f" % np.median(tot))
    for j, nm in enumerate(names):
        print(f"  {nm:16s} {np.median(a[:, j]):10.0f}  ({np.median(a[:, j] / tot) * 100:5.1f}%)")
