"""Pure-read and copy bandwidth probes with stock torch ops (context for the roofline)."""
import torch
x = torch.randn(512 * 1024 * 1024, device="cuda", dtype=torch.bfloat16)   # 1 GiB
y = torch.empty_like(x)
def t(f, n=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(n):
        a.record(); f(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best / 1000
nb = x.numel() * 2
print("copy  GB/s (r+w):", 2 * nb / t(lambda: y.copy_(x)) / 1e9)
print("amax  GB/s (read):", nb / t(lambda: torch.amax(x)) / 1e9)
print("sum   GB/s (read):", nb / t(lambda: x.sum(dtype=torch.float32)) / 1e9)
xv = x.view(4096, -1)
print("row amax GB/s (read):", nb / t(lambda: torch.amax(xv, dim=1)) / 1e9)
s = x[: 256 * 151936].view(256, 151936)
print("dream-size amax (77.8MB, L2-cold? no) GB/s:", s.numel() * 2 / t(lambda: torch.amax(s, dim=1), 50) / 1e9)
