"""LM head (fused Conf) time vs rows at Dream shapes: V = 151936, K = 3584, two alternating
1.09 GB weight copies; CUDA events around 30 back-to-back calls per row count."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_16229_b200 import lopa  # noqa: E402

dev = torch.device("cuda:0")
V, K = 151936, 3584
g = torch.Generator(device=dev).manual_seed(0)
Ws = [(torch.randn(V, K, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16) for _ in range(2)]
heads = [lopa.LMHead(w, max_rows=256) for w in Ws]
for rows in (16, 32, 64, 128, 129, 160, 192, 256):
    H = (torch.randn(rows, K, device=dev, generator=g) * 1.5).to(torch.bfloat16)
    for i in range(4):
        heads[i % 2](H)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 30
    for i in range(n):
        heads[i % 2](H)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / n
    print(f"rows {rows:4d}: {us:7.1f} us  weights {V * K * 2 / us / 1e3:6.0f} GB/s  "
          f"{2 * rows * K * V / us / 1e6:6.0f} TF/s", flush=True)
