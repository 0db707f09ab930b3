import sys, os, torch
sys.path.insert(0, ".")
from paper_2512_16229_b200 import lopa as L
DEV = "cuda:0"
x = torch.zeros(1, device=DEV); y = torch.zeros(1, device=DEV)
fb = torch.zeros(1, dtype=torch.bool, device=DEV); w = torch.ones(1, dtype=torch.int32, device=DEV)
big_src = torch.arange(64, dtype=torch.int32, device=DEV); big_dst = torch.zeros(64, dtype=torch.int32, device=DEV)
def body():
    x.add_(1)
    y.copy_(x)
    big_dst.copy_(big_src + 0) if False else big_dst.copy_(big_src)
    big_src.add_(1)
    torch.lt(x, 5, out=fb)
    w.copy_(fb)
wg = L.WhileGraph(body, w, until_zero=True, max_iters=100)
x.zero_(); y.zero_(); w.fill_(1); big_src.copy_(torch.arange(64, dtype=torch.int32, device=DEV))
wg.launch(); torch.cuda.synchronize()
print("iters", wg.iterations(), "x", x.item(), "y", y.item(), "big_dst[:4]", big_dst[:4].tolist(), "big_src[:4]", big_src[:4].tolist())
