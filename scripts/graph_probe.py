"""Which part of lopa_step breaks CUDA-graph capture?  Harness only."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2512_16229_b200 import lopa
dev = "cuda:0"
V, W, k = 1000, 32, 5
st = lopa.Stepper(V, W, k + 1, k, 0.9, dev)
tok = torch.zeros((k + 1, W), dtype=torch.int32, device=dev)
msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=dev)
msk[0] = 1
nb = torch.ones(1, dtype=torch.int32, device=dev)
lg = torch.randn((k + 1, W, 1000), device=dev).to(torch.bfloat16)
st.step(lg, nb, tok, msk)
c = torch.rand(W, device=dev); am = torch.zeros(W, dtype=torch.int32, device=dev)
lopa.anchor_fill(c, am, tok[0], msk[0], 0.9)
torch.cuda.synchronize()
L = lopa.lib()


def try_capture(name, fn):
    g = torch.cuda.CUDAGraph()
    rcs = []
    try:
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            rcs.append(fn())
        g.replay(); torch.cuda.synchronize()
        print(name, "ok", rcs)
    except Exception as e:
        print(name, "FAIL", rcs, str(e).splitlines()[0])
        torch.cuda.synchronize()


try_capture("torch add", lambda: (tok.add_(0), 0)[1])
try_capture("anchor_fill", lambda: (lopa.anchor_fill(c, am, tok[0], msk[0], 0.9), 0)[1])
try_capture("syn_generate", lambda: (lopa.syn_generate(1, 0, V, tok, msk, out=lg), 0)[1])
a = st.args(lg, nb, tok, msk)
try_capture("lopa_step", lambda: L.lopa_step(ctypes.byref(a), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
