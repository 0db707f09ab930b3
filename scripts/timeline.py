"""Per-CTA phase timeline of the fused step kernel (needs the LOPA_TIMELINE build:
python -m paper_2512_16229_b200.build --variant tl -D LOPA_TIMELINE; run with LOPA_LIB_VARIANT=tl)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2512_16229_b200 import lopa

dev = torch.device("cuda", 0)
V, W, k, tau = 151936, 32, int(os.environ.get("K", 7)), 0.9
st, tok, msk, nb, full, bufs, rows, _ = bench.build_workload(lopa, dev, V, W, k, tau, 1, 8)
for i in range(30):
    st.step(bufs[i % 8], nb, tok, msk, validate=False)
torch.cuda.synchronize()
n = torch.cuda.get_device_properties(0).multi_processor_count
buf = (ctypes.c_ulonglong * (n * 24))()
for rep in range(int(os.environ.get('REPS', 3))):
    st.step(bufs[rep % 8], nb, tok, msk, validate=False)
    torch.cuda.synchronize()
    slots = lopa.lib().lopa_debug_timeline(buf, n)
    a = np.array(buf[:], dtype=np.uint64).reshape(n, 24).astype(np.int64)
    t0 = a[:, 0][a[:, 0] > 0].min()
    rel = (a - t0) / 1000.0
    names = ["cta_start", "producer", "first_data", "cons_exit", "k1_cta_end", "k2_end",
             "k2_start", "k2_folded", "gp_loaded", "anchored", "gp_bar", "rows_folded", "sp_rank", "sp_write", "prod_done", "fold_bar"]
    c = a[0]
    print(f"rep {rep}: rows={rows} k2 clocks after wait: row0 folded {c[17]-c[16]}, loop end {c[18]-c[16]}, "
          f"partials staged {c[23]-c[16]}, one read {c[21]-c[16]}, row0 divided {c[22]-c[16]}, fold barrier {c[19]-c[16]}, scores barrier {c[22]-c[16]}, end {c[20]-c[16]}")
    for j, nm in enumerate(names):
        col = rel[:, j]
        col = col[(a[:, j] > 0) & (a[:, j] >= t0)]
        if len(col):
            print(f"  {nm:11s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us  (n={len(col)})")
lu = rel[:, 3]
order = np.argsort(lu)
print("last_unit percentiles", np.percentile(lu, [0, 10, 25, 50, 75, 90, 95, 100]).round(2))
print("slowest CTAs (block, last_unit, first_data):", [(int(b), round(float(lu[b]), 2), round(float(rel[b, 2]), 2)) for b in order[-16:]])
print("fastest CTAs:", [(int(b), round(float(lu[b]), 2)) for b in order[:8]])
# K2 alone, back to back (warm): event timing
import ctypes as C
L = lopa.lib()
if hasattr(L, "lopa_debug_tail_only"):
    f = L.lopa_debug_tail_only
    f.argtypes = [C.POINTER(lopa.StepArgs), C.c_void_p]
    a = st.args(bufs[0], nb, tok, msk)
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(10): f(C.byref(a), sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): f(C.byref(a), sp)
    e1.record(); torch.cuda.synchronize()
    print("K2 alone back-to-back: %.2f us/launch" % (e0.elapsed_time(e1) * 1000 / 200))
    e0.record()
    for _ in range(200): st.step(bufs[0], nb, tok, msk, validate=False)
    e1.record(); torch.cuda.synchronize()
    print("full step same buffer (L2-warm logits) back-to-back: %.2f us/step" % (e0.elapsed_time(e1) * 1000 / 200))
