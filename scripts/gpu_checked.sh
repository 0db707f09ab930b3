# The library's own sanitizer tier (compute-sanitizer is closed on this pool): the whole GPU suite
# and the every-kernel driver on the -DLOPA_CHECKED build, exact-size allocations
mkdir -p gpurun_out
export LOPA_LIB_VARIANT=checked
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1400 -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_checked.log
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 600 python - > gpurun_out/checked_drive.log 2>&1 <<'PY'
import ctypes, subprocess, sys
sys.path.insert(0, ".")
from paper_2512_16229_b200 import lopa
import scripts.sanitize_drive as d
out = (ctypes.c_uint32 * 3)()
for part in (d.part_core, d.part_bp, d.part_lmhead):
    part()
    st = lopa.lib().lopa_debug_check_read(ctypes.cast(out, ctypes.c_void_p))
    print(part.__name__, "status", st, "violations", out[0], "first site", out[1], "sites", hex(out[2]))
PY
echo "rc=$?" >> gpurun_out/checked_drive.log
