mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
LOPA_LIB_VARIANT=p1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_p1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_p1.log
VARIANTS="p1 p2" bash scripts/ab.sh
