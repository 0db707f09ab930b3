mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
LOPA_LIB_VARIANT=checked PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_checked.log
VARIANTS="nopoll" REPS=2 bash scripts/ab_variants.sh
