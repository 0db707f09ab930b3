mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
LOPA_LIB_VARIANT=checked PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_checked.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
