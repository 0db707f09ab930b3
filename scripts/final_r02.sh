# Round-2 full check: GPU suite, checked suite, smoke, default bench, loop / D2F / lmhead configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest_gpu.log
LOPA_LIB_VARIANT=checked PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider > gpurun_out/final_pytest_checked.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest_checked.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 400 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final_bench.log
timeout 400 python bench.py --config dream-loop --steps 300 > gpurun_out/final_bench_loop.log 2>&1
timeout 400 python bench.py --config diffucoder-loop --steps 300 --no-cpu-baseline > gpurun_out/final_bench_dcloop.log 2>&1
timeout 400 python bench.py --config d2f-graph --steps 500 > gpurun_out/final_bench_d2f.log 2>&1
timeout 400 python bench.py --config lmhead-dream --steps 200 --warmup 5 > gpurun_out/final_bench_lmhead.log 2>&1
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1
