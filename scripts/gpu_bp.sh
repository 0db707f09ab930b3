# BP round: new BP GPU tests, the loop configs (1 GPU; FORCE_BP = the N > 1 code path), default bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bp.py -q -x --timeout 1100 -p no:cacheprovider > gpurun_out/pytest_bp.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bp.log
timeout 600 python bench.py --config dream-loop --steps 200 --warmup 5 > gpurun_out/b_loop.log 2>&1; echo "rc=$?" >> gpurun_out/b_loop.log
LOPA_BENCH_FORCE_BP=1 timeout 600 python bench.py --config dream-loop --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/b_loop_bp.log 2>&1; echo "rc=$?" >> gpurun_out/b_loop_bp.log
LOPA_BENCH_FORCE_BP=1 timeout 600 python bench.py --config diffucoder-loop --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b_loop_dc.log 2>&1; echo "rc=$?" >> gpurun_out/b_loop_dc.log
LOPA_BENCH_FORCE_BP=1 timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/b_forcebp.log 2>&1; echo "rc=$?" >> gpurun_out/b_forcebp.log
timeout 300 python bench.py --config dream-loop --impl reference --steps 20 --warmup 3 > gpurun_out/b_loop_ref.log 2>&1; echo "rc=$?" >> gpurun_out/b_loop_ref.log
