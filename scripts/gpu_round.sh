# one gpurun call: GPU tests, smoke, bench A/B over tuning variants, ncu of the top kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for v in "" ${VARIANTS}; do
  LOPA_LIB_VARIANT=$v timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_${v:-base}.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${v:-base}.log
done
timeout 300 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "${NCU}" ]; then
timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b20.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lopa_reduce -s 6 -c 2 -o gpurun_out/prof_full -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/b20.log
fi
