# A/B the bench over library variants (no tests): VARIANTS="a b" bash scripts/ab.sh
mkdir -p gpurun_out
for v in "" ${VARIANTS}; do
  LOPA_LIB_VARIANT=$v timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_${v:-base}.log 2>&1; echo "rc=$?" >> gpurun_out/bench_${v:-base}.log
done
