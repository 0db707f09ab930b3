# interleaved A/B of the bench over library variants, ROUNDS times: VARIANTS="a b" ROUNDS=2 bash scripts/ab2.sh
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
for v in base ${VARIANTS}; do
  vv=$v; [ "$v" = base ] && vv=""
  LOPA_LIB_VARIANT=$vv timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1e3,3), round(d['roofline']['kernel_ms_mean']*1e3,3), d['clocks']['sm_mhz'])" >> gpurun_out/ab.log 2>&1
done
done
