# A/B the Dream step over library variants: VARIANTS="a b" REPS=2 BENCH_ARGS="--config x" bash scripts/ab_variants.sh
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-2}); do for v in "" ${VARIANTS}; do
  LOPA_LIB_VARIANT=$v timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline ${BENCH_ARGS} > /tmp/b.log 2>&1
  echo "$rep ${v:-base} ${BENCH_ARGS} $(python -c "
import json,sys; d=json.loads(open('/tmp/b.log').read().strip().splitlines()[-1])
print(round(d['ms_per_step']*1000,3), round(d['roofline']['frac'],4), round(d['dense_roofline']['frac'],4) if d.get('dense_roofline') else '', 'graph_loop', (d.get('graph_loop') or {}).get('us_per_iteration'))")" >> gpurun_out/ab.txt
done; done
