# A/B of library variants over several bench configs: VARIANTS="a b" CONFIGS="x y" bash scripts/ab_configs.sh
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do for c in ${CONFIGS}; do for v in "" ${VARIANTS}; do
  LOPA_LIB_VARIANT=$v timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline > /tmp/c.log 2>&1
  echo "$rep $c ${v:-base} $(python -c "
import json; d=json.loads([l for l in open('/tmp/c.log') if l.startswith('{')][-1])
print(round(d['ms_per_step']*1000,2), d['config'].get('masked_rows'), round(d['roofline']['frac'],3), (d.get('step_time_distribution') or {}).get('isolated_step_us',{}).get('p50'))" 2>&1 | tail -1)" >> gpurun_out/ab_configs.txt
done; done; done
