# Small launches (BP-shard-sized steps): k = 0 / 1 / 3 (32 / 64 / 128 rows), product vs variants
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do for kk in 0 1 3; do for v in "" ${VARIANTS}; do
  LOPA_LIB_VARIANT=$v timeout 300 python bench.py --k $kk --steps 2000 --warmup 20 --no-cpu-baseline > /tmp/s.log 2>&1
  echo "$rep k=$kk ${v:-base} $(python -c "
import json; d=json.loads([l for l in open('/tmp/s.log') if l.startswith('{')][-1])
print(round(d['ms_per_step']*1000,3), d['config'].get('masked_rows'), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms_mean']*1000,2) if 'kernel_ms_mean' in d['roofline'] else '')" 2>&1 | tail -1)" >> gpurun_out/ab_small.txt
done; done; done
