# LM-head A/B of library variants on --config lmhead-dream (100 steps, alternated)
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2 3; do for v in "" ${VARIANTS}; do
  LOPA_LIB_VARIANT=$v timeout 300 python bench.py --config lmhead-dream --steps 100 --warmup 5 --no-cpu-baseline > /tmp/l.log 2>&1
  python -c "
import json
d=json.loads([l for l in open('/tmp/l.log') if l.startswith('{')][-1])
print('$rep ${v:-base}', round(d['ms_per_step']*1e3,2), round(d['roofline']['kernel_ms_mean']*1e3,2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])
" >> gpurun_out/lmh_ab3.txt 2>&1 || tail -3 /tmp/l.log >> gpurun_out/lmh_ab3.txt
done; done
