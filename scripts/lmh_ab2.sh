# LM-head A/B: pair kernel vs one CTA per SM, 200 steps each, alternated (clocks in the lines)
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2 3; do for v in pair single; do
  if [ $v = single ]; then export LOPA_LMH_SINGLE=1; else unset LOPA_LMH_SINGLE; fi
  timeout 300 python bench.py --config lmhead-dream --steps 200 --warmup 5 --no-cpu-baseline > /tmp/l.log 2>&1
  python -c "
import json
d=json.loads([l for l in open('/tmp/l.log') if l.startswith('{')][-1])
print('$rep $v', round(d['ms_per_step']*1e3,2), round(d['roofline']['kernel_ms_mean']*1e3,2), round(d['roofline']['frac'],3), d['clocks'])
" >> gpurun_out/lmh_ab2.txt 2>&1
done; done
nvidia-smi --query-gpu=temperature.gpu,power.draw,clocks.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/lmh_ab2.txt
