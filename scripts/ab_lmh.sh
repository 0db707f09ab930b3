mkdir -p gpurun_out
for rep in 1 2; do for v in "" lmh0; do
  LOPA_LIB_VARIANT=$v timeout 300 python bench.py --config lmhead-dream --steps 300 --warmup 5 --no-cpu-baseline > /tmp/b.log 2>&1
  echo "lmh $rep ${v:-base} $(python -c "import json,sys; d=json.loads(open('/tmp/b.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,3), round(d['roofline']['frac'],4), d['clocks'])")" >> gpurun_out/ab.txt
done; done
VARIANTS="ec0" REPS=2 bash scripts/ab_variants.sh
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
