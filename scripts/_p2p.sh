mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "bp" tests/test_gpu_bp.py -q -x -p no:cacheprovider > gpurun_out/pytest_p2p.log 2>&1; echo rc=$? >> gpurun_out/pytest_p2p.log
: > gpurun_out/ab_p2p.txt
for rep in 1 2; do
for v in base p2p3k; do
  for p2p in 0 1; do
    if [ $v = p2p3k ] && [ $p2p = 0 ]; then continue; fi
    if [ $v = base ]; then unset LOPA_LIB_VARIANT; else export LOPA_LIB_VARIANT=$v; fi
    LOPA_BENCH_FORCE_BP=1 LOPA_BP_P2P=$p2p timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline > /tmp/b.log 2>&1
    echo "$rep $v p2p=$p2p $(python -c "
import json; d=json.loads([l for l in open('/tmp/b.log') if l.startswith('{')][-1]); print(round(d['ms_per_step']*1000,3), d['config']['parallelism'], d['step_time_distribution']['isolated_step_us']['p50'])")" >> gpurun_out/ab_p2p.txt
  done
done; done
unset LOPA_LIB_VARIANT
