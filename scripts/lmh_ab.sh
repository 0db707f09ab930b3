cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in base st4 st6 single; do
  unset LOPA_LIB_VARIANT LOPA_LMH_SINGLE
  [ $v = st4 ] && export LOPA_LIB_VARIANT=st4
  [ $v = st6 ] && export LOPA_LIB_VARIANT=st6
  [ $v = single ] && export LOPA_LMH_SINGLE=1
  timeout 300 python bench.py --config lmhead-dream --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_lmh_$v.log 2>&1
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/b_lmh_$v.log') if l.startswith('{')][-1])
print('$v', round(d['ms_per_step']*1e3,2), round(d['roofline']['kernel_ms_mean']*1e3,2), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])
" >> gpurun_out/lmh_ab.txt 2>&1 || tail -3 gpurun_out/b_lmh_$v.log >> gpurun_out/lmh_ab.txt
done; done
unset LOPA_LIB_VARIANT LOPA_LMH_SINGLE
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lopa_lmhead_pair -s 3 -c 1 -o gpurun_out/lmh_pair_full python bench.py --config lmhead-dream --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_lmh.log 2>&1
echo ncu rc=$? >> gpurun_out/lmh_ab.txt
