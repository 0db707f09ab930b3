# Round-end evidence, one gpurun call: bench lines (each plain run exits 0 before its ncu pass),
# the launch list, --set full of K1/K2 and of the fused LM head.
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 400 python bench.py --config lmhead-dream --steps 500 > gpurun_out/bench_lmh.log 2>&1; echo "rc=$?" >> gpurun_out/bench_lmh.log
timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b20.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?" >> gpurun_out/b20.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lopa_(reduce|tail)" -s 8 -c 4 -o gpurun_out/prof_full -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/b20.log
N=3 NW=1 timeout 300 python scripts/lmhead_bench.py > gpurun_out/lmhb_plain.log 2>&1 && \
N=3 NW=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:lopa_lmhead_kernel -s 2 -c 1 -o gpurun_out/prof_lmh -f python scripts/lmhead_bench.py > gpurun_out/ncu_lmh.log 2>&1; echo "ncu lmh rc=$?" >> gpurun_out/b20.log
LOPA_LIB_VARIANT=tl REPS=2 timeout 120 python scripts/timeline.py > gpurun_out/tl.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
