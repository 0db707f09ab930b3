# Late round-2 refresh of the default bench's launch list and the --set full capture of K1 / K2
mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b20.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lopa_reduce_kernel|lopa_tail" -s 8 -c 2 -o gpurun_out/prof_full_r02 -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full.log
