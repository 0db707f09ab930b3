# Round-2 evidence: sweep over every config (bench), ncu metrics of K1 per config, launch list of
# the default bench, one --set full capture of K1 (traffic)
mkdir -p gpurun_out
bash scripts/sweep.sh
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:lopa_reduce --csv --log-file gpurun_out/ncu_configs.csv python scripts/ncu_configs.py > gpurun_out/ncu_configs_order.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_configs_order.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b20.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lopa_reduce_kernel|lopa_tail" -s 8 -c 2 -o gpurun_out/prof_full_r02 -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full.log
