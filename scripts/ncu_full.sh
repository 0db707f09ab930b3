# ncu --set full of the step kernels (K1 reduce + K2 tail) on the Dream bench; plain run first
mkdir -p gpurun_out
timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b20.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lopa_(reduce|tail)" -s 8 -c 4 -o gpurun_out/prof_full -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/b20.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/b20.log
