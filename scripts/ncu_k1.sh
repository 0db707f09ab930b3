mkdir -p gpurun_out
timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b20.log 2>&1 && \
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"lopa_reduce" -s 8 -c 1 -o gpurun_out/prof_k1 -f python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k1.log 2>&1; echo "ncu rc=$?" >> gpurun_out/b20.log
