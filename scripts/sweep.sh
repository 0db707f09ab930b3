# bench over BASELINE configs (not the headline): JSON lines to gpurun_out/sweep.jsonl
mkdir -p gpurun_out; : > gpurun_out/sweep.jsonl
for c in dream dream-k15 diffucoder sweep-k1-w16 sweep-k3-w16 sweep-k7-w32 sweep-k15-w32 sweep-k15-w64 sweep-k31-w32 sweep-k31-w64; do
  timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu-baseline --config $c 2>/dev/null | grep '^{' >> gpurun_out/sweep.jsonl
done
