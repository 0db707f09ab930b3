# bench over BASELINE configs (not the headline): JSON lines to gpurun_out/sweep.jsonl
mkdir -p gpurun_out; : > gpurun_out/sweep.jsonl
for c in dream dream-k15 diffucoder sweep-k1-w16 sweep-k1-w32 sweep-k1-w64 sweep-k3-w16 sweep-k3-w32 sweep-k3-w64 sweep-k7-w16 sweep-k7-w32 sweep-k7-w64 sweep-k15-w16 sweep-k15-w32 sweep-k15-w64 sweep-k31-w16 sweep-k31-w32 sweep-k31-w64 d2f-k7-w64 d2f-k7-w128 d2f-k3-w256 d2f-k7-w256; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --config $c 2>/dev/null | grep '^{' >> gpurun_out/sweep.jsonl
done
