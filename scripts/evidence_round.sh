# round-end evidence in one gpurun call: profile_round.sh + the sweep + D2F / LM-head config lines
bash scripts/profile_round.sh
bash scripts/sweep.sh
: > gpurun_out/extra.jsonl
for c in lmhead-gsm8k d2f-k7-w128 d2f-k7-w256; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --config $c 2>/dev/null | grep '^{' >> gpurun_out/extra.jsonl
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
