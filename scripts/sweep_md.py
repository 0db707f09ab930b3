"""profiles/<tag>_sweep.jsonl (scripts/sweep.sh output) -> profiles/<tag>_sweep.md."""
import json, os, sys
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(root, "profiles", f"{tag}_sweep.jsonl")
lines = [json.loads(l) for l in open(src)]
peak = lines[0]["roofline"]["peak"] if lines else float("nan")
out = [f"# {tag} sweep (bench.py --config ..., --steps 300, 1 x B200)\n",
       "K1 GB/s = algorithmic bytes (2 V per masked row) / K1's average launch duration (CUDA events "
       "around back-to-back K1 launches, `roofline.kernel_timing`); frac = / "
       f"{peak:.1f} GB/s (MEASURED_PEAKS.json copy peak, as read by bench.py in this run); "
       "conf-call = the same rows through `lopa_confidence` (K1 + fold kernel); "
       "isolated p50 = median of individually timed steps.\n",
       "| config | masked rows | us/step | steps/s | isolated p50 us | K1 us | K1 GB/s | frac | conf-call us |",
       "|---|---|---|---|---|---|---|---|---|"]
for d in lines:
    r = d["roofline"]
    iso = d.get("step_time_distribution", {}).get("isolated_step_us", {}).get("p50", float("nan"))
    out.append(f"| {d['config']['workload']} | {d['config']['masked_rows']} | {d['ms_per_step'] * 1e3:.1f} | "
               f"{d['value']:.0f} | {iso:.1f} | {r['kernel_ms_mean'] * 1e3:.1f} | {r['achieved']:.0f} | {r['frac']:.3f} | "
               f"{r.get('conf_call_ms', float('nan')) * 1e3:.1f} |")
open(os.path.join(root, "profiles", f"{tag}_sweep.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
