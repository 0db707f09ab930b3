"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

    python scripts/summarize_ncu.py <round-tag>
reads gpurun_out/launches.csv (gpu__time_duration per launch) and gpurun_out/prof_full.ncu-rep
(--set full of the step kernels), writes profiles/<tag>_launches.csv, profiles/<tag>_ncu_summary.md
and profiles/traffic.json (dram bytes per K1 launch, read by bench.py)."""
import csv, io, json, os, subprocess, sys
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out"); pr = os.path.join(root, "profiles")
os.makedirs(pr, exist_ok=True)
out = []
rows = list(csv.reader(open(os.path.join(go, "launches.csv"))))
hdr = None; launches = []
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); launches.append((d["ID"], d["Kernel Name"], float(d["Metric Value"])))
with open(os.path.join(pr, f"{tag}_launches.csv"), "w") as f:
    f.write("id,kernel,gpu__time_duration_ns\n")
    for i, k, v in launches: f.write(f'{i},"{k}",{v:.0f}\n')
# bench.py's timed regions each start behind a spin kernel (head_start): region 1 = the headline
# steps (K1 + K2 pairs), region 2 = the lopa_confidence chain, region 3 = K1 alone (roofline)
regions, cur = [], None
for _, k, v in launches:
    if "spin_kernel" in k:
        cur = []
        regions.append(cur)
    elif cur is not None:
        cur.append((k, v))
def _mean(xs):
    return sum(xs) / len(xs) if xs else float("nan")
steps = regions[0][:40] if regions else []
lk = [v for k, v in steps if "lopa_reduce" in k]
tk = [v for k, v in steps if "lopa_tail" in k]
k1_alone = [v for k, v in (regions[2] if len(regions) > 2 else []) if "lopa_reduce" in k][:20]
out.append(f"# ncu summary ({tag})\n")
out.append("Command: `python bench.py --steps 20 --warmup 3 --no-cpu-baseline` (Dream verify step, 241 masked rows x V=151936).\n")
out.append("## Launch list (gpu__time_duration.sum, --clock-control none; serialised, cold-cache)\n")
if lk and tk:
    mk, mt = sum(lk) / len(lk), sum(tk) / len(tk)
    out.append(f"- timed steps (first region): K1 lopa_reduce_kernel mean {mk/1000:.2f} us over {len(lk)} launches")
    out.append(f"- K2 lopa_tail_kernel: mean {mt/1000:.2f} us")
    out.append(f"- K1 share of the step (K1/(K1+K2)): {mk/(mk+mt):.1%} -- ncu serialises the two kernels, so"
               " K2's prologue and polling fold, which overlap K1 in the PDL chain, count in full here;"
               " in the bench's chain K1 alone is ~16.3 of ~20.3 us per step (~80 %)")
    if k1_alone:
        out.append(f"- K1 alone (the roofline region, lopa_debug_reduce_only): mean {_mean(k1_alone)/1000:.2f} us over {len(k1_alone)} launches")
    out.append("")
rep = os.path.join(go, "prof_full.ncu-rep")
traffic = None
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "dram__bytes_read.sum.pct_of_peak_sustained_elapsed",
            "sm__cycles_elapsed.avg.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct"]
    out.append("## --set full (one launch of each kernel)\n")
    out.append("| kernel | " + " | ".join(want) + " |")
    out.append("|---|" + "---|" * len(want))
    for r in rr[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "")[:28]
        vals = [d.get(w, "") for w in want]
        out.append(f"| {name} | " + " | ".join(vals) + " |")
        if "lopa_reduce" in name and traffic is None:
            try:
                sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                ur = sc.get(rr[1][h.index("dram__bytes_read.sum")], 1)
                uw = sc.get(rr[1][h.index("dram__bytes_write.sum")], 1)  # the two can differ
                traffic = float(d["dram__bytes_read.sum"]) * ur + float(d["dram__bytes_write.sum"]) * uw
            except Exception:
                traffic = None
    out.append("")
    out.append("Units row: " + ", ".join(f"{w}={rr[1][h.index(w)]}" for w in want if w in h))
rep2 = os.path.join(go, "prof_lmh.ncu-rep")
if os.path.exists(rep2):
    raw = subprocess.run(["ncu", "-i", rep2, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    want = ["gpu__time_duration.sum", "sm__cycles_active.avg", "dram__bytes_read.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread"]
    want = [w for w in want if w in h]
    out.append("\n## NEXT-4 fused LM head (`lopa_lmhead_kernel`, --set full, one launch; "
               "`scripts/lmhead_bench.py`, 241 rows x K=3584 x V=151936)\n")
    out.append("| kernel | " + " | ".join(want) + " |")
    out.append("|---|" + "---|" * len(want))
    for r in rr[2:]:
        d = dict(zip(h, r))
        out.append(f"| {d.get('Kernel Name', '')[:24]} | " + " | ".join(d.get(w, "") for w in want) + " |")
    out.append("")
    out.append("Units row: " + ", ".join(f"{w}={rr[1][h.index(w)]}" for w in want))
if traffic:
    json.dump({"bytes_per_launch": traffic, "kernel": "lopa_reduce_kernel", "source": f"profiles/{tag}_ncu_summary.md"},
              open(os.path.join(pr, "traffic.json"), "w"))
    out.append(f"\nK1 DRAM traffic per launch (read+write): {traffic/1e6:.2f} MB (algorithmic: 73.23 MB)")
open(os.path.join(pr, f"{tag}_ncu_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
