"""ncu launch CSV of scripts/ncu_configs.py -> profiles/<tag>_ncu_configs.md (per config: K1's
DRAM bytes per launch vs the algorithmic bytes, dram__throughput, XU pipe, duration)."""
import csv
import json
import os
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, csvf, orderf = sys.argv[1], sys.argv[2], sys.argv[3]
order = json.loads([l for l in open(orderf) if l.startswith("[")][-1])
rows = [r for r in csv.reader(l for l in open(csvf) if not l.startswith("=="))]
h = rows[0]
idx = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
launches = {}
for r in rows[1:]:
    if len(r) < len(h) or "lopa_reduce" not in r[idx["Kernel Name"]]:
        continue
    lid = int(r[idx["ID"]])
    launches.setdefault(lid, {})[r[idx["Metric Name"]]] = (float(r[idx["Metric Value"]].replace(",", "")), r[idx["Metric Unit"]])
ids = sorted(launches)
out = [f"# {tag}: ncu metrics of K1 on every config (`scripts/ncu_configs.py`)\n",
       "One process, every BASELINE / sweep config; ncu `--clock-control none`, caches flushed before "
       "each replay (cold).  Per config: the second K1-alone launch (lopa_debug_reduce_only on the "
       "masked rows) and K1 inside the fused step.  DRAM MB = dram__bytes_read.sum + "
       "dram__bytes_write.sum; alg MB = 2 V x masked rows.\n",
       "| config | rows | alg MB | launch | us | DRAM MB | DRAM/alg | dram__throughput % | XU % active |",
       "|---|---|---|---|---|---|---|---|---|"]
k = 0
for o in order:
    kinds = o["launches"]
    if kinds[0] != "k1_initial_predict":   # order files written before the a0 launch was listed
        kinds = ["k1_initial_predict"] + kinds
    for pos, kind in enumerate(kinds):
        if k >= len(ids):
            break
        m = launches[ids[k]]
        k += 1
        if kind == "k1_initial_predict" or (kind == "k1_alone" and kinds[pos + 1] == "k1_alone"):
            continue  # report the second of the two K1-alone launches and the step's K1
        def g(name, scale=1.0):
            v = m.get(name)
            return v[0] * scale if v else float("nan")
        t = g("gpu__time_duration.sum")
        unit = m.get("gpu__time_duration.sum", (0, "ns"))[1]
        t_us = t / 1000.0 if unit == "nsecond" or unit == "ns" else t
        rd = m.get("dram__bytes_read.sum", (float("nan"), "byte"))
        wr = m.get("dram__bytes_write.sum", (float("nan"), "byte"))
        sc = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
        mb = rd[0] * sc.get(rd[1], 1e-6) + wr[0] * sc.get(wr[1], 1e-6)
        alg = o["alg_bytes"] / 1e6
        out.append(f"| {o['config']} | {o['masked_rows']} | {alg:.1f} | {kind} | {t_us:.2f} | {mb:.1f} | "
                   f"{mb / alg:.3f} | {g('dram__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                   f"{g('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'):.1f} |")
open(os.path.join(root, "profiles", f"{tag}_ncu_configs.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
