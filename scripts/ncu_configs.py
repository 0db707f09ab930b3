"""K1 on every BASELINE / sweep config in ONE process, for an ncu metrics pass (cold caches:
ncu flushes L2 before every replay).  For each config: the workload bench.py builds (branch
states after the initial forward of a fresh block, SYN-D2F verify logits), then K1 alone
(lopa_debug_reduce_only on the masked rows, 2 launches) and one fused lopa_step; the workload
builder's own initial-predict step comes first (4 K1 launches per config).  Prints the
config order so scripts/ncu_configs_md.py can label the launches.

    ncu --metrics ... -k regex:lopa_reduce --csv --log-file out.csv python scripts/ncu_configs.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_16229_b200 import lopa  # noqa: E402

CONFIGS = ["dream", "dream-k15", "diffucoder"] + [f"sweep-k{k}-w{w}" for k in (1, 3, 7, 15, 31)
                                                  for w in (16, 32, 64)] + \
          ["d2f-k7-w64", "d2f-k7-w128", "d2f-k3-w256", "d2f-k7-w256"]


def main():
    dev = torch.device("cuda:0")
    order = []
    for name in CONFIGS:
        c = bench.CONFIGS[name]
        st, tok, msk, nb, full, bufs, rows_total, _ = bench.build_workload(
            lopa, dev, c["V"], c["W"], c["k"], c["tau"], 1, 1)
        b = bufs[0]
        n_rows = b.shape[0] * c["W"]
        rmask = msk.reshape(-1).contiguous().clone()
        n = int(nb.item())
        rmask[n * c["W"]:] = 0
        ws = lopa.new_workspace(n_rows, c["V"], dev)
        status = lopa.new_status(dev)
        L, P = lopa.lib(), lopa._p
        s = lopa._stream(dev)
        for _ in range(2):
            lopa._check(L.lopa_debug_reduce_only(P(b), b.shape[-1], n_rows, c["V"], P(rmask), P(status),
                                                 P(ws), ws.numel(), s), "reduce_only")
        st.step(b, nb, tok, msk)
        torch.cuda.synchronize()
        order.append({"config": name, "masked_rows": rows_total, "alg_bytes": 2 * c["V"] * rows_total,
                      "launches": ["k1_initial_predict", "k1_alone", "k1_alone", "k1_in_step"]})
        del bufs, full
        torch.cuda.empty_cache()
    print(json.dumps(order))


if __name__ == "__main__":
    main()
