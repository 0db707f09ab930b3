"""Write tests/golden/oracle_decode_configs.json: the CPU oracle's Alg. 1 decode (P:154-180,
oracle.lopa_oracle.decode_block) of BASELINE configs[2] and configs[3] on SYN-D2F logits.
Calls only oracle/ and syngen/ (inputs); never the CUDA path.

    python scripts/make_golden_decode.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import syngen  # noqa: E402
from oracle import lopa_oracle as O  # noqa: E402

CASES = {
    # configs[2]: D2F-Dream shape full decode loop, 256-token generation (8 sequential blocks of
    # 32, R22), k = 15 (16 branches: 2 per rank at 8 GPUs), tau = 0.9
    "dream_k15_256": dict(V=151936, W=32, k=15, tau=0.9, seed=1, blocks=8,
                          cite="BASELINE.json configs[2]; PAPER.md:154-180 (Alg. 1), :293 (BP)"),
    # configs[3]: D2F-DiffuCoder shape, k = 10, tau = 0.95, multi-block decode (4 blocks)
    "diffucoder_k10_128": dict(V=151936, W=32, k=10, tau=0.95, seed=3, blocks=4,
                               cite="BASELINE.json configs[3]; PAPER.md:154-180, :535 (tau 0.95)"),
}


def decode(c, blocks=None):
    toks, fws, wins = [], [], []
    for blk in range(c["blocks"] if blocks is None else blocks):
        fwd = lambda t, m, blk=blk: syngen.gen_logits(c["seed"], blk, c["V"], t, m)
        tok0, msk0 = syngen.fresh_block(c["W"])
        tr = O.decode_block(fwd, tok0, msk0, c["k"], c["tau"])
        toks.extend(int(x) for x in tr.tokens)
        fws.append(int(tr.forwards))
        wins.append([int(w) for w in tr.winners])
    return toks, fws, wins


def main():
    out = {}
    for name, c in CASES.items():
        t0 = time.time()
        toks, fws, wins = decode(c)
        out[name] = dict(c, tokens=toks, forwards_per_block=fws, winners_per_block=wins,
                         generator="syngen.gen_logits (SYN-D2F), block b of the generation = blk b")
        print(name, "forwards", fws, "TPF", len(toks) / sum(fws), f"{time.time() - t0:.1f} s")
    path = os.path.join(ROOT, "tests", "golden", "oracle_decode_configs.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
