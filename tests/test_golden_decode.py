"""The stored oracle decodes of BASELINE configs[2] / configs[3] (tests/golden/
oracle_decode_configs.json, written by scripts/make_golden_decode.py from oracle/ only) still
equal the oracle: block 0 of each is recomputed here (the GPU BP tests compare against all
blocks)."""
import json
import os

import numpy as np
import pytest

import syngen
from oracle import lopa_oracle as O

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_decode_configs.json")))


@pytest.mark.parametrize("case", sorted(GOLDEN))
def test_golden_block0_matches_oracle(case):
    c = GOLDEN[case]
    fwd = lambda t, m: syngen.gen_logits(c["seed"], 0, c["V"], t, m)
    tok0, msk0 = syngen.fresh_block(c["W"])
    tr = O.decode_block(fwd, tok0, msk0, c["k"], c["tau"])
    assert tr.forwards == c["forwards_per_block"][0]
    assert [int(x) for x in tr.tokens] == c["tokens"][: c["W"]]
    assert [int(w) for w in tr.winners] == c["winners_per_block"][0]
    assert len(c["tokens"]) == c["W"] * c["blocks"]
    # every block decodes to a complete block: W tokens, each a valid vocabulary id
    assert all(0 <= t < c["V"] for t in c["tokens"])
