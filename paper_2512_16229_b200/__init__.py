"""paper_2512_16229_b200 — the LoPA verify step (arXiv 2512.16229) on B200 (sm_100a).

The product is liblopa.so (C ABI, include/liblopa.h); `lopa` is its thin ctypes binding.
"""
from . import lopa  # noqa: F401
from .lopa import (BranchParallel, LopaError, Stepper, anchor_fill, bp_shard, confidence,  # noqa: F401
                   spawn_branches, syn_generate, verify_select)

__all__ = ["lopa", "Stepper", "BranchParallel", "LopaError", "confidence", "anchor_fill",
           "spawn_branches", "verify_select", "syn_generate", "bp_shard"]
