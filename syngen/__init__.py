"""SYN-D2F: the seeded, integer-exact synthetic-logits generator (stand-in for the dLLM forward).

This module is the ONE piece shared by the oracle side (tests, `oracle/`) and the CUDA
side (bench, GPU tests): it produces inputs only and holds none of LoPA's arithmetic
(no softmax, no confidence, no Eq. 1 / Eq. 2, no top-k).  The CUDA kernel
`lopa_syn_generate` (paper_2512_16229_b200/csrc/lopa_syn.cu) implements the same
counter-based definition independently; `tests/test_gpu_parity.py::test_syn_generate_matches_numpy` checks the two
agree bit for bit.

Definition ("SYN-D2F"; DESIGN.md §3 "Input recipe"):

* ``mix64``  — the splitmix64 finaliser, uint64 wrap-around.
* ``H(a0, a1, ...)``: ``h = mix64(seed); for a in args: h = mix64(h ^ a)``.
* ``state_hash(S)`` = XOR over filled positions p of the block of ``H(2, blk, p, tok_p)``.
* ``row_key(i)``   = ``H(1, blk, i, state_hash)``.
* noise: for ``v = 8q + r``: ``l_v = (byte_r(mix64(row_key ^ q)) - 128) / 64`` in [-2, 2).
* spike token ``t_i = H(3, blk, i) mod V``.
* ``cV8 = round(8 ln(1.8 (V-1)))`` (centre, in eighths; 100 at V=151936, 38 at V=64).
* ``h0_8 = cV8 - 28 + (H(4, blk, i) mod 49)``; ``jit8 = (H(row_key, 5) mod 9) - 4``;
  ``nb_i`` = number of filled positions at distance 1..3 from i (neighbour coupling:
  filling order changes later confidences, the paper's TFO sensitivity).
* spike value ``l_{t_i} = min(h0_8 + 16 nb_i + jit8, cV8 + 60) / 8``.
* toy extras (flag ``EXTRAS_TIES_FLAT``): ``sel = H(row_key, 6) mod 16``; sel == 0 -> the
  whole row is 0.0 (flat row); sel == 1 -> a second token ``t2 = H(7, blk, i) mod V``
  gets the same spike value (argmax tie, lowest id wins).

Every value is a multiple of 1/64 with < 256 units, hence exactly representable in bf16;
the generator returns raw bf16 bit patterns (uint16).
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
EXTRAS_NONE = 0
EXTRAS_TIES_FLAT = 1

_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def mix64(z: int) -> int:
    """splitmix64 finaliser on a Python int (uint64 wrap-around)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def mix64_np(z: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 arrays."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _C1
        z ^= z >> np.uint64(27)
        z *= _C2
        z ^= z >> np.uint64(31)
    return z


def H(seed: int, *args: int) -> int:
    h = mix64(seed)
    for a in args:
        h = mix64(h ^ (a & MASK64))
    return h


def cv8(vocab: int) -> int:
    """Centre of the spike heights in eighths: round(8 ln(1.8 (V-1)))."""
    if vocab < 2:
        return 0
    return int(round(8.0 * math.log(1.8 * (vocab - 1))))


def state_hash(seed: int, blk: int, tokens, mask) -> int:
    h = 0
    for p in range(len(mask)):
        if not mask[p]:
            h ^= H(seed, 2, blk, p, int(tokens[p]))
    return h


def neighbour_count(mask, i: int) -> int:
    W = len(mask)
    n = 0
    for d in (1, 2, 3):
        for q in (i - d, i + d):
            if 0 <= q < W and not mask[q]:
                n += 1
    return n


def row_params(seed: int, blk: int, i: int, vocab: int, tokens, mask, extras: int = EXTRAS_NONE):
    """Per-row parameters: (row_key, spike_tok, spike8, tie_tok or -1, flat)."""
    sh = state_hash(seed, blk, tokens, mask)
    rk = H(seed, 1, blk, i, sh)
    t = H(seed, 3, blk, i) % vocab
    c8 = cv8(vocab)
    h0 = c8 - 28 + (H(seed, 4, blk, i) % 49)
    jit = (H(seed, rk, 5) % 9) - 4
    nb = neighbour_count(mask, i)
    s8 = min(h0 + 16 * nb + jit, c8 + 60)
    tie, flat = -1, False
    if extras & EXTRAS_TIES_FLAT:
        sel = H(seed, rk, 6) % 16
        if sel == 0:
            flat = True
        elif sel == 1:
            t2 = H(seed, 7, blk, i) % vocab
            if t2 != t:
                tie = t2
    return rk, t, s8, tie, flat


def _f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Exact conversion for values that are representable in bf16 (checked)."""
    b = x.astype(np.float32).view(np.uint32)
    assert np.all((b & np.uint32(0xFFFF)) == 0), "value not bf16-exact"
    return (b >> np.uint32(16)).astype(np.uint16)


def gen_row(seed: int, blk: int, i: int, vocab: int, tokens, mask, extras: int = EXTRAS_NONE,
            ld: int | None = None) -> np.ndarray:
    """bf16 bit patterns (uint16[ld]) of one logits row; entries >= vocab are 0."""
    ld = vocab if ld is None else ld
    rk, t, s8, tie, flat = row_params(seed, blk, i, vocab, tokens, mask, extras)
    nq = (vocab + 7) // 8
    out = np.zeros(ld, dtype=np.uint16)
    if flat:
        return out  # bf16 +0.0 everywhere in [0, vocab)
    q = np.arange(nq, dtype=np.uint64)
    h = mix64_np(np.uint64(rk) ^ q)
    shifts = (np.arange(8, dtype=np.uint64) * np.uint64(8))[None, :]
    byts = ((h[:, None] >> shifts) & np.uint64(0xFF)).astype(np.int32).reshape(-1)[:vocab]
    vals = (byts - 128).astype(np.float32) / np.float32(64.0)
    vals[t] = np.float32(s8) / np.float32(8.0)
    if tie >= 0:
        vals[tie] = np.float32(s8) / np.float32(8.0)
    out[:vocab] = _f32_to_bf16_bits(vals)
    return out


def gen_logits(seed: int, blk: int, vocab: int, branch_tokens, branch_mask, n_branches: int | None = None,
               extras: int = EXTRAS_NONE, ld: int | None = None) -> np.ndarray:
    """Logits (bf16 bits, uint16[n_br][W][ld]) for a batch of branch states (the 'forward')."""
    branch_tokens = np.asarray(branch_tokens)
    branch_mask = np.asarray(branch_mask)
    nb, W = branch_mask.shape
    n_branches = nb if n_branches is None else n_branches
    ld = vocab if ld is None else ld
    out = np.zeros((n_branches, W, ld), dtype=np.uint16)
    for j in range(n_branches):
        for i in range(W):
            out[j, i] = gen_row(seed, blk, i, vocab, branch_tokens[j], branch_mask[j], extras, ld)
    return out


def bf16_bits_to_f32(u16: np.ndarray) -> np.ndarray:
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def fresh_block(window: int):
    """A fully masked block: tokens all 0, mask all 1."""
    return np.zeros(window, dtype=np.int32), np.ones(window, dtype=np.uint8)


# ----------------------------------------------------------------------------- LM-head inputs
def _f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bits, round to nearest even (inputs only; finite values)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def lmhead_inputs(seed: int, rows: int, hidden_dim: int, vocab: int, sigma: float = 1.5,
                  spike_lo: float = 4.0, spike_hi: float = 16.0, chunk: int = 8192):
    """Seeded SYN-LMH inputs: weight W [V][K] ~ N(0, 1/K) (rows of norm ~1, the
    scale of a trained output projection), hidden rows h_r = sigma·z + beta_r·W[t_r]/|W[t_r]|^2
    with a planted target token t_r and logit margin beta_r ~ U[spike_lo, spike_hi], so the
    logit of t_r sits ~beta_r above a N(0, sigma^2) background: conf spans ~1e-4 .. 0.99 at
    V = 151936.  Returns (hidden bf16 bits [rows][K], weight bf16 bits [V][K], targets)."""
    rng = np.random.default_rng(seed)
    W = np.empty((vocab, hidden_dim), dtype=np.uint16)
    for v0 in range(0, vocab, chunk):
        n = min(chunk, vocab - v0)
        W[v0:v0 + n] = _f32_to_bf16_rne(rng.standard_normal((n, hidden_dim), dtype=np.float32)
                                        / np.float32(math.sqrt(hidden_dim)))
    t = rng.integers(0, vocab, size=rows)
    beta = rng.uniform(spike_lo, spike_hi, size=rows)
    Wt = bf16_bits_to_f32(W[t]).astype(np.float64)
    z = rng.standard_normal((rows, hidden_dim))
    h = sigma * z + (beta / (Wt * Wt).sum(axis=1))[:, None] * Wt
    return _f32_to_bf16_rne(h.astype(np.float32)), W, t
