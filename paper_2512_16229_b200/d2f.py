"""D2F block pipeline around the fused LoPA step.

"LoPA integrates seamlessly with D2F by treating all active blocks as a single window for
branch exploration".  The window is the union of the active blocks (contiguous:
blocks activate and commit in index order), up to LOPA_MAX_WINDOW = 256 positions; every
iteration is ONE `lopa_step` launch over that window with per-position Eq. 1 thresholds
(tau_act on the newest active block, tau_conf on older ones — reading R25).  The block rules
are reading R26 (D2F's parameters from the Appendix table,
PAPER.md:519-536):

  (a) after each step, active blocks that the selected branch B* fills completely are
      committed, oldest first, stopping at the first block that is not full;
  (b) if no block is active the next one is activated; otherwise the next block is activated
      when the newest active block's fill ratio >= tau_add and the window stays <= max_window;
  the spawned branches carry over: committed columns are dropped, newly activated columns are
  appended fully masked; a step that completes its window (R21) is followed by the new
  window's initial predict (R17).

decode_d2f is host control flow (a few integers per iteration); all per-position work is in
liblopa's kernels.  D2FDeviceLoop runs the same rules on the device (lopa_d2f_*: no host read,
CUDA-graph capturable).  This module never imports the oracle.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import lopa

INACTIVE, ACTIVE, COMMITTED = 0, 1, 2


@dataclass
class BlockConfig:
    """D2F parameters (Appendix table)."""
    block_size: int = 32
    tau_add: float = 0.1
    tau_act: float = 0.95
    tau_conf: float = 0.90
    max_window: int = lopa.MAX_WINDOW


@dataclass
class D2FResult:
    tokens: torch.Tensor                      # int32 [gen_len] on the device
    forwards: int = 0
    windows: list = field(default_factory=list)
    winners: list = field(default_factory=list)
    branch_counts: list = field(default_factory=list)
    commits: list = field(default_factory=list)

    @property
    def tpf(self) -> float:
        return self.tokens.numel() / self.forwards if self.forwards else 0.0


class BlockPipeline:
    """Block status bookkeeping (R26).  Status per block: INACTIVE -> ACTIVE -> COMMITTED."""

    def __init__(self, n_blocks: int, cfg: BlockConfig):
        if cfg.block_size < 1 or cfg.block_size > cfg.max_window or cfg.max_window > lopa.MAX_WINDOW:
            raise lopa.LopaError("block_size must be in [1, max_window] and max_window <= 256")
        self.cfg = cfg
        self.status = [INACTIVE] * n_blocks
        self.status[0] = ACTIVE

    def active(self):
        return [b for b, s in enumerate(self.status) if s == ACTIVE]

    def window(self):
        """(first position, width) of the active window."""
        a = self.active()
        B = self.cfg.block_size
        return (a[0] * B, len(a) * B) if a else (0, 0)

    def thresholds(self):
        """Per-position Eq. 1 thresholds over the window (float32 list)."""
        a = self.active()
        B = self.cfg.block_size
        out = []
        for b in a:
            out += [self.cfg.tau_act if b == a[-1] else self.cfg.tau_conf] * B
        return out

    def update(self, masked_per_block):
        """Apply rules (a), (b).  masked_per_block[b] = masked count of B* in block b (active
        blocks only).  Returns the list of newly committed blocks."""
        st, B = self.status, self.cfg.block_size
        committed = []
        for b in range(len(st)):
            if st[b] == COMMITTED:
                continue
            if st[b] == ACTIVE and masked_per_block[b] == 0:
                st[b] = COMMITTED
                committed.append(b)
                continue
            break
        a = self.active()
        nxt = next((b for b, s in enumerate(st) if s == INACTIVE), None)
        if nxt is not None:
            if not a:
                st[nxt] = ACTIVE
            elif ((B - masked_per_block[a[-1]]) / B >= float(self.cfg.tau_add)
                  and (len(a) + 1) * B <= self.cfg.max_window):
                st[nxt] = ACTIVE
        return committed

    def done(self):
        return all(s == COMMITTED for s in self.status)


def decode_d2f(forward_block, gen_len: int, k: int, cfg: BlockConfig, vocab: int, device,
               tokens0: torch.Tensor | None = None, max_forwards: int | None = None,
               metric: int = lopa.METRIC_MEAN, metric_param: float = 0.0,
               on_step=None) -> D2FResult:
    """LoPA decoding of a ``gen_len``-token region through the D2F block pipeline.

    ``forward_block(b, tokens[n][B], mask[n][B]) -> bf16 [n][B][ld]`` is the model stand-in for
    the positions of block b under n branch states (device tensors); a window forward is one
    call per active block, placed side by side in the window's logits buffer.
    ``on_step(iteration, logits, branch_tokens, branch_mask, n, thresholds, outputs)`` (optional,
    for tests and tracing) sees every step's inputs and outputs right after the step."""
    B = cfg.block_size
    if gen_len % B:
        raise lopa.LopaError("gen_len must be a multiple of block_size")
    dev = torch.device(device)
    n_blk = gen_len // B
    pipe = BlockPipeline(n_blk, cfg)
    tok = torch.zeros(gen_len, dtype=torch.int32, device=dev) if tokens0 is None else tokens0.clone()
    msk = torch.ones(gen_len, dtype=torch.uint8, device=dev)
    max_br = k + 1
    ld = ((vocab + 7) // 8) * 8
    steppers = {}
    res = D2FResult(tokens=tok)
    p0, W = pipe.window()
    br_tok = torch.zeros((max_br, W), dtype=torch.int32, device=dev)
    br_msk = torch.zeros((max_br, W), dtype=torch.uint8, device=dev)
    br_tok[0], br_msk[0] = tok[p0:p0 + W], msk[p0:p0 + W]
    n = 1
    nb_dev = torch.ones(1, dtype=torch.int32, device=dev)
    while True:
        if W not in steppers:
            tp = torch.empty(W, dtype=torch.float32, device=dev)
            steppers[W] = (lopa.Stepper(vocab, W, max_br, k, cfg.tau_act, dev, metric=metric,
                                        metric_param=metric_param, tau_pos=tp),
                           torch.empty((max_br, W, ld), dtype=torch.bfloat16, device=dev))
        st, logits = steppers[W]
        st.tau_pos.copy_(torch.tensor(pipe.thresholds(), dtype=torch.float32))
        for c, b in enumerate(pipe.active()):
            logits[:n, c * B:(c + 1) * B] = forward_block(b, br_tok[:n, c * B:(c + 1) * B].contiguous(),
                                                           br_msk[:n, c * B:(c + 1) * B].contiguous())
        nb_dev.fill_(n)
        out = st.step(logits, nb_dev, br_tok, br_msk)
        if on_step is not None:
            on_step(res.forwards, logits, br_tok, br_msk, n, pipe.thresholds(), out)
        res.forwards += 1
        res.windows.append((p0, W))
        res.branch_counts.append(n)
        w, n_next = (int(x) for x in torch.stack([out.winner[0], out.n_next[0]]).cpu())
        res.winners.append(w)
        # x_{t+1} = B* on the window
        tok[p0:p0 + W] = br_tok[w]
        msk[p0:p0 + W] = br_msk[w]
        masked = msk.view(n_blk, B).sum(dim=1).cpu().tolist()
        res.commits += pipe.update(masked)
        if pipe.done() or (max_forwards is not None and res.forwards >= max_forwards):
            break
        q0, WN = pipe.window()
        nt = torch.zeros((max_br, WN), dtype=torch.int32, device=dev)
        nm = torch.zeros((max_br, WN), dtype=torch.uint8, device=dev)
        if n_next == 0:
            # the window is complete (R21): the new window starts with its initial predict
            nt[0], nm[0] = tok[q0:q0 + WN], msk[q0:q0 + WN]
            n = 1
        else:
            # carry the spawned branches over: keep the surviving columns, append new blocks
            lo, hi = max(p0, q0), min(p0 + W, q0 + WN)
            nt[:n_next] = tok[q0:q0 + WN]
            nm[:n_next] = msk[q0:q0 + WN]
            if hi > lo:
                nt[:n_next, lo - q0:hi - q0] = out.next_tokens[:n_next, lo - p0:hi - p0]
                nm[:n_next, lo - q0:hi - q0] = out.next_mask[:n_next, lo - p0:hi - p0]
            n = n_next
        p0, W, br_tok, br_msk = q0, WN, nt, nm
    res.tokens = tok
    return res


class D2FDesc(ctypes.Structure):
    """Mirror of lopa_d2f_t (include/liblopa.h)."""
    _fields_ = [
        ("gen_len", ctypes.c_int32), ("block_size", ctypes.c_int32), ("k", ctypes.c_int32),
        ("max_window", ctypes.c_int32), ("tau_add", ctypes.c_double), ("tau_act", ctypes.c_float),
        ("tau_conf", ctypes.c_float), ("trace_cap", ctypes.c_int32),
        ("region_tokens", ctypes.c_void_p), ("region_mask", ctypes.c_void_p),
        ("block_status", ctypes.c_void_p), ("sched", ctypes.c_void_p), ("tau_pos", ctypes.c_void_p),
        ("branch_tokens", ctypes.c_void_p), ("branch_mask", ctypes.c_void_p),
        ("commit_order", ctypes.c_void_p), ("trace", ctypes.c_void_p),
    ]


class D2FDeviceLoop:
    """The D2F decode with the block scheduler on the device (lopa_d2f_*; rules R26 as in
    BlockPipeline): one iteration = the harness forward of the device window
    (lopa_d2f_syn_forward, the model stand-in) + one lopa_step whose window, branch count and
    thresholds are read on the device + lopa_d2f_update.  No host read anywhere, so `iters`
    iterations can be issued blindly (iterations after the last commit are no-ops) or captured
    in one CUDA graph (capture()).  trace() reads the windows, branch counts, winners and commit
    order back for comparison with decode_d2f / the oracle."""

    def __init__(self, gen_len: int, k: int, cfg: BlockConfig, vocab: int, device, seed: int,
                 extras: int = 0, tokens0: torch.Tensor | None = None, trace_cap: int = 1024,
                 metric: int = lopa.METRIC_MEAN, metric_param: float = 0.0):
        B, mw = cfg.block_size, cfg.max_window
        if gen_len % B or B > mw or mw > lopa.MAX_WINDOW:
            raise lopa.LopaError("gen_len % block_size == 0 and block_size <= max_window <= 256")
        d = torch.device(device)
        self.dev, self.seed, self.extras, self.vocab, self.k, self.cfg = d, seed, extras, vocab, k, cfg
        self.gen_len, self.nblk, self.max_br = gen_len, gen_len // B, k + 1
        self.tokens0 = (torch.zeros(gen_len, dtype=torch.int32, device=d) if tokens0 is None
                        else tokens0.to(torch.int32).clone())
        self.region_tokens = self.tokens0.clone()
        self.region_mask = torch.ones(gen_len, dtype=torch.uint8, device=d)
        self.block_status = torch.zeros(self.nblk, dtype=torch.int32, device=d)
        self.sched = torch.zeros(8, dtype=torch.int32, device=d)
        self.tau_pos = torch.empty(mw, dtype=torch.float32, device=d)
        self.branch_tokens = torch.zeros((self.max_br, mw), dtype=torch.int32, device=d)
        self.branch_mask = torch.zeros((self.max_br, mw), dtype=torch.uint8, device=d)
        self.commit_order = torch.full((self.nblk,), -1, dtype=torch.int32, device=d)
        self.trace_buf = torch.zeros((trace_cap, 4), dtype=torch.int32, device=d)
        self.st = lopa.Stepper(vocab, mw, self.max_br, k, cfg.tau_act, d, metric=metric,
                               metric_param=metric_param, tau_pos=self.tau_pos)
        self.logits = torch.zeros((self.max_br, mw, self.st.ld), dtype=torch.bfloat16, device=d)
        self.desc = D2FDesc(gen_len, B, k, mw, float(cfg.tau_add), float(cfg.tau_act),
                            float(cfg.tau_conf), trace_cap, self.region_tokens.data_ptr(),
                            self.region_mask.data_ptr(), self.block_status.data_ptr(),
                            self.sched.data_ptr(), self.tau_pos.data_ptr(),
                            self.branch_tokens.data_ptr(), self.branch_mask.data_ptr(),
                            self.commit_order.data_ptr(), self.trace_buf.data_ptr())
        a = self.st.args(self.logits, self.sched[2:3], self.branch_tokens, self.branch_mask)
        a.window_dev = self.sched.data_ptr() + 4        # &sched[1]
        self.args = a
        self.graph = None

    def reset(self):
        """Back to the initial state (tokens0, region masked, block 0 active)."""
        self.region_tokens.copy_(self.tokens0)
        lopa._check(lopa.lib().lopa_d2f_init(ctypes.byref(self.desc), lopa._stream(self.dev)),
                    "lopa_d2f_init")

    def iteration(self):
        L, s = lopa.lib(), lopa._stream(self.dev)
        lopa._check(L.lopa_d2f_syn_forward(self.seed & ((1 << 64) - 1), self.vocab, self.st.ld,
                                           self.extras, ctypes.byref(self.desc),
                                           lopa._p(self.logits), s), "lopa_d2f_syn_forward")
        lopa._check(L.lopa_step(ctypes.byref(self.args), s), "lopa_step")
        o = self.st.out
        lopa._check(L.lopa_d2f_update(ctypes.byref(self.desc), lopa._p(o.winner), lopa._p(o.n_next),
                                      lopa._p(o.next_tokens), lopa._p(o.next_mask), s),
                    "lopa_d2f_update")

    def run(self, iters: int):
        for _ in range(iters):
            self.iteration()

    def capture(self, iters: int):
        """`iters` iterations in one CUDA graph (reset() not included; replay() after reset())."""
        self.reset()
        self.iteration()                      # warm-up outside the capture (attributes, modules)
        torch.cuda.synchronize(self.dev)
        self.reset()
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(iters)
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()

    def capture_while(self, max_iters: int = 1 << 16):
        """The whole decode as ONE device-terminated CUDA graph (lopa.WhileGraph): iterations
        repeat on the device until every block is committed (sched[3] != 0) -- no iteration
        count needed.  launch_while() after reset()."""
        self.reset()
        self.iteration()                      # warm-up outside the capture
        torch.cuda.synchronize(self.dev)
        self.reset()
        torch.cuda.synchronize(self.dev)
        self.while_graph = lopa.WhileGraph(self.iteration, self.sched[3:4], until_zero=False,
                                           max_iters=max_iters)
        return self.while_graph

    def launch_while(self):
        self.while_graph.launch()

    def done(self) -> bool:
        return bool(int(self.sched[3].item()))

    def trace(self) -> D2FResult:
        s = self.sched.cpu().tolist()
        f = s[4]
        tr = self.trace_buf[:min(f, self.trace_buf.shape[0])].cpu().tolist()
        res = D2FResult(tokens=self.region_tokens.clone(), forwards=f)
        res.windows = [(t[0], t[1]) for t in tr]
        res.branch_counts = [t[2] for t in tr]
        res.winners = [t[3] for t in tr]
        res.commits = [b for b in self.commit_order.cpu().tolist() if b >= 0]
        return res
