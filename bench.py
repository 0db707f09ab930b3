#!/usr/bin/env python
"""Benchmark of the LoPA verify step (liblopa on B200) — BASELINE.json metric
"LoPA verify-steps/s and logits HBM GB/s (V=151936, k+1 branches) at 1/2/4/8 B200".

A "step" is one pass of the whole hot path (+ a5 at N > 1) over one batch of
synthetic verify logits: reduce every masked (branch, position) row, score and select, anchor,
spawn.  Workload (BASELINE configs[1], D2F-Dream shape): V = 151936, W = 32, k = 7 (8 branches),
tau = 0.9; branch states = the spawn of a fresh fully-masked block after its initial forward;
logits = SYN-D2F.  Inputs are larger than L2: the timed steps rotate over 8
logits buffers (622 MB >= 4 x 126 MB L2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lopa|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (branch-parallel, one rank per GPU)

--impl reference times the CPU oracle (oracle/, NumPy fp64) as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "LoPA verify-steps/s and logits HBM GB/s (V=151936,k+1 branches) at 1/2/4/8 B200"
UNIT = "verify-steps/s"
CFG = dict(V=151936, W=32, k=7, tau=0.9, seed=1, n_buf=8)
# other BASELINE.json configs, selectable with --config (the headline is configs[1] = "dream")
CONFIGS = {
    "dream": dict(V=151936, W=32, k=7, tau=0.9, name="D2F-Dream verify step V=151936 W=32 k=7 tau=0.9 (configs[1])"),
    "dream-k15": dict(V=151936, W=32, k=15, tau=0.9, name="D2F-Dream verify step V=151936 W=32 k=15 tau=0.9 (configs[2] shape)"),
    "diffucoder": dict(V=151936, W=32, k=10, tau=0.95, name="D2F-DiffuCoder verify step V=151936 W=32 k=10 tau=0.95 (configs[3] shape)"),
}
# BASELINE configs[2] / configs[3]: whole Alg. 1 decode loops, branch-parallel at N > 1
CONFIGS["dream-loop"] = dict(V=151936, W=32, k=15, tau=0.9, loop_blocks=8, seed=1,
                             name="D2F-Dream full decode loop: 256-token generation (8 blocks of 32), k=15, tau=0.9, branch-parallel (configs[2])")
CONFIGS["diffucoder-loop"] = dict(V=151936, W=32, k=10, tau=0.95, loop_blocks=4, seed=3,
                                  name="D2F-DiffuCoder multi-block decode: 4 blocks of 32, k=10, tau=0.95, branch-parallel (configs[3])")
# NEXT-1: the D2F block pipeline over a 256-token generation (configs[2] shape, k = 15, D2F GSM8K
# parameters block 32 / tau_add 0.1 / tau_act 0.95 / tau_conf 0.90): the device
# scheduler's captured loop beside the host-driven loop
CONFIGS["d2f-graph"] = dict(V=151936, W=256, k=15, tau=0.95, d2f_len=256, seed=11,
                            name="D2F multi-block decode, 256 tokens, k=15, block 32, tau_add 0.1, tau_act 0.95, tau_conf 0.90: device-resident scheduler in one CUDA graph")
# NEXT-4: the same step from the verify forward's hidden states (fused LM-head a1), Dream-7B
# output projection K = 3584 (Qwen2.5-7B hidden size; outside the paper), one GPU
CONFIGS["lmhead-dream"] = dict(V=151936, W=32, k=7, tau=0.9, K=3584,
                               name="D2F-Dream verify step from hidden states: fused LM head K=3584 V=151936 W=32 k=7 tau=0.9")
CONFIGS["lmhead-gsm8k"] = dict(V=151936, W=32, k=14, tau=0.9, K=3584,
                               name="D2F-Dream GSM8K (k=14, PAPER.md:528) verify step from hidden states: fused LM head, 480 rows in two 256-row passes")
# NEXT-1: D2F multi-block windows (2, 4 and 8 active blocks of 32)
for _k, _w in ((7, 64), (7, 128), (3, 256), (7, 256)):
    CONFIGS[f"d2f-k{_k}-w{_w}"] = dict(V=151936, W=_w, k=_k, tau=0.9,
                                       name=f"D2F multi-block window V=151936 W={_w} k={_k} tau=0.9")
for _k in (1, 3, 7, 15, 31):
    for _w in (16, 32, 64):
        CONFIGS[f"sweep-k{_k}-w{_w}"] = dict(V=151936, W=_w, k=_k, tau=0.9,
                                             name=f"sweep V=151936 W={_w} k={_k} tau=0.9 (configs[4])")


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.idx, self.period, self.samples, self.reasons = device_index, period_s, [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workload
def make_branch_parallel(lopa, st, rank, world, dist, dev):
    """The branch-parallel driver of this rank: the record exchange over peer memory
    (lopa_bp_step_p2p: K2 stores its record into every peer over NVLink and finishes the step
    itself) by default at N > 1; LOPA_BP_P2P=0 forces the NCCL all-gather (the default at N = 1,
    where there is no peer).  If the peer-memory setup fails on any rank, every rank uses NCCL.
    Returns (driver, note or None)."""
    want_p2p = os.environ.get("LOPA_BP_P2P", "1" if world > 1 else "0") == "1"
    bp, note, ok = None, None, False
    if want_p2p:
        try:
            bp = lopa.BranchParallel(st, rank, world, p2p=True)
            ok = True
        except Exception as e:  # noqa: BLE001 - reported in the bench line
            note = f"peer-memory setup failed ({type(e).__name__}: {e}); NCCL all-gather used"
    if dist is not None and want_p2p:
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if ok and int(flag.item()) == 0:
            bp.close()
            ok = False
            note = note or "peer-memory setup failed on another rank; NCCL all-gather used"
    if not ok:
        bp = lopa.BranchParallel(st, rank, world, p2p=False)
    if dist is not None:
        dist.barrier()  # the first exchange starts together on every rank
    return bp, note


def build_workload(lopa, dev, V, W, k, tau, seed, n_buf, lo=0, hi=None, b_loc=None):
    """Branch states after the initial forward (a0) of a fresh block, and n_buf copies of their
    verify logits (branches [lo, hi) only, padded to b_loc rows when sharded)."""
    st = lopa.Stepper(V, W, k + 1, k, tau, dev)
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=dev)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=dev)
    msk[0] = 1
    nb = torch.ones(1, dtype=torch.int32, device=dev)
    logits0 = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=dev)
    lopa.syn_generate(seed, 0, V, tok, msk, n_branches=1, out=logits0[:1])
    out = st.step(logits0, nb, tok, msk)
    torch.cuda.synchronize()
    tok, msk, nb = out.next_tokens.clone(), out.next_mask.clone(), out.n_next.clone()
    n = int(nb.item())
    full = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=dev)
    lopa.syn_generate(seed, 0, V, tok, msk, n_branches=n, out=full[:n])
    del logits0
    hi = k + 1 if hi is None else hi
    rows = (b_loc if b_loc else k + 1)
    bufs = []
    for _ in range(n_buf):
        b = torch.zeros((rows, W, st.ld), dtype=torch.bfloat16, device=dev)
        if hi > lo:
            b[: hi - lo] = full[lo:hi]
        bufs.append(b)
    torch.cuda.synchronize()
    masked_rows_total = int(msk[:n].sum().item())
    local_rows = int(msk[lo:min(hi, n)].sum().item()) if hi > lo else 0
    return st, tok, msk, nb, full, bufs, masked_rows_total, local_rows


def cpu_baseline_oracle(full, tok, msk, nb, k, tau, budget_s=12.0):
    """The oracle as it stands (NumPy fp64, single thread) on whole verify steps of the same
    workload, repeated until ~budget_s of CPU time."""
    from oracle import lopa_oracle as O
    from threadpoolctl import threadpool_limits
    n = int(nb.item())
    L16 = full.view(torch.int16).cpu().numpy().view(np.uint16)[:n]
    t_np, m_np = tok.cpu().numpy()[:n], msk.cpu().numpy()[:n]
    reps, t0 = 0, time.perf_counter()
    with threadpool_limits(limits=1):  # the stated core count: one thread
        while True:
            O.step(L16, t_np, m_np, k, tau)
            reps += 1
            el = time.perf_counter() - t0
            if el >= budget_s:
                break
    return {"value": reps / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{reps} full verify steps (n_br={n}, {int(m_np.sum())} masked rows x V=151936) "
                      f"in {el:.1f} s, NumPy fp64 single thread"}


def oracle_step_report(full, tok, msk, nb, k, tau, out, bp_conf=None):
    """The bench step's inputs through the oracle once (rank 0): near-tie counts of the step's
    decisions (R16: governing gap < 1e-6, SURVEY §8(d) "near-tie count") and the GPU step's
    agreement with the oracle on exactly the timed inputs (conf max |err|, argmax, winner, the
    spawned tables)."""
    from oracle import lopa_oracle as O
    n = int(nb.item())
    L16 = full.view(torch.int16).cpu().numpy().view(np.uint16)[:n]
    t_np, m_np = tok.cpu().numpy()[:n], msk.cpu().numpy()[:n]
    r = O.step(L16, t_np, m_np, k, tau)
    sel = m_np.astype(bool)
    near = {"select": 0, "anchor": 0, "fallback": 0, "spawn": 0}
    gaps = {}
    sc = sorted([x for x in r.scores if np.isfinite(x)], reverse=True)
    gaps["select"] = float(sc[0] - sc[1]) if len(sc) > 1 else None
    cw = r.conf[r.winner]
    Mw = [i for i in range(m_np.shape[1]) if m_np[r.winner, i]]
    if Mw:
        gaps["anchor"] = float(min(abs(float(cw[i]) - float(np.float32(tau))) for i in Mw))
        c = sorted((float(cw[i]) for i in Mw), reverse=True)
        gaps["fallback"] = float(c[0] - c[1]) if len(c) > 1 else None
    if not r.done:
        M0 = [i for i in range(m_np.shape[1]) if r.anchor.mask[i]]
        c = sorted((float(cw[i]) for i in M0), reverse=True)[: k + 1]
        gaps["spawn"] = float(min((c[q] - c[q + 1] for q in range(len(c) - 1)), default=float("inf")))
    for key, g in gaps.items():
        if g is not None and g < 1e-6:
            near[key] += 1
    rep = {"near_ties": near, "min_gaps": gaps}
    g_w = int(out.winner.item())
    par = {"winner_equal": g_w == r.winner}
    if bp_conf is None:
        gc = out.conf.cpu().numpy()[:n].astype(np.float64)
        ga = out.argmax.cpu().numpy()[:n]
        par["conf_max_abs_err"] = float(np.abs(gc[sel] - r.conf[sel]).max())
        par["argmax_equal"] = bool(np.array_equal(ga[sel], r.argmax[sel]))
    if not r.done:
        nn = int(out.n_next.item())
        par["spawn_equal"] = bool(nn == len(r.spawn.lookahead) + 1 and
                                  np.array_equal(out.next_tokens.cpu().numpy()[:nn], r.spawn.tokens) and
                                  np.array_equal(out.next_mask.cpu().numpy()[:nn], r.spawn.mask))
    rep["oracle_parity"] = par
    return rep


def cpu_baseline_all_cores(full, tok, msk, nb, k, tau, budget_s=8.0):
    """The same oracle step with its row reductions spread over every host core (threads;
    NumPy releases the GIL inside the vectorised exp / sum), as SURVEY §8(d) asks next to the
    one-core figure.  The decisions (O(W k)) stay single-threaded."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import lopa_oracle as O
    n = int(nb.item())
    L16 = full.view(torch.int16).cpu().numpy().view(np.uint16)[:n]
    t_np, m_np = tok.cpu().numpy()[:n], msk.cpu().numpy()[:n]
    rows = [(j, i) for j in range(n) for i in range(m_np.shape[1]) if m_np[j, i]]
    cores = len(os.sched_getaffinity(0))
    shards = [rows[c::cores] for c in range(cores)]

    def reduce_shard(sh):
        return [(j, i, O.row_confidence(L16[j, i])) for (j, i) in sh]

    reps, t0 = 0, time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        while True:
            conf = np.full(m_np.shape, np.nan)
            amax = np.full(m_np.shape, -1, dtype=np.int64)
            for part in ex.map(reduce_shard, shards):
                for (j, i, (c, a, _)) in part:
                    conf[j, i], amax[j, i] = c, a
            scores = [O.branch_score(conf[j], m_np[j]) for j in range(n)]
            w = O.verify_select(scores)
            anc = O.anchor_fill(conf[w], amax[w], t_np[w], m_np[w], tau)
            O.spawn_branches(conf[w], amax[w], anc.tokens, anc.mask, k)
            reps += 1
            el = time.perf_counter() - t0
            if el >= budget_s:
                break
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": reps / el, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": model,
            "sample": f"{reps} full verify steps, row reductions over {cores} threads, in {el:.1f} s"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if CFG.get("K"):
        return run_reference_lmhead(args)
    if CFG.get("d2f_len"):
        from oracle import d2f_oracle as D
        import syngen
        from threadpoolctl import threadpool_limits
        V, k, seed, Lg = CFG["V"], CFG["k"], CFG["seed"], CFG["d2f_len"]
        gen_s = 0.0

        def fwd(b, t, m):
            nonlocal gen_s
            g0 = time.perf_counter()
            x = syngen.gen_logits(seed, b, V, t, m)
            gen_s += time.perf_counter() - g0
            return x
        nf = 6
        with threadpool_limits(limits=1):
            t0 = time.perf_counter()
            tr = D.decode_d2f(fwd, Lg, 32, k, 0.1, 0.95, 0.9, max_window=256, max_forwards=nf)
            el = time.perf_counter() - t0 - gen_s
        value = tr.forwards / el
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (SYN-D2F seeded logits; no weights)", "config": {"workload": CFG["name"]},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                                 "sample": f"the first {tr.forwards} iterations of the D2F decode (oracle/d2f_oracle.py), "
                                           f"generator time ({gen_s:.1f} s) excluded, NumPy fp64 single thread"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "gpu_launches": 0}
        print(json.dumps(line), flush=True)
        return 0
    if CFG.get("loop_blocks"):
        cb = cpu_baseline_loop(CFG["V"], CFG["W"], CFG["k"], CFG["tau"], CFG["seed"],
                               budget_s=max(20.0, min(100.0, 2.0 * (args.steps + args.warmup))))
        value = cb["value"]
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (SYN-D2F seeded logits; no weights)",
                "config": {"workload": CFG["name"]}, "cpu_baseline": cb,
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "gpu_launches": 0}
        print(json.dumps(line), flush=True)
        return 0
    from oracle import lopa_oracle as O
    import syngen
    V, W, k, tau, seed = CFG["V"], CFG["W"], CFG["k"], CFG["tau"], CFG["seed"]
    # same workload as the liblopa arm, built on the CPU with the NumPy generator
    tok0, msk0 = syngen.fresh_block(W)
    L0 = syngen.gen_logits(seed, 0, V, tok0[None], msk0[None])
    r0 = O.step(L0, tok0[None].astype(np.int64), msk0[None], k, tau)
    tok, msk = r0.spawn.tokens, r0.spawn.mask
    L = syngen.gen_logits(seed, 0, V, tok, msk)
    n_rows = int(msk.sum())
    # bounded sample per step so that warmup + steps ends in ~2 minutes
    est = 0.9 * n_rows / 256.0                      # s per full step (1 core)
    frac = min(1.0, 110.0 / max(1, args.steps + args.warmup) / est)
    rows = [(j, i) for j in range(len(msk)) for i in range(W) if msk[j, i]]
    n_s = max(1, int(round(frac * len(rows))))
    sub = rows[:n_s]

    def one():
        # a1 on the sampled rows, then a2-a4 on full-size conf (decisions are O(W k))
        conf = np.full(msk.shape, np.nan)
        for (j, i) in sub:
            conf[j, i], _, _ = O.row_confidence(L[j, i])
        c = np.where(msk.astype(bool), np.nan_to_num(conf, nan=0.5), np.nan)
        scores = [O.branch_score(c[j], msk[j]) for j in range(len(msk))]
        w = O.verify_select(scores)
        a = O.anchor_fill(c[w], np.zeros(W, np.int64), tok[w], msk[w], tau)
        O.spawn_branches(c[w], np.zeros(W, np.int64), a.tokens, a.mask, k)

    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):  # the stated core count: one thread
        for _ in range(args.warmup):
            one()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one()
        el = time.perf_counter() - t0
    f = n_s / len(rows)
    value = args.steps * f / el                     # full verify steps per second
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SYN-D2F seeded logits; no weights)",
            "config": {"workload": CFG.get("name", "D2F-Dream verify step V=151936 W=32 k=7 tau=0.9 (configs[1])"),
                       "masked_rows": len(rows), "sampled_rows_per_step": n_s},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{n_s} of {len(rows)} masked rows per step (+ full a2-a4), "
                                       f"scaled by {len(rows)}/{n_s}; NumPy fp64 single thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- liblopa arm
def head_start(stream, cycles: int = 20_000_000):
    """Keep the device busy ~10 ms (a spin kernel, outside every timed interval) while the host
    queues the launches that follow, so device-side event timestamps measure device work only."""
    with torch.cuda.stream(stream):
        torch.cuda._sleep(cycles)


def run_lopa(args):
    from paper_2512_16229_b200 import lopa
    import ctypes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    V, W, k, tau, seed, n_buf = CFG["V"], CFG["W"], CFG["k"], CFG["tau"], CFG["seed"], CFG["n_buf"]
    # LOPA_BENCH_FORCE_BP=1 runs the branch-parallel path (NCCL communicator of one rank) at N=1,
    # to exercise the N > 1 code path on a single GPU
    use_bp = world > 1 or os.environ.get("LOPA_BENCH_FORCE_BP") == "1"
    if use_bp:
        b_loc, lo, hi = lopa.bp_shard(k + 1, world, rank)
    else:
        b_loc, lo, hi = k + 1, 0, k + 1
    st, tok, msk, nb, full, bufs, rows_total, rows_local = build_workload(
        lopa, dev, V, W, k, tau, seed, n_buf, lo, hi, b_loc if use_bp else None)
    stream = torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    L = lopa.lib()

    bp, p2p_note = (make_branch_parallel(lopa, st, rank, world, dist, dev) if use_bp else (None, None))

    # prebuilt argument structs (one per rotating buffer): the timed loop only launches
    def make_launch(bp):
        if bp is None:
            argv = [st.args(b, nb, tok, msk) for b in bufs]
            refs = [ctypes.byref(a) for a in argv]

            def launch(i):
                s = L.lopa_step(refs[i % n_buf], sptr)
                if s:
                    raise lopa.LopaError(f"lopa_step status {s}")
            return launch, argv
        argv = []
        for b in bufs:
            a = st.args(b, nb, tok, msk)
            a.conf, a.argmax = bp.conf.data_ptr(), bp.argmax.data_ptr()
            a.workspace, a.workspace_bytes = bp.ws.data_ptr(), bp.ws.numel()
            a.scores = bp.scores.data_ptr()
            argv.append(a)
        refs = [ctypes.byref(a) for a in argv]
        rec = ctypes.c_void_p(bp.records.data_ptr())

        def launch(i):
            if bp.p2p:
                s = L.lopa_bp_step_p2p(bp.h, refs[i % n_buf], bp.b_loc, sptr)
            else:
                s = L.lopa_bp_step(bp.h, refs[i % n_buf], bp.b_loc, rec, sptr)
            if s:
                raise lopa.LopaError(f"lopa_bp_step status {s}")
        return launch, argv

    launch, argv = make_launch(bp)
    # warm-up (ranks start it together)
    if dist:
        dist.barrier()
    for i in range(args.warmup):
        launch(i)
    torch.cuda.synchronize()
    if bp is not None and bp.p2p:
        bad = torch.tensor([1 if int(st.out.status.item()) & 4 else 0], device=dev)  # PEER_TIMEOUT
        if not int(bad.item()):
            # cross-check the peer-memory exchange against the NCCL one on the same step: any
            # difference on any rank (winner, branch count, next tables, scores) -> NCCL is used
            o = st.out
            snap = lambda: [o.winner.clone(), o.n_next.clone(), o.next_tokens.clone(), o.next_mask.clone(),
                            bp.scores.clone()]
            r0 = ctypes.byref(argv[0])
            if L.lopa_bp_step(bp.h, r0, bp.b_loc, ctypes.c_void_p(bp.records.data_ptr()), sptr):
                raise lopa.LopaError("lopa_bp_step (cross-check) failed")
            torch.cuda.synchronize()
            ref = snap()
            if L.lopa_bp_step_p2p(bp.h, r0, bp.b_loc, sptr):
                raise lopa.LopaError("lopa_bp_step_p2p (cross-check) failed")
            torch.cuda.synchronize()
            got = snap()
            same = all(torch.equal(x.view(torch.int32) if x.dtype == torch.float32 else x,
                                   y.view(torch.int32) if y.dtype == torch.float32 else y)
                       for x, y in zip(ref, got))
            bad = torch.tensor([0 if same else 2], device=dev)
            if int(st.out.status.item()) & 4:
                bad.fill_(1)
        if dist is not None:
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
        if int(bad.item()) == 2:
            p2p_note = "peer-memory exchange disagreed with the NCCL exchange on the warm-up step; NCCL all-gather used"
        if int(bad.item()):
            # a peer's record never arrived within the bounded wait: measure the NCCL exchange
            # instead (and say so in the line) rather than fail the run
            bp.close()
            bp = lopa.BranchParallel(st, rank, world, p2p=False)
            p2p_note = p2p_note or "peer-memory exchange timed out during the warm-up; NCCL all-gather used"
            st.out.status.zero_()
            launch, argv = make_launch(bp)
            if dist:
                dist.barrier()
            for i in range(args.warmup):
                launch(i)
            torch.cuda.synchronize()

    # timed region (headline): K steps back to back, events only at the ends (so the PDL overlap
    # between a step's kernels and the next step's is not broken by interleaved event records)
    K = args.steps
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        head_start(stream)
        t_start.record(stream)
        for i in range(K):
            launch(i)
        t_end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    el_ms = t_start.elapsed_time(t_end)
    if dist:
        t = torch.tensor([el_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el_ms = float(t.item())
    # roofline pass A: K1's duration as launched inside the step, i.e. PDL-chained so that its
    # launch latency overlaps the previous kernel: CUDA events around K back-to-back
    # lopa_confidence calls (K1 + its one-CTA fold kernel) over exactly this rank's masked rows
    # of the rotating buffers -> an upper bound of K1's average duration
    n_rows = bufs[0].shape[0] * W
    nb_i = int(nb.item())
    rmask = torch.zeros((bufs[0].shape[0], W), dtype=torch.uint8, device=dev)
    for j in range(bufs[0].shape[0]):
        if lo + j < min(hi, nb_i):
            rmask[j] = msk[lo + j]
    rmask = rmask.reshape(-1).contiguous()
    c_out = torch.empty(n_rows, dtype=torch.float32, device=dev)
    a_out = torch.empty(n_rows, dtype=torch.int32, device=dev)
    c_st = lopa.new_status(dev)
    c_ws = lopa.new_workspace(n_rows, V, dev)
    ldv = bufs[0].shape[-1]
    P_ = lopa._p

    def conf_call(i):
        s_ = L.lopa_confidence(P_(bufs[i % n_buf]), ldv, n_rows, V, P_(rmask), P_(c_out), P_(a_out),
                               P_(c_st), P_(c_ws), c_ws.numel(), sptr)
        if s_:
            raise lopa.LopaError(f"lopa_confidence status {s_}")

    for i in range(args.warmup):
        conf_call(i)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    head_start(stream)
    c0.record(stream)
    for i in range(K):
        conf_call(i)
    c1.record(stream)
    torch.cuda.synchronize()
    chain_ms = c0.elapsed_time(c1) / K
    if int(c_st.item()) != 0:
        raise lopa.LopaError(f"device status {int(c_st.item())}")

    # K1 alone (lopa_debug_reduce_only: the step's launch configuration, no fold kernel),
    # K back-to-back PDL-chained launches over the same rows: K1's average launch duration
    def k1_call(i):
        s_ = L.lopa_debug_reduce_only(P_(bufs[i % n_buf]), ldv, n_rows, V, P_(rmask), P_(c_st),
                                      P_(c_ws), c_ws.numel(), sptr)
        if s_:
            raise lopa.LopaError(f"lopa_debug_reduce_only status {s_}")

    for i in range(args.warmup):
        k1_call(i)
    torch.cuda.synchronize()
    head_start(stream)
    c0.record(stream)
    for i in range(K):
        k1_call(i)
    c1.record(stream)
    torch.cuda.synchronize()
    k1_ms = c0.elapsed_time(c1) / K
    # roofline pass B (context): an event pair around every K1 inside the same K steps; each
    # pair also holds K1's launch latency, which the step's PDL chain otherwise hides
    # (in batches, each behind a device-side head start, so that host launch overhead never
    # shows up between a K1's start and end events)
    lopa.profile_enable(K)
    for b0 in range(0, K, 200):
        head_start(stream)
        for i in range(b0, min(K, b0 + 200)):
            launch(i)
        torch.cuda.synchronize()
    per = lopa.profile_read(K)
    if int(st.out.status.item()) != 0:
        raise lopa.LopaError(f"device status {int(st.out.status.item())}")
    if bp is not None:
        bp.check()
    value = K / (el_ms / 1000.0)
    pair_ms = statistics.mean(per) if per else float("nan")
    # step-time distribution: N_LAT individually timed steps, each bracketed by its
    # own CUDA event pair on the stream (queued behind a device-side head start, so host launch
    # time never falls inside a pair).  The events sit between consecutive steps, so each step
    # runs ISOLATED: K1's launch cannot overlap the previous step's tail as in the PDL-chained
    # timed region (whose mean is the headline).  Percentiles over the per-step latencies.
    N_LAT = max(1000, min(K, 2000))
    lat_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(N_LAT)]
    lat = []
    for b0 in range(0, N_LAT, 250):
        head_start(stream)
        for i in range(b0, min(N_LAT, b0 + 250)):
            lat_ev[i][0].record(stream)
            launch(i)
            lat_ev[i][1].record(stream)
        torch.cuda.synchronize()
    lat = sorted(a.elapsed_time(b) * 1000.0 for a, b in lat_ev)

    def pct(q):
        return lat[min(len(lat) - 1, int(q * (len(lat) - 1) + 0.5))]

    step_dist = {"isolated_step_us": {"p10": pct(0.10), "p50": pct(0.50), "p90": pct(0.90),
                                      "p99": pct(0.99), "min": lat[0], "max": lat[-1], "n": len(lat)},
                 "chained_mean_us": el_ms / K * 1000.0,
                 "note": "isolated: one event pair per step (no PDL overlap with the neighbouring "
                         "steps); chained: the headline's mean over K back-to-back steps"}
    # dense kernel roofline (SURVEY §8(d) mode (i)): every (branch, position) row of the
    # buffers reduced, (k + 1) * W rows, same CUDA-event chain as pass A
    dense = None
    if bp is None:
        dmask = torch.ones(n_rows, dtype=torch.uint8, device=dev)

        def dense_call(i):
            s_ = L.lopa_debug_reduce_only(P_(bufs[i % n_buf]), ldv, n_rows, V, P_(dmask), P_(c_st),
                                          P_(c_ws), c_ws.numel(), sptr)
            if s_:
                raise lopa.LopaError(f"lopa_debug_reduce_only status {s_}")

        for i in range(args.warmup):
            dense_call(i)
        torch.cuda.synchronize()
        head_start(stream)
        c0.record(stream)
        for i in range(K):
            dense_call(i)
        c1.record(stream)
        torch.cuda.synchronize()
        d_ms = c0.elapsed_time(c1) / K
        d_bytes = 2.0 * V * n_rows
        dense = {"rows": n_rows, "kernel_ms_mean": d_ms, "achieved_gbs": d_bytes / (d_ms / 1000.0) / 1e9}
    kern_ms = k1_ms
    alg_bytes = 2.0 * V * rows_local                 # 2 B per logit of a masked row
    achieved = alg_bytes / (kern_ms / 1000.0) / 1e9
    pk = peaks()
    peak = float(pk.get("hbm_gbs", 6650.0))

    # Alg. 1 loop captured in one CUDA graph (lopa.StepLoopGraph): 32 iterations whose tables
    # feed back on the device, replayed; per-iteration time of the captured loop
    graph_loop = None
    if world == 1 and bp is None:
        g_tok, g_msk, g_nb = tok.clone(), msk.clone(), nb.clone()
        st_g = lopa.Stepper(V, W, k + 1, k, tau, dev)
        GL = 32
        gl = lopa.StepLoopGraph(st_g, bufs, g_nb, g_tok, g_msk, GL)
        reps = 20
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gl.replay()
        torch.cuda.synchronize()
        g0.record(stream)
        for _ in range(reps):
            g_tok.copy_(tok), g_msk.copy_(msk), g_nb.copy_(nb)
            gl.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        graph_loop = {"us_per_iteration": g0.elapsed_time(g1) * 1000.0 / (reps * GL), "iterations": GL,
                      "replays": reps, "note": "one CUDA graph per 32-iteration loop (tables fed back on "
                      "the device; fixed logits buffers, so later iterations have fewer masked rows)"}

    # BP: the exchange's collective alone (SURVEY §8(d) "comm µs"): the same all-gather size
    # through the torch NCCL process group, CUDA events around 200 back-to-back calls
    comm = None
    if bp is not None and dist is not None:
        sendb = torch.zeros(bp.rb, dtype=torch.uint8, device=dev)
        recvb = torch.empty(world * bp.rb, dtype=torch.uint8, device=dev)
        for _ in range(10):
            dist.all_gather_into_tensor(recvb, sendb)
        torch.cuda.synchronize()
        dist.barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(200):
            dist.all_gather_into_tensor(recvb, sendb)
        x1.record(stream)
        torch.cuda.synchronize()
        comm = {"allgather_us": x0.elapsed_time(x1) * 1000.0 / 200, "bytes_per_rank": bp.rb,
                "note": "torch all_gather_into_tensor of the record size (the exchange's collective)"}

    # the Alg. 1 loop over whole blocks (SURVEY §8(d) "TPF, loop only"): lopa.decode_block on the
    # SYN-D2F forward (generator + step per iteration, device time), 8 blocks of this shape
    loop = None
    if world == 1 and bp is None:
        fw_total, tok_total = 0, 0
        l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st_l = lopa.Stepper(V, W, k + 1, k, tau, dev)
        l0.record(stream)
        for blk in range(8):
            fwd = lambda t, m, out, blk=blk: lopa.syn_generate(seed, blk, V, t, m, out=out)
            t0_ = torch.zeros(W, dtype=torch.int32, device=dev)
            m0_ = torch.ones(W, dtype=torch.uint8, device=dev)
            _, fw = lopa.decode_block(fwd, t0_, m0_, k, tau, V, stepper=st_l)
            fw_total += fw
            tok_total += W
        l1.record(stream)
        torch.cuda.synchronize()
        loop = {"blocks": 8, "tokens": tok_total, "forwards": fw_total, "tpf": tok_total / fw_total,
                "ms_per_block_incl_generator": l0.elapsed_time(l1) / 8,
                "note": "one host read per iteration (branch count); SYN-D2F forward on the GPU"}
        # the same 8 blocks, each ONE self-terminating CUDA graph launch (conditional WHILE node:
        # the loop stops on the device when the selected branch is complete; no host read)
        graphs = [lopa.DecodeBlockGraph(lopa.Stepper(V, W, k + 1, k, tau, dev), seed, blk) for blk in range(8)]
        t0_ = torch.zeros(W, dtype=torch.int32, device=dev)
        m0_ = torch.ones(W, dtype=torch.uint8, device=dev)
        for g_ in graphs:
            g_.run(t0_, m0_)
        torch.cuda.synchronize()
        l0.record(stream)
        for g_ in graphs:
            g_.run(t0_, m0_)
        l1.record(stream)
        torch.cuda.synchronize()
        fw_g = sum(g_.forwards() for g_ in graphs)
        loop["graph_ms_per_block_incl_generator"] = l0.elapsed_time(l1) / 8
        loop["graph_forwards"] = fw_g
        loop["graph_note"] = "each block one device-terminated CUDA graph (lopa.DecodeBlockGraph)"
        for g_ in graphs:
            g_.graph.close()

    # e2e through the public API with HOST buffers: pinned logits -> device, step, results -> host.
    # At N > 1 (branch-parallel) each rank copies its own shard of the logits (its branches'
    # rows) and runs BranchParallel.step; the time is the max over ranks.
    src = full if bp is None else bufs[0]
    host = src.cpu().pin_memory()
    h_tok, h_msk, h_nb = tok.cpu().pin_memory(), msk.cpu().pin_memory(), nb.cpu().pin_memory()
    d_log = torch.empty_like(src)
    d_tok, d_msk, d_nb = torch.empty_like(tok), torch.empty_like(msk), torch.empty_like(nb)
    o = st.out
    out_t = (o.winner, o.scores, o.next_tokens, o.next_mask, o.n_next, o.status)
    h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in out_t]
    K2 = max(3, min(K, 50))

    def e2e_step():
        d_log.copy_(host, non_blocking=True)
        d_tok.copy_(h_tok, non_blocking=True)
        d_msk.copy_(h_msk, non_blocking=True)
        d_nb.copy_(h_nb, non_blocking=True)
        if bp is None:
            st.step(d_log, d_nb, d_tok, d_msk, validate=False)
        else:
            bp.step(d_log, d_nb, d_tok, d_msk)
        for h, t in zip(h_out, out_t):
            h.copy_(t, non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K2):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    h2d = src.numel() * 2 + tok.numel() * 4 + msk.numel() + nb.numel() * 4
    d2h = sum(t.numel() * t.element_size() for t in h_out)
    e2e = {"value": K2 / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": K2}
    if bp is not None:
        e2e["note"] = "per rank: its logits shard (b_loc branches) + the replicated tables from pinned host memory; max over ranks"

    if rank == 0:
        cpu = cpu_all = None
        if not args.no_cpu_baseline:
            # rank 0 only, on the whole step's workload (all ranks' branches): the CPU baseline
            # of the same metric, independent of N
            cpu = cpu_baseline_oracle(full, tok, msk, nb, k, tau)
            cpu_all = cpu_baseline_all_cores(full, tok, msk, nb, k, tau)
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            try:
                traffic = json.load(open(tf)).get("bytes_per_launch")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": el_ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (SYN-D2F seeded logits; transformer forward out of scope)",
            "config": {"workload": CFG.get("name", "D2F-Dream verify step V=151936 W=32 k=7 tau=0.9 (configs[1])"),
                       "branches": int(nb.item()), "masked_rows": rows_total,
                       "masked_rows_this_rank": rows_local,
                       "parallelism": (f"bp{world}" + ("-p2p" if bp.p2p else "")) if bp is not None else "single",
                       "bp_exchange": (None if bp is None else
                                       ("peer memory, fused into K2 (lopa_bp_step_p2p)" if bp.p2p else "NCCL all-gather")
                                       + ("" if p2p_note is None else f" [{p2p_note}]")),
                       "l2": f"rotating {n_buf} logits buffers ({n_buf * full.numel() * 2 / 1e6:.0f} MB >= 4x L2)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "frac_datasheet_8tbs": achieved / 8000.0,
                         "kernel": "lopa_reduce_kernel (K1, a1 vocabulary reduction)",
                         "kernel_ms_mean": kern_ms,
                         "kernel_timing": f"CUDA events around {K} back-to-back K1 launches (lopa_debug_reduce_only: the step's grid, PDL-chained as in lopa_step, each waiting for the previous to complete) over this rank's {rows_local} masked rows of the rotating buffers",
                         "conf_call_ms": chain_ms,
                         "conf_call_note": "the same rows through lopa_confidence (K1 + its 1-CTA fold kernel), back to back",
                         "k1_event_pair_ms": pair_ms,
                         "k1_event_pair_note": "event pair around each K1 inside lopa_step; includes K1's launch latency that PDL hides in the timed steps",
                         "alg_bytes_per_launch": alg_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "_fallback" not in pk else "fallback"},
            "logits_gbs_step": alg_bytes / (el_ms / K / 1000.0) / 1e9,
            "clocks": clk.summary(),
            "gpu_launches": K * (2 if bp is None or bp.p2p else 3),
        }
        if e2e is not None:
            line["e2e"] = e2e
        if graph_loop is not None:
            line["graph_loop"] = graph_loop
        line["step_time_distribution"] = step_dist
        if loop is not None:
            line["decode_loop"] = loop
        if comm is not None:
            line["bp_comm"] = comm
        if dense is not None:
            dense["frac"] = dense["achieved_gbs"] / peak
            line["dense_roofline"] = dense
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if cpu_all is not None:
            line["cpu_baseline_all_cores"] = cpu_all
        if not args.no_cpu_baseline:
            try:
                line["decisions"] = oracle_step_report(full, tok, msk, nb, k, tau, st.out,
                                                       bp_conf=None if bp is None else bp.conf)
            except Exception as e:  # report, never hide the bench line
                line["decisions"] = {"error": repr(e)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()  # rank 0's CPU baseline runs while the others wait here
    if bp is not None:
        bp.close()
    if dist:
        dist.destroy_process_group()
    return 0


class _SingleGPU:
    """decode_block_bp's driver interface over the fused single-GPU step (no exchange)."""

    def __init__(self, st):
        self.s = st
        self.local = torch.zeros((st.max_branches, st.window, st.ld), dtype=torch.bfloat16, device=st.device)

    def ranks(self):
        return [(0, 0, self.s.max_branches, self.local)]

    def step(self, *a):
        if len(a) == 3:
            a = (self.local, *a)
        return self.s.step(*a, validate=False)


def run_loop(args):
    """BASELINE configs[2] / configs[3]: whole Alg. 1 decode loops over
    `loop_blocks` sequential blocks (R22), branch-parallel over the N ranks at N > 1 (each
    rank reduces only its own branches; one record all-gather per step).  A "step" = one verify
    step of the loop (a block's initial predict counts as a step with one branch).  The SYN-D2F
    logits of every step are generated once, by a recording pass of the same loop, and kept
    resident in HBM -- each rank holds only its own branches' logits; the timed region replays
    the loop from the start (one host read of the branch count per step, as lopa.decode_block)
    until exactly K steps have run."""
    from paper_2512_16229_b200 import lopa

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    V, W, k, tau, seed, nblk = CFG["V"], CFG["W"], CFG["k"], CFG["tau"], CFG["seed"], CFG["loop_blocks"]
    st = lopa.Stepper(V, W, k + 1, k, tau, dev)
    use_bp = world > 1 or os.environ.get("LOPA_BENCH_FORCE_BP") == "1"
    drv = make_branch_parallel(lopa, st, rank, world, dist, dev)[0] if use_bp else _SingleGPU(st)
    _, lo, hi, _buf = drv.ranks()[0]
    stream = torch.cuda.current_stream(dev)

    # recording pass: the loop with the generator as the forward; each step's local logits kept
    rec, fw_blocks, tokens = [], [], []
    for blk in range(nblk):
        steps = []
        fwd = lambda t, m, out, blk=blk: lopa.syn_generate(seed, blk, V, t, m, out=out)
        on_step = lambda out, n, t, m: steps.append((n, drv.local[: max(0, min(hi, n) - lo)].clone()))
        t0 = torch.zeros(W, dtype=torch.int32, device=dev)
        m0 = torch.ones(W, dtype=torch.uint8, device=dev)
        tk, fw = lopa.decode_block_bp(drv, fwd, t0, m0, on_step=on_step)
        rec.append(steps)
        fw_blocks.append(fw)
        tokens.append(tk)
    torch.cuda.synchronize()
    steps_per_pass = sum(fw_blocks)
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=dev)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=dev)
    nb = torch.ones(1, dtype=torch.int32, device=dev)
    lbuf = torch.zeros((drv.ranks()[0][3].shape), dtype=torch.bfloat16, device=dev)
    # per step: this rank's logits rows, copied into the step's buffer view (zero copies: a view
    # padded to b_loc rows is made once per recorded step)
    padded = []
    for steps in rec:
        pb = []
        for n, x in steps:
            b = torch.zeros_like(lbuf)
            if x.shape[0]:
                b[: x.shape[0]] = x
            pb.append(b)
        padded.append(pb)
    del rec
    torch.cuda.synchronize()

    def run_steps(count, check=True):
        """Replay the recorded loop from block 0 for exactly `count` verify steps."""
        done, blk, si = 0, 0, 0
        while done < count:
            if si == 0:
                tok.zero_()
                msk.zero_()
                msk[0] = 1
                nb.fill_(1)
            out = drv.step(padded[blk][si], nb, tok, msk)
            done += 1
            n = int(out.n_next.item())
            si += 1
            if n == 0:
                if check and si != fw_blocks[blk]:
                    raise RuntimeError(f"replay diverged: block {blk} ended after {si} steps, recorded {fw_blocks[blk]}")
                blk, si = (blk + 1) % nblk, 0
            else:
                tok.copy_(out.next_tokens)
                msk.copy_(out.next_mask)
                nb.copy_(out.n_next)

    run_steps(max(args.warmup, 3))
    torch.cuda.synchronize()
    K = args.steps
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        run_steps(K)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    el_ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([el_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el_ms = float(t.item())
    if int(st.out.status.item()) != 0:
        raise lopa.LopaError(f"device status {int(st.out.status.item())}")
    if use_bp:
        drv.check()

    # e2e: the same loop through the public API with each step's logits shard copied from pinned
    # host memory (block 0, every step) and the step's results read back, inside the timed region
    host0 = [b.cpu().pin_memory() for b in padded[0]]
    o = st.out
    h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory()
             for t in (o.winner, o.next_tokens, o.next_mask, o.n_next, o.status)]
    d_l = torch.empty_like(lbuf)

    def e2e_block():
        tok.zero_()
        msk.zero_()
        msk[0] = 1
        nb.fill_(1)
        for si, hb in enumerate(host0):
            d_l.copy_(hb, non_blocking=True)
            out = drv.step(d_l, nb, tok, msk)
            for h, t in zip(h_out, (o.winner, o.next_tokens, o.next_mask, o.n_next, o.status)):
                h.copy_(t, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
            if int(h_out[3].item()) == 0:
                return si + 1
            tok.copy_(out.next_tokens)
            msk.copy_(out.next_mask)
            nb.copy_(out.n_next)
        return len(host0)

    e2e_block()
    if dist:
        dist.barrier()
    reps = 3
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    n_e2e = sum(e2e_block() for _ in range(reps))
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    h2d = sum(b.numel() * 2 for b in host0) / len(host0)
    d2h = sum(t.numel() * t.element_size() for t in h_out)

    # the recorded trajectory replayed as ONE static CUDA graph (the step count of every block from
    # the recording; no host read): the device time of the LoPA loop itself on resident logits
    graph_replay = None
    if True:  # both exchanges are graph safe (the peer-memory epoch lives on the device)
        def replay_all():
            for blk in range(nblk):
                tok.zero_()
                msk.zero_()
                msk[0].fill_(1)
                nb.fill_(1)
                for si in range(fw_blocks[blk]):
                    out = drv.step(padded[blk][si], nb, tok, msk)
                    tok.copy_(out.next_tokens)
                    msk.copy_(out.next_mask)
                    nb.copy_(out.n_next)
        replay_all()
        torch.cuda.synchronize()
        cgr = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            with torch.cuda.graph(cgr, stream=cs):
                replay_all()
        torch.cuda.synchronize()
        for _ in range(2):
            cgr.replay()
        torch.cuda.synchronize()
        if int(st.out.n_next.item()) != 0:
            raise RuntimeError("graph replay did not end its last block")
        reps_g = max(2, min(20, K // max(1, steps_per_pass)))
        if dist:
            dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(reps_g):
            cgr.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gr_ms = g0.elapsed_time(g1)
        if dist:
            t = torch.tensor([gr_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gr_ms = float(t.item())
        graph_replay = {"us_per_step": gr_ms * 1000.0 / (reps_g * steps_per_pass),
                        "verify_steps_per_s": reps_g * steps_per_pass / (gr_ms / 1000.0),
                        "passes": reps_g,
                        "note": "the recorded loop (every step's resident logits shard, tables fed "
                                "back on the device, block starts reset on the device) as one static "
                                "CUDA graph; the step counts come from the recording pass"}
        del cgr

    # the same decode with each block ONE device-terminated CUDA graph (conditional WHILE node;
    # no host read at all; the SYN-D2F forward of this rank's branches inside the loop)
    dev_loop = None
    if True:
        graphs = [(lopa.DecodeBlockGraphBP(drv, seed, blk) if use_bp else lopa.DecodeBlockGraph(st, seed, blk))
                  for blk in range(nblk)]
        t0_ = torch.zeros(W, dtype=torch.int32, device=dev)
        m0_ = torch.ones(W, dtype=torch.uint8, device=dev)
        for g_ in graphs:
            g_.run(t0_, m0_)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for g_ in graphs:
            g_.run(t0_, m0_)
        d1.record(stream)
        torch.cuda.synchronize()
        dl_ms = d0.elapsed_time(d1)
        if dist:
            t = torch.tensor([dl_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dl_ms = float(t.item())
        fw_dl = [g_.forwards() for g_ in graphs]
        if fw_dl != fw_blocks:
            raise RuntimeError(f"device-terminated loop diverged: {fw_dl} vs {fw_blocks}")
        dev_loop = {"us_per_step_incl_forward": dl_ms * 1000.0 / steps_per_pass,
                    "ms_per_pass": dl_ms, "forwards_per_block": fw_dl,
                    "note": "each block one device-terminated CUDA graph (lopa.DecodeBlockGraph"
                            + (("BP, peer-memory exchange fused into K2, epoch on the device" if getattr(drv, "p2p", False)
                                else "BP, NCCL all-gather inside the graph") if use_bp else "") +
                            "): no host read; includes the SYN-D2F forward of this rank's branches"}
        for g_ in graphs:
            g_.graph.close()

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline_loop(V, W, k, tau, seed)
        tok_total = W * nblk
        line = {
            "metric": METRIC, "value": K / (el_ms / 1000.0), "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": el_ms / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (SYN-D2F seeded logits of each step, generated once and resident in HBM; transformer forward out of scope)",
            "config": {"workload": CFG["name"], "blocks": nblk, "tokens_per_pass": tok_total,
                       "verify_steps_per_pass": steps_per_pass, "forwards_per_block": fw_blocks,
                       "tpf": tok_total / steps_per_pass,
                       "parallelism": (f"bp{world}" + ("-p2p" if getattr(drv, "p2p", False) else "")) if use_bp else "single",
                       "branches_this_rank": [lo, hi],
                       "l2": "each step reads its own logits (resident, >= 4x L2 over a pass)"},
            "tokens_per_s": tok_total * (K / steps_per_pass) / (el_ms / 1000.0),
            "loop_note": "one host read (branch count) per step, as lopa.decode_block; the loop restarts at block 0 after the last block",
            "clocks": clk.summary(),
            "gpu_launches": K * (3 if use_bp else 2),
            "e2e": {"value": n_e2e / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": n_e2e,
                    "note": "block 0 replayed 3x: each step's logits shard (this rank's branches) from pinned host memory, results to host, max over ranks"},
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if dev_loop is not None:
            line["device_loop"] = dev_loop
        if graph_replay is not None:
            line["graph_replay"] = graph_replay
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()  # rank 0's CPU baseline runs while the others wait here
    if use_bp:
        drv.close()
    if dist:
        dist.destroy_process_group()
    return 0


def run_d2f(args):
    """--config d2f-graph (NEXT-1): the D2F decode of a 256-token region with the block scheduler
    on the device (d2f.D2FDeviceLoop: harness forward + lopa_step on the device window +
    lopa_d2f_update per iteration, no host read), captured in ONE CUDA graph and replayed; beside
    it the host-driven pipeline (d2f.decode_d2f: two host reads and a few torch ops per
    iteration) on the same decode.  Both include the SYN-D2F forward stand-in of every
    iteration (it cannot be precomputed without the decode's trajectory); a step = one
    iteration.  One GPU."""
    from paper_2512_16229_b200 import d2f, lopa
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != 1:
        print(json.dumps({"error": "d2f-graph runs on one GPU"}))
        return 0
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    V, k, seed, Lg = CFG["V"], CFG["k"], CFG["seed"], CFG["d2f_len"]
    cfg = d2f.BlockConfig(32, 0.1, 0.95, 0.9, 256)
    fwd = lambda b, t, m: lopa.syn_generate(seed, b, V, t, m)
    h = d2f.decode_d2f(fwd, Lg, k, cfg, V, dev)          # trajectory length, warm-up
    iters = h.forwards
    loop = d2f.D2FDeviceLoop(Lg, k, cfg, V, dev, seed)
    loop.capture(iters)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(3, min(args.steps // max(1, iters), 50))
    for _ in range(2):
        loop.reset()
        loop.replay()
    torch.cuda.synchronize()
    dev_ms = 0.0
    with ClockSampler(0) as clk:
        for _ in range(reps):
            loop.reset()
            e0.record(stream)
            loop.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            dev_ms += e0.elapsed_time(e1)
    g = loop.trace()
    if g.forwards != iters or g.winners != h.winners or not torch.equal(g.tokens, h.tokens):
        raise RuntimeError("device D2F loop diverged from the host pipeline")
    # host-driven pipeline on the same decode (device time between its first and last kernel)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hreps = 3
    host_ms = 0.0
    for _ in range(hreps):
        h0.record(stream)
        d2f.decode_d2f(fwd, Lg, k, cfg, V, dev)
        h1.record(stream)
        torch.cuda.synchronize()
        host_ms += h0.elapsed_time(h1)
    # the harness forward alone, as the same captured loop runs it: one graph of the forwards of
    # the recorded windows (the scheduler state replayed from the trace is not needed: the
    # forward's cost depends on the window size and branch count only)
    # the same decode as ONE self-terminating graph (conditional WHILE: stops on the device when
    # every block is committed; no iteration count)
    wg = loop.capture_while()
    wg_ms = 0.0
    for r_ in range(reps + 2):
        loop.reset()
        e0.record(stream)
        loop.launch_while()
        e1.record(stream)
        torch.cuda.synchronize()
        if r_ >= 2:
            wg_ms += e0.elapsed_time(e1)
    if wg.iterations() != iters or not torch.equal(loop.trace().tokens, h.tokens):
        raise RuntimeError("device-terminated D2F loop diverged from the host pipeline")
    wg.close()
    per_it = dev_ms / reps / iters
    line = {
        "metric": METRIC, "value": 1000.0 / per_it, "unit": UNIT, "n_gpus": 1, "steps": reps * iters,
        "warmup": 2 * iters, "ms_per_step": per_it, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (SYN-D2F forward generated on the device inside the loop)",
        "config": {"workload": CFG["name"], "gen_len": Lg, "iterations_per_decode": iters,
                   "tokens_per_forward": Lg / iters, "max_window": max(w[1] for w in g.windows),
                   "parallelism": "single"},
        "d2f": {"device_graph_us_per_iteration": per_it * 1000.0,
                "device_while_graph_us_per_iteration": wg_ms / reps / iters * 1000.0,
                "host_pipeline_us_per_iteration": host_ms / hreps / iters * 1000.0,
                "speedup": (host_ms / hreps) / (dev_ms / reps),
                "note": "both include the SYN-D2F forward of every iteration (windows up to 256 "
                        "positions x up to 16 branches); the graph has no host read"},
        "clocks": clk.summary(),
        "gpu_launches": reps * iters * 4,
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_loop(V, W, k, tau, seed, budget_s=15.0):
    """The oracle's Alg. 1 loop (NumPy fp64, one thread) on the same workload: whole blocks
    (generator included, as the CPU stand-in for the forward) until ~budget_s."""
    from oracle import lopa_oracle as O
    from threadpoolctl import threadpool_limits
    import syngen
    steps, blocks, gen_s = 0, 0, 0.0
    t0 = time.perf_counter()
    with threadpool_limits(limits=1):
        while time.perf_counter() - t0 < budget_s:
            def fwd(t, m, blk=blocks):
                nonlocal gen_s
                g0 = time.perf_counter()
                x = syngen.gen_logits(seed, blk, V, t, m)
                gen_s += time.perf_counter() - g0
                return x
            tok0, msk0 = syngen.fresh_block(W)
            steps += O.decode_block(fwd, tok0, msk0, k, tau).forwards
            blocks += 1
    el = time.perf_counter() - t0 - gen_s
    return {"value": steps / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{blocks} whole blocks ({steps} verify steps) of the loop, NumPy fp64 single thread; "
                      f"the generator's time ({gen_s:.1f} s) excluded"}


def run_lmhead(args):
    """--config lmhead-dream: lopa_step_lmhead (tcgen05 LM head with the Conf epilogue, then the
    decision kernel) on synthetic hidden states and a random-init output projection."""
    from paper_2512_16229_b200 import lopa
    import ctypes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or os.environ.get("LOPA_BENCH_FORCE_BP") == "1":
        return run_lmhead_bp(args)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    V, W, k, tau, Kd = CFG["V"], CFG["W"], CFG["k"], CFG["tau"], CFG["K"]
    st, tok, msk, nb, full, bufs, rows_total, _ = build_workload(lopa, dev, V, W, k, tau, CFG["seed"], 1)
    del full, bufs
    rows = (k + 1) * W
    g = torch.Generator(device=dev).manual_seed(CFG["seed"])
    NW = 2   # two 1.09 GB weight copies, alternated: every step streams its weights from HBM
    Ws = [(torch.randn(V, Kd, device=dev, generator=g) / Kd ** 0.5).to(torch.bfloat16) for _ in range(NW)]
    NH = 8
    Hs = [(torch.randn(rows, Kd, device=dev, generator=g) * 1.5).to(torch.bfloat16) for _ in range(NH)]
    heads = [lopa.LMHead(w, max_rows=rows) for w in Ws]
    L = lopa.lib()
    stream = torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    argv = [st.args(Hs[0], nb, tok, msk) for _ in range(NW)]
    refs = [ctypes.byref(a) for a in argv]
    P_ = lopa._p

    def launch(i):
        hd = heads[i % NW]
        s_ = L.lopa_step_lmhead(refs[i % NW], P_(Hs[i % NH]), Kd, P_(hd.weight), Kd, Kd,
                                P_(hd.ws), hd.ws.numel(), sptr)
        if s_:
            raise lopa.LopaError(f"lopa_step_lmhead status {s_}")

    for i in range(args.warmup):
        launch(i)
    torch.cuda.synchronize()
    K = args.steps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        head_start(stream)
        t0.record(stream)
        for i in range(K):
            launch(i)
        t1.record(stream)
        torch.cuda.synchronize()
    el_ms = t0.elapsed_time(t1)
    if int(st.out.status.item()) != 0:
        raise lopa.LopaError(f"device status {int(st.out.status.item())}")
    # roofline: the LM-head kernel (+ its fold) chained back to back, CUDA events at the ends
    for i in range(3):
        heads[i % NW](Hs[i % NH])
    torch.cuda.synchronize()
    head_start(stream)
    t0.record(stream)
    for i in range(K):
        heads[i % NW](Hs[i % NH])
    t1.record(stream)
    torch.cuda.synchronize()
    kern_ms = t0.elapsed_time(t1) / K
    flops = 2.0 * rows * Kd * V
    pk = peaks()
    peak = float(pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1416.0)))
    achieved = flops / (kern_ms / 1000.0) / 1e12
    # e2e: hidden states + tables from pinned host memory, results back, inside the timed region
    hh = Hs[0].cpu().pin_memory()
    h_tok, h_msk, h_nb = tok.cpu().pin_memory(), msk.cpu().pin_memory(), nb.cpu().pin_memory()
    d_h = torch.empty_like(Hs[0])
    d_tok, d_msk, d_nb = torch.empty_like(tok), torch.empty_like(msk), torch.empty_like(nb)
    o = st.out
    h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory()
             for t in (o.winner, o.scores, o.next_tokens, o.next_mask, o.n_next, o.status)]
    ea = st.args(d_h, d_nb, d_tok, d_msk)
    K2 = max(3, min(K, 200))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(K2):
        d_h.copy_(hh, non_blocking=True)
        d_tok.copy_(h_tok, non_blocking=True)
        d_msk.copy_(h_msk, non_blocking=True)
        d_nb.copy_(h_nb, non_blocking=True)
        hd = heads[i % NW]
        s_ = L.lopa_step_lmhead(ctypes.byref(ea), P_(d_h), Kd, P_(hd.weight), Kd, Kd, P_(hd.ws),
                                hd.ws.numel(), sptr)
        if s_:
            raise lopa.LopaError(f"lopa_step_lmhead status {s_}")
        for hbuf, dsrc in zip(h_out, (o.winner, o.scores, o.next_tokens, o.next_mask, o.n_next, o.status)):
            hbuf.copy_(dsrc, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    h2d = hh.numel() * 2 + tok.numel() * 4 + msk.numel() + nb.numel() * 4
    d2h = sum(t.numel() * t.element_size() for t in h_out)
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline_lmhead(Hs[0].view(torch.int16).cpu().numpy().view(np.uint16),
                                  Ws[0].view(torch.int16).cpu().numpy().view(np.uint16), rows)
    line = {
        "metric": METRIC, "value": K / (el_ms / 1000.0), "unit": UNIT, "n_gpus": 1, "steps": K,
        "warmup": args.warmup, "ms_per_step": el_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init output projection, Gaussian hidden states; transformer body out of scope)",
        "config": {"workload": CFG["name"], "rows": rows, "masked_rows": rows_total, "hidden": Kd,
                   "parallelism": "single",
                   "l2": f"{NW} rotating weight copies ({NW * V * Kd * 2 / 1e9:.2f} GB >= L2)"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": (("lopa_lmhead_pair_kernel (CTA pairs, tcgen05.mma.cta_group::2 M=256, double-buffered TMEM accumulators)"
                                 if rows > 128 and os.environ.get("LOPA_LMH_SINGLE") != "1" else
                                 "lopa_lmhead_kernel (one CTA per SM, tcgen05.mma.cta_group::1)")
                                + " + Conf epilogue + its fold"),
                     "kernel_ms_mean": kern_ms,
                     "kernel_timing": f"CUDA events around {K} back-to-back LMHead calls (GEMM+epilogue kernel and fold kernel)",
                     "alg_flops_per_launch": flops,
                     "weight_stream_gbs": V * Kd * 2 / (kern_ms / 1000.0) / 1e9,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16, back to back)"},
        "clocks": clk.summary(),
        "gpu_launches": K * 3,
        "e2e": {"value": K2 / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": K2},
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    return 0


def run_lmhead_bp(args):
    """--config lmhead-* on N GPUs (branch parallelism, lopa_bp_step_lmhead): every rank runs the
    LM head + Conf on its own branches' hidden-state rows (b_loc * W of them) and the step's
    exchange and decisions; the same random-init output projection on every rank."""
    from paper_2512_16229_b200 import lopa
    import ctypes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    V, W, k, tau, Kd = CFG["V"], CFG["W"], CFG["k"], CFG["tau"], CFG["K"]
    st, tok, msk, nb, full, bufs, rows_total, _ = build_workload(lopa, dev, V, W, k, tau, CFG["seed"], 1)
    del full, bufs
    bp, p2p_note = make_branch_parallel(lopa, st, rank, world, dist, dev)
    b_loc, lo, hi = bp.b_loc, bp.lo, bp.hi
    rows_local = b_loc * W
    g = torch.Generator(device=dev).manual_seed(CFG["seed"])
    NW = 2
    Ws = [(torch.randn(V, Kd, device=dev, generator=g) / Kd ** 0.5).to(torch.bfloat16) for _ in range(NW)]
    NH = 8
    rows = (k + 1) * W
    Hs = []
    for _ in range(NH):
        full_h = (torch.randn(rows, Kd, device=dev, generator=g) * 1.5).to(torch.bfloat16)
        loc = torch.zeros(rows_local, Kd, dtype=torch.bfloat16, device=dev)
        n_own = max(0, min(hi, k + 1) - lo) * W
        if n_own:
            loc[:n_own] = full_h[lo * W: lo * W + n_own]
        Hs.append(loc)
    L = lopa.lib()
    stream = torch.cuda.current_stream(dev)
    sptr = ctypes.c_void_p(stream.cuda_stream)
    lmh_ws = torch.empty(L.lopa_lmhead_workspace_bytes(rows_local), dtype=torch.uint8, device=dev)
    P_ = lopa._p
    argv = []
    for _ in range(NH):
        a = st.args(Hs[0], nb, tok, msk)
        a.conf, a.argmax = bp.conf.data_ptr(), bp.argmax.data_ptr()
        a.workspace, a.workspace_bytes = bp.ws.data_ptr(), bp.ws.numel()
        a.scores = bp.scores.data_ptr()
        argv.append(a)
    rec = None if bp.p2p else P_(bp.records)

    def launch(i, h=None):
        s_ = L.lopa_bp_step_lmhead(bp.h, ctypes.byref(argv[i % NH]), b_loc, P_(Hs[i % NH] if h is None else h),
                                   Kd, P_(Ws[i % NW]), Kd, Kd, rec, P_(lmh_ws), lmh_ws.numel(), sptr)
        if s_:
            raise lopa.LopaError(f"lopa_bp_step_lmhead status {s_}")

    if dist:
        dist.barrier()
    for i in range(args.warmup):
        launch(i)
    torch.cuda.synchronize()
    if int(st.out.status.item()) != 0:
        raise lopa.LopaError(f"device status {int(st.out.status.item())} after the warm-up")
    K = args.steps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        head_start(stream)
        t0.record(stream)
        for i in range(K):
            launch(i)
        t1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    el_ms = t0.elapsed_time(t1)
    if dist:
        t = torch.tensor([el_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el_ms = float(t.item())
    if int(st.out.status.item()) != 0:
        raise lopa.LopaError(f"device status {int(st.out.status.item())}")
    # e2e: this rank's hidden-state shard from pinned host memory, results to the host
    hh = Hs[0].cpu().pin_memory()
    d_h = torch.empty_like(Hs[0])
    o = st.out
    h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory()
             for t in (o.winner, o.next_tokens, o.next_mask, o.n_next, o.status)]
    K2 = max(3, min(K, 200))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(K2):
        d_h.copy_(hh, non_blocking=True)
        launch(i, d_h)
        for hbuf, dsrc in zip(h_out, (o.winner, o.next_tokens, o.next_mask, o.n_next, o.status)):
            hbuf.copy_(dsrc, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    h2d = hh.numel() * 2
    d2h = sum(t.numel() * t.element_size() for t in h_out)
    flops = 2.0 * rows_local * Kd * V
    pk = peaks()
    peak = float(pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", 1416.0)))
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        h_full = torch.cat([Hs[0]], 0)
        cpu = cpu_baseline_lmhead(h_full.view(torch.int16).cpu().numpy().view(np.uint16),
                                  Ws[0].view(torch.int16).cpu().numpy().view(np.uint16), rows_local)
    if dist:
        dist.barrier()
    line = {
        "metric": METRIC, "value": K / (el_ms / 1000.0), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": el_ms / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init output projection, Gaussian hidden states; transformer body out of scope)",
        "config": {"workload": CFG["name"], "rows": rows, "rows_this_rank": rows_local,
                   "masked_rows": rows_total, "hidden": Kd,
                   "parallelism": f"bp{world}" + ("-p2p" if bp.p2p else ""),
                   "bp_exchange": ("peer memory, fused into K2" if bp.p2p else "NCCL all-gather")
                                  + ("" if p2p_note is None else f" [{p2p_note}]"),
                   "l2": f"{NW} rotating weight copies ({NW * V * Kd * 2 / 1e9:.2f} GB >= L2)"},
        "roofline": {"bound": "tensor", "achieved": flops / (el_ms / K / 1000.0) / 1e12, "peak": peak,
                     "unit": "TFLOP/s", "frac": flops / (el_ms / K / 1000.0) / 1e12 / peak, "traffic": None,
                     "kernel": "the whole BP step (LM head + Conf on this rank's rows, exchange, decisions)",
                     "alg_flops_per_launch": flops,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16, back to back)"},
        "clocks": clk.summary(),
        "gpu_launches": K * (2 * ((rows_local + 255) // 256) + (1 if bp.p2p else 2)),
        "e2e": {"value": K2 / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": K2, "note": "each rank: its hidden-state shard H2D, results D2H; max over ranks"},
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    bp.close()
    if dist:
        dist.destroy_process_group()
    return 0


def cpu_baseline_lmhead(h16, w16, rows, budget_s=12.0):
    """The NEXT-4 oracle (fp64 logits of bf16 inputs, Conf) on a bounded row sample, one BLAS
    thread, scaled to steps/s for `rows` rows (the decisions' cost is negligible next to the
    projection).  h16 / w16: bf16 bit patterns (uint16) on the host."""
    from oracle import lmhead_oracle as LO
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        n = 0
        while n < rows and (time.perf_counter() - t0) < budget_s:
            LO.lmhead_confidence(h16, w16, [n])
            n += 1
        dt = time.perf_counter() - t0
    return {"value": n / dt / rows, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{n} of {rows} rows (fp64 logits over V x K, Conf) in {dt:.1f} s, scaled to one step; NumPy 1 thread"}


def run_reference_lmhead(args):
    """Reference arm for --config lmhead-dream: the fp64 oracle on a bounded row sample."""
    import syngen
    V, W, k, Kd = CFG["V"], CFG["W"], CFG["k"], CFG["K"]
    rows = (k + 1) * W
    h16, w16, _ = syngen.lmhead_inputs(CFG["seed"], rows, Kd, V)
    cb = cpu_baseline_lmhead(h16, w16, rows, budget_s=20.0)
    value = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SYN-LMH seeded hidden states and output projection)",
            "config": {"workload": CFG["name"], "rows": rows, "hidden": Kd},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="lopa", choices=["lopa", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="dream", choices=sorted(CONFIGS))
    # overrides of the selected config (SPEC.md:493's --k/--W/--V/--tau/--seed)
    ap.add_argument("--k", type=int, default=None, help="lookahead branches")
    ap.add_argument("--W", type=int, default=None, help="window (block) length")
    ap.add_argument("--V", type=int, default=None, help="vocabulary size")
    ap.add_argument("--tau", type=float, default=None, help="Eq. 1 threshold")
    ap.add_argument("--seed", type=int, default=None, help="SYN-D2F seed")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    CFG.update(V=c["V"], W=c["W"], k=c["k"], tau=c["tau"], name=c["name"])
    CFG["loop_blocks"] = c.get("loop_blocks")
    CFG["d2f_len"] = c.get("d2f_len")
    if c.get("seed") is not None:
        CFG["seed"] = c["seed"]
    for key in ("k", "tau", "seed"):
        if getattr(args, key) is not None:
            CFG[key] = getattr(args, key)
    if args.V is not None:
        CFG["V"] = args.V
    if args.W is not None:
        CFG["W"] = args.W
    if any(getattr(args, x) is not None for x in ("k", "tau", "seed", "V", "W")):
        CFG["name"] += f" [overridden: V={CFG['V']} W={CFG['W']} k={CFG['k']} tau={CFG['tau']} seed={CFG['seed']}]"
    if args.warmup < 3:
        args.warmup = 3
    CFG["K"] = c.get("K")
    if args.impl == "reference":
        return run_reference(args)
    if CFG["K"]:
        return run_lmhead(args)
    if CFG["loop_blocks"]:
        return run_loop(args)
    if CFG["d2f_len"]:
        return run_d2f(args)
    return run_lopa(args)


if __name__ == "__main__":
    sys.exit(main())
