"""Thin ctypes binding of liblopa (include/liblopa.h).  Argument marshalling only: every step of
the LoPA verify path runs in the library's sm_100a kernels.  PyTorch provides device memory,
streams and process groups.  There is no CPU fallback: if liblopa.so is missing or the device is
not a B200 (sm_100), calls raise.

Names follow the paper (arXiv 2512.16229): Conf, Eq. 1 anchor fill,
lookahead spawn (Alg. 1 step 2), Eq. 2 branch confidence + select.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liblopa.so")
if os.environ.get("LOPA_LIB_VARIANT"):   # tuning builds (paper_2512_16229_b200/build.py --variant)
    LIB_PATH = os.path.join(_PKG, f"liblopa_{os.environ['LOPA_LIB_VARIANT']}.so")

LOPA_OK = 0
METRIC_MEAN = 0            # Eq. 2
METRIC_SLIDING_MIN = 1     # P:204 sliding window
METRIC_BOTTOM_FRACTION = 2 # P:204 least-confident segment
DEV_EMPTY_MASK = 1
DEV_NONFINITE = 2
DEV_PEER_TIMEOUT = 4
IPC_HANDLE_BYTES = 64
MAX_WINDOW = 256
MAX_BRANCHES = 32
MAX_ROWS = 4096
UNIQUE_ID_BYTES = 128

_c_void_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_f32 = ctypes.c_float
_size = ctypes.c_size_t


class LopaError(RuntimeError):
    pass


class StepArgs(ctypes.Structure):
    """Mirror of lopa_step_args_t (include/liblopa.h)."""
    _fields_ = [
        ("logits", _c_void_p), ("ld", _i64), ("vocab", _i32), ("window", _i32),
        ("max_branches", _i32), ("n_branches", _c_void_p), ("branch_tokens", _c_void_p),
        ("branch_mask", _c_void_p), ("k", _i32), ("tau", _f32),
        ("conf", _c_void_p), ("argmax", _c_void_p), ("scores", _c_void_p), ("winner", _c_void_p),
        ("next_tokens", _c_void_p), ("next_mask", _c_void_p), ("lookahead_pos", _c_void_p),
        ("n_branches_next", _c_void_p), ("dev_status", _c_void_p),
        ("workspace", _c_void_p), ("workspace_bytes", _size),
        ("metric", _i32), ("metric_param", _f32), ("tau_pos", _c_void_p),
        ("window_dev", _c_void_p),
    ]


_SIGS = {
    "lopa_version": (_i32, []),
    "lopa_status_string": (ctypes.c_char_p, [_i32]),
    "lopa_last_cuda_error": (ctypes.c_char_p, []),
    "lopa_set_logits_prefetch": (_i32, [_i32]),
    "lopa_debug_k1_attrs": (_i32, [ctypes.c_void_p]),
    "lopa_debug_check_read": (_i32, [ctypes.c_void_p]),
    "lopa_d2f_init": (_i32, [_c_void_p, _c_void_p]),
    "lopa_while_begin": (_i32, [_c_void_p, _c_void_p, _i32, _i32, _c_void_p]),
    "lopa_while_end": (_i32, [_c_void_p]),
    "lopa_while_launch": (_i32, [_c_void_p, _c_void_p]),
    "lopa_while_iterations": (_i32, [_c_void_p, _c_void_p]),
    "lopa_while_destroy": (None, [_c_void_p]),
    "lopa_syn_generate_dev": (_i32, [ctypes.c_uint64, _i32, _i32, _i64, _i32, _i32, _c_void_p, _i32,
                                     _c_void_p, _c_void_p, _i32, _c_void_p, _c_void_p]),
    "lopa_d2f_update": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "lopa_d2f_syn_forward": (_i32, [ctypes.c_uint64, _i32, _i64, _i32, _c_void_p, _c_void_p, _c_void_p]),
    "lopa_workspace_bytes": (_size, [_i32, _i32]),
    "lopa_num_segments": (_i32, [_i32]),
    "lopa_confidence": (_i32, [_c_void_p, _i64, _i32, _i32, _c_void_p, _c_void_p, _c_void_p,
                               _c_void_p, _c_void_p, _size, _c_void_p]),
    "lopa_debug_reduce_only": (_i32, [_c_void_p, _i64, _i32, _i32, _c_void_p, _c_void_p,
                                      _c_void_p, _size, _c_void_p]),
    "lopa_anchor_fill": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i32, _f32,
                                _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "lopa_anchor_fill_ex": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i32, _f32, _c_void_p,
                                   _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "lopa_spawn_branches": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p, _i32, _i32,
                                   _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "lopa_verify_select": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i32, _i32, _c_void_p,
                                  _c_void_p, _c_void_p]),
    "lopa_verify_select_ex": (_i32, [_c_void_p, _c_void_p, _c_void_p, _i32, _i32, _i32, _f32,
                                     _c_void_p, _c_void_p, _c_void_p]),
    "lopa_step": (_i32, [ctypes.POINTER(StepArgs), _c_void_p]),
    "lopa_bp_record_bytes": (_size, [_i32, _i32]),
    "lopa_bp_local": (_i32, [ctypes.POINTER(StepArgs), _i32, _i32, _c_void_p, _c_void_p]),
    "lopa_bp_finish": (_i32, [ctypes.POINTER(StepArgs), _i32, _i32, _c_void_p, _c_void_p]),
    "lopa_bp_get_unique_id": (_i32, [_c_void_p]),
    "lopa_bp_create": (_i32, [_c_void_p, _i32, _i32, _i32, ctypes.POINTER(_c_void_p)]),
    "lopa_bp_step": (_i32, [_c_void_p, ctypes.POINTER(StepArgs), _i32, _c_void_p, _c_void_p]),
    "lopa_bp_check": (_i32, [_c_void_p]),
    "lopa_bp_p2p_alloc": (_i32, [_c_void_p, _i32, _i32, _size, _c_void_p]),
    "lopa_bp_payload_slots": (_c_void_p, [_c_void_p, _i32]),
    "lopa_bp_commit_winner_p2p": (_i32, [_c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "lopa_bp_p2p_open": (_i32, [_c_void_p, _c_void_p]),
    "lopa_bp_step_p2p": (_i32, [_c_void_p, ctypes.POINTER(StepArgs), _i32, _c_void_p]),
    "lopa_bp_step_lmhead": (_i32, [_c_void_p, ctypes.POINTER(StepArgs), _i32, _c_void_p, _i64,
                                   _c_void_p, _i64, _i32, _c_void_p, _c_void_p, _size, _c_void_p]),
    "lopa_bp_commit_winner": (_i32, [_c_void_p, _c_void_p, _i32, _c_void_p, _size, _c_void_p, _c_void_p]),
    "lopa_bp_destroy": (None, [_c_void_p]),
    "lopa_debug_timeline": (_i32, [_c_void_p, _i32]),
    "lopa_debug_ldg_timeline": (_i32, [_c_void_p, _i32]),
    "lopa_debug_k1_timeline": (_i32, [_c_void_p, _i32]),
    "lopa_debug_chain_timeline": (_i32, [_c_void_p, _i32]),
    "lopa_profile_enable": (_i32, [_i32]),
    "lopa_profile_read": (_i32, [ctypes.POINTER(ctypes.c_float), _i32, ctypes.POINTER(_i32)]),
    "lopa_syn_generate": (_i32, [_u64, _i32, _i32, _i64, _i32, _i32, _c_void_p, _c_void_p, _i32,
                                 _c_void_p, _c_void_p]),
    "lopa_lmhead_workspace_bytes": (_size, [_i32]),
    "lopa_lmhead_confidence": (_i32, [_c_void_p, _i64, _c_void_p, _i64, _i32, _i32, _i32, _c_void_p,
                                      _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size, _c_void_p]),
    "lopa_step_lmhead": (_i32, [ctypes.POINTER(StepArgs), _c_void_p, _i64, _c_void_p, _i64, _i32,
                                _c_void_p, _size, _c_void_p]),
}
EXPORTS = tuple(_SIGS)

_lib = None


def lib() -> ctypes.CDLL:
    """Load liblopa.so (built in-tree by paper_2512_16229_b200.build).  Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LopaError(f"{LIB_PATH} is not built; run `python -m paper_2512_16229_b200.build` "
                            "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int, what: str):
    if st != LOPA_OK:
        msg = lib().lopa_status_string(st).decode()
        if st == 3:  # LOPA_ERR_CUDA: the runtime's own message
            msg += ": " + lib().lopa_last_cuda_error().decode()
        raise LopaError(f"{what}: liblopa status {st} ({msg})")


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise LopaError("liblopa takes CUDA tensors (no CPU fallback)")


def _u8(mask: torch.Tensor) -> torch.Tensor:
    return mask.view(torch.uint8) if mask.dtype == torch.bool else mask


def num_segments(vocab: int) -> int:
    return int(lib().lopa_num_segments(vocab))


def workspace_bytes(max_rows: int, vocab: int) -> int:
    return int(lib().lopa_workspace_bytes(max_rows, vocab))


def new_workspace(max_rows: int, vocab: int, device) -> torch.Tensor:
    """Zeroed device workspace (zero once before first use; the library keeps its counters and
    the partial epoch in it, liblopa.h conventions)."""
    return torch.zeros(workspace_bytes(max_rows, vocab), dtype=torch.uint8, device=device)


def new_status(device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


# ----------------------------------------------------------------------------- a1
def confidence(logits: torch.Tensor, vocab: int | None = None, row_mask: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None, status: torch.Tensor | None = None):
    """Conf and greedy token of each row of bf16 logits [n_rows][ld].

    Returns (conf f32[n_rows], argmax i32[n_rows], status i32[1]); rows not selected by
    row_mask hold NaN / -1."""
    _need_cuda(logits, row_mask)
    if logits.dtype != torch.bfloat16 or logits.dim() != 2 or logits.stride(1) != 1:
        raise LopaError("logits must be a 2-D bf16 tensor with unit inner stride")
    n_rows, ld = logits.shape[0], logits.stride(0)
    vocab = logits.shape[1] if vocab is None else vocab
    dev = logits.device
    conf = torch.full((n_rows,), float("nan"), dtype=torch.float32, device=dev)
    amax = torch.full((n_rows,), -1, dtype=torch.int32, device=dev)
    status = new_status(dev) if status is None else status
    if workspace is None:
        workspace = new_workspace(max(n_rows, 1), vocab, dev)
    rm = None if row_mask is None else _u8(row_mask).contiguous()
    _check(lib().lopa_confidence(_p(logits), ld, n_rows, vocab, _p(rm), _p(conf), _p(amax),
                                 _p(status), _p(workspace), workspace.numel(), _stream(dev)),
           "lopa_confidence")
    return conf, amax, status


# ----------------------------------------------------------------------------- NEXT-4
class LMHead:
    """LM-head projection with Conf fused into the GEMM epilogue (tcgen05): conf / argmax of
    each row of ``hidden`` (bf16 [rows][K]) against ``weight`` (bf16 [V][K]) without
    materialising the logits.  Owns its workspace; rows <= max_rows <= 4096 (256 rows per pass
    over the weights), K % 64 == 0."""

    def __init__(self, weight: torch.Tensor, max_rows: int = 256):
        _need_cuda(weight)
        if weight.dtype != torch.bfloat16 or weight.dim() != 2 or weight.stride(1) != 1:
            raise LopaError("weight must be a 2-D bf16 tensor [V][K] with unit inner stride")
        self.weight = weight
        self.vocab, self.hidden_dim = weight.shape
        dev = weight.device
        self.ws = torch.empty(lib().lopa_lmhead_workspace_bytes(max_rows), dtype=torch.uint8, device=dev)
        self.status = new_status(dev)
        self.conf = torch.empty(max_rows, dtype=torch.float32, device=dev)
        self.argmax = torch.empty(max_rows, dtype=torch.int32, device=dev)

    def __call__(self, hidden: torch.Tensor, row_mask: torch.Tensor | None = None):
        _need_cuda(hidden, row_mask)
        if hidden.dtype != torch.bfloat16 or hidden.dim() != 2 or hidden.stride(1) != 1:
            raise LopaError("hidden must be a 2-D bf16 tensor [rows][K] with unit inner stride")
        rows = hidden.shape[0]
        if hidden.shape[1] != self.hidden_dim or rows > self.conf.numel():
            raise LopaError("hidden shape does not match the weight / max_rows")
        _check(lib().lopa_lmhead_confidence(_p(hidden), hidden.stride(0), _p(self.weight),
                                            self.weight.stride(0), rows, self.hidden_dim, self.vocab,
                                            _p(None if row_mask is None else _u8(row_mask).contiguous()),
                                            _p(self.conf), _p(self.argmax), _p(self.status),
                                            _p(self.ws), self.ws.numel(), _stream(hidden.device)),
               "lopa_lmhead_confidence")
        return self.conf[:rows], self.argmax[:rows], self.status

    def step(self, stepper: "Stepper", hidden: torch.Tensor, n_branches, branch_tokens, branch_mask):
        """lopa_step from the verify forward's hidden states (bf16 [max_br][W][K] or
        [max_br*W][K]): fused LM-head a1, then the stepper's a2-a4.  Returns stepper.out."""
        _need_cuda(hidden, n_branches, branch_tokens, branch_mask)
        if stepper.vocab != self.vocab:
            raise LopaError("stepper vocab does not match the LM-head weight")
        h = hidden.reshape(-1, hidden.shape[-1])
        if h.dtype != torch.bfloat16 or h.stride(1) != 1 or h.shape[0] != stepper.max_branches * stepper.window:
            raise LopaError("hidden must be bf16 [max_branches * window][K] with unit inner stride")
        a = stepper.args(h, n_branches, branch_tokens, branch_mask)
        _check(lib().lopa_step_lmhead(ctypes.byref(a), _p(h), h.stride(0), _p(self.weight),
                                      self.weight.stride(0), self.hidden_dim, _p(self.ws),
                                      self.ws.numel(), _stream(h.device)), "lopa_step_lmhead")
        return stepper.out


# ----------------------------------------------------------------------------- a3
def anchor_fill(conf, argmax, tokens, mask, tau: float, status=None, tau_pos=None):
    """Eq. 1 + Alg. 1 step 1.  tau_pos: optional per-position thresholds
    (float32 [W], the D2F window).  Returns (tokens_B0, mask_B0, status)."""
    _need_cuda(conf, argmax, tokens, mask, tau_pos)
    W = mask.numel()
    dev = mask.device
    tok_out = torch.empty(W, dtype=torch.int32, device=dev)
    msk_out = torch.empty(W, dtype=torch.uint8, device=dev)
    status = new_status(dev) if status is None else status
    tp = None if tau_pos is None else tau_pos.contiguous()
    _check(lib().lopa_anchor_fill_ex(_p(conf.contiguous()), _p(argmax.contiguous()),
                                     _p(tokens.contiguous()), _p(_u8(mask).contiguous()), W, tau,
                                     _p(tp), _p(tok_out), _p(msk_out), _p(status), _stream(dev)),
           "lopa_anchor_fill_ex")
    return tok_out, msk_out, status


# ----------------------------------------------------------------------------- a4
def spawn_branches(conf, argmax, tokens_b0, mask_b0, k: int):
    """Alg. 1 step 2.  Returns (branch_tokens[k+1][W], branch_mask[k+1][W],
    lookahead_pos[k], n_branches[1]); rows >= n_branches are zero."""
    _need_cuda(conf, argmax, tokens_b0, mask_b0)
    W = mask_b0.numel()
    dev = mask_b0.device
    bt = torch.zeros((k + 1, W), dtype=torch.int32, device=dev)
    bm = torch.zeros((k + 1, W), dtype=torch.uint8, device=dev)
    look = torch.full((max(k, 1),), -1, dtype=torch.int32, device=dev)
    nb = torch.zeros(1, dtype=torch.int32, device=dev)
    _check(lib().lopa_spawn_branches(_p(conf.contiguous()), _p(argmax.contiguous()),
                                     _p(tokens_b0.contiguous()), _p(_u8(mask_b0).contiguous()),
                                     W, k, _p(bt), _p(bm), _p(look), _p(nb), _stream(dev)),
           "lopa_spawn_branches")
    return bt, bm, look[:k], nb


# ----------------------------------------------------------------------------- a2
def verify_select(conf, branch_mask, n_branches, metric: int = METRIC_MEAN, param: float = 0.0):
    """Eq. 2 (or a P:204 variant) + select.  conf/branch_mask [max_br][W];
    n_branches device int32[1].  Returns (scores f32[max_br], winner i32[1])."""
    _need_cuda(conf, branch_mask, n_branches)
    max_br, W = branch_mask.shape
    dev = branch_mask.device
    scores = torch.empty(max_br, dtype=torch.float32, device=dev)
    winner = torch.zeros(1, dtype=torch.int32, device=dev)
    if metric == METRIC_MEAN:
        _check(lib().lopa_verify_select(_p(conf.contiguous()), _p(_u8(branch_mask).contiguous()),
                                        _p(n_branches), max_br, W, _p(scores), _p(winner),
                                        _stream(dev)),
               "lopa_verify_select")
    else:
        _check(lib().lopa_verify_select_ex(_p(conf.contiguous()), _p(_u8(branch_mask).contiguous()),
                                           _p(n_branches), max_br, W, metric, param, _p(scores),
                                           _p(winner), _stream(dev)),
               "lopa_verify_select_ex")
    return scores, winner


# ----------------------------------------------------------------------------- fused step
@dataclass
class StepOutputs:
    conf: torch.Tensor          # f32 [max_br][W] (NaN where not reduced)
    argmax: torch.Tensor        # i32 [max_br][W]
    scores: torch.Tensor        # f32 [max_br]
    winner: torch.Tensor        # i32 [1]
    next_tokens: torch.Tensor   # i32 [k+1][W]
    next_mask: torch.Tensor     # u8  [k+1][W]
    lookahead: torch.Tensor     # i32 [max(k,1)]
    n_next: torch.Tensor        # i32 [1]
    status: torch.Tensor        # i32 [1]


class Stepper:
    """Owns the workspace and output buffers of `lopa_step` for one (V, W, max_br, k, tau)
    configuration, so that repeated steps allocate nothing (CUDA-graph friendly)."""

    def __init__(self, vocab: int, window: int, max_branches: int, k: int, tau: float, device,
                 ld: int | None = None, metric: int = METRIC_MEAN, metric_param: float = 0.0,
                 tau_pos: torch.Tensor | None = None):
        self.vocab, self.window, self.max_branches, self.k, self.tau = vocab, window, max_branches, k, tau
        self.metric, self.metric_param = metric, metric_param
        self.tau_pos = tau_pos  # optional device float32 [window] (D2F per-position thresholds)
        self.ld = ld if ld is not None else ((vocab + 7) // 8) * 8
        self.device = torch.device(device)
        d = self.device
        self.ws = new_workspace(max_branches * window, vocab, d)
        self.out = StepOutputs(
            conf=torch.full((max_branches, window), float("nan"), dtype=torch.float32, device=d),
            argmax=torch.full((max_branches, window), -1, dtype=torch.int32, device=d),
            scores=torch.empty(max_branches, dtype=torch.float32, device=d),
            winner=torch.zeros(1, dtype=torch.int32, device=d),
            next_tokens=torch.zeros((k + 1, window), dtype=torch.int32, device=d),
            next_mask=torch.zeros((k + 1, window), dtype=torch.uint8, device=d),
            lookahead=torch.full((max(k, 1),), -1, dtype=torch.int32, device=d),
            n_next=torch.zeros(1, dtype=torch.int32, device=d),
            status=new_status(d),
        )

    def args(self, logits, n_branches, branch_tokens, branch_mask) -> StepArgs:
        o = self.out
        return StepArgs(
            logits=logits.data_ptr(), ld=logits.stride(-2), vocab=self.vocab, window=self.window,
            max_branches=self.max_branches, n_branches=n_branches.data_ptr(),
            branch_tokens=branch_tokens.data_ptr(), branch_mask=_u8(branch_mask).data_ptr(),
            k=self.k, tau=self.tau, conf=o.conf.data_ptr(), argmax=o.argmax.data_ptr(),
            scores=o.scores.data_ptr(), winner=o.winner.data_ptr(),
            next_tokens=o.next_tokens.data_ptr(), next_mask=o.next_mask.data_ptr(),
            lookahead_pos=o.lookahead.data_ptr(), n_branches_next=o.n_next.data_ptr(),
            dev_status=o.status.data_ptr(), workspace=self.ws.data_ptr(),
            workspace_bytes=self.ws.numel(), metric=self.metric, metric_param=self.metric_param,
            tau_pos=None if self.tau_pos is None else self.tau_pos.data_ptr())

    def _validate(self, logits, n_branches, branch_tokens, branch_mask):
        _need_cuda(logits, n_branches, branch_tokens, branch_mask)
        if logits.dtype != torch.bfloat16 or logits.stride(-1) != 1:
            raise LopaError("logits must be bf16 with unit inner stride")
        rows = logits.numel() // logits.shape[-1]
        if rows < self.max_branches * self.window or not logits.is_contiguous():
            raise LopaError("logits must be contiguous [max_branches][window][ld]")
        if branch_tokens.dtype != torch.int32 or tuple(branch_tokens.shape) != (self.max_branches, self.window):
            raise LopaError("branch_tokens must be int32 [max_branches][window]")
        if tuple(branch_mask.shape) != (self.max_branches, self.window):
            raise LopaError("branch_mask must be [max_branches][window]")

    def step(self, logits, n_branches, branch_tokens, branch_mask, validate: bool = True) -> StepOutputs:
        """One fused verify step (a1 -> a2 -> a3 -> a4) in one kernel launch."""
        if validate:
            self._validate(logits, n_branches, branch_tokens, branch_mask)
        a = self.args(logits, n_branches, branch_tokens, branch_mask)
        _check(lib().lopa_step(ctypes.byref(a), _stream(self.device)), "lopa_step")
        return self.out


def decode_block(forward, tokens0: torch.Tensor, mask0: torch.Tensor, k: int, tau: float, vocab: int,
                 stepper: "Stepper | None" = None, max_forwards: int | None = None):
    """Alg. 1 over one window: initial predict, then verify steps until the
    selected branch has no masked position (R21).  ``forward(branch_tokens[n][W],
    branch_mask[n][W], out=logits[n][W][ld])`` fills the bf16 logits of the n present branch
    states (the model).  Returns (tokens int32 [W] on the device, forwards); forwards =
    1 + verify passes.  One host read per iteration (the branch count)."""
    W = tokens0.numel()
    dev = tokens0.device
    st = stepper or Stepper(vocab, W, k + 1, k, tau, dev)
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=dev)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=dev)
    tok[0], msk[0] = tokens0.to(torch.int32), _u8(mask0)
    nb = torch.ones(1, dtype=torch.int32, device=dev)
    logits = torch.zeros((k + 1, W, st.ld), dtype=torch.bfloat16, device=dev)
    forwards, n = 0, 1
    while True:
        forward(tok[:n], msk[:n], out=logits[:n])
        out = st.step(logits, nb, tok, msk)
        forwards += 1
        n = int(out.n_next.item())
        if n == 0 or (max_forwards is not None and forwards >= max_forwards):
            return out.next_tokens[0].clone(), forwards
        tok.copy_(out.next_tokens)
        msk.copy_(out.next_mask)
        nb.copy_(out.n_next)


class StepLoopGraph:
    """`iters` Alg. 1 iterations captured in ONE CUDA graph (no tracing compiler, no host
    round trip between steps): each iteration is a lopa_step on logits[i % len(logits)]
    followed by a device copy of the spawned tables into the step's input tables.  The logits
    buffers are the caller's (a model would write them between steps; the graph reads whatever
    they hold at replay).  replay() runs the whole loop; the stepper's outputs and the input
    tables then hold the last iteration's state (a complete block rests at its fixed point:
    n_branches = 0 passes row 0 through)."""

    def __init__(self, stepper: Stepper, logits: list, n_branches, branch_tokens, branch_mask,
                 iters: int):
        _need_cuda(n_branches, branch_tokens, branch_mask, *logits)
        self.s, self.logits, self.iters = stepper, logits, iters
        self.nb, self.tok, self.msk = n_branches, branch_tokens, _u8(branch_mask)
        for lg in logits:
            stepper._validate(lg, n_branches, branch_tokens, self.msk)
        self._args = [stepper.args(lg, n_branches, branch_tokens, self.msk) for lg in logits]
        # warm up outside the capture (kernel attributes, lazy module loading) on a snapshot of
        # the caller's tables, restored afterwards: the first replay starts from the caller's state
        snap = (self.tok.clone(), self.msk.clone(), self.nb.clone())
        self._iteration(0)
        self.tok.copy_(snap[0])
        self.msk.copy_(snap[1])
        self.nb.copy_(snap[2])
        torch.cuda.synchronize(stepper.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            for i in range(iters):
                self._iteration(i)

    def _iteration(self, i):
        o = self.s.out
        a = self._args[i % len(self._args)]
        _check(lib().lopa_step(ctypes.byref(a), _stream(self.s.device)), "lopa_step")
        k1 = o.next_tokens.shape[0]
        self.tok[:k1].copy_(o.next_tokens)
        self.msk[:k1].copy_(o.next_mask)
        self.nb.copy_(o.n_next)

    def replay(self):
        self.graph.replay()
        return self.s.out


class WhileGraph:
    """A CUDA graph whose body repeats ON THE DEVICE until a condition word stops it (conditional
    WHILE node, lopa_while_*): ``body()`` is issued once, captured into the loop body (it must not
    allocate or synchronise); after every iteration the loop continues while ``cond_word`` (a
    device int32) is non-zero (until_zero=True) or zero (until_zero=False), at most max_iters
    times.  launch() runs the whole loop with no host involvement."""

    def __init__(self, body, cond_word: torch.Tensor, until_zero: bool = True, max_iters: int = 1 << 20):
        _need_cuda(cond_word)
        self.device = cond_word.device
        self.stream = torch.cuda.Stream(self.device)
        torch.cuda.synchronize(self.device)
        h = ctypes.c_void_p()
        _check(lib().lopa_while_begin(ctypes.c_void_p(self.stream.cuda_stream), _p(cond_word),
                                      1 if until_zero else 0, max_iters, ctypes.byref(h)), "lopa_while_begin")
        self.h = h
        try:
            with torch.cuda.stream(self.stream):
                body()
        finally:
            st = lib().lopa_while_end(h)
        _check(st, "lopa_while_end")

    def launch(self):
        """Run the loop on the current stream (asynchronous)."""
        _check(lib().lopa_while_launch(self.h, _stream(self.device)), "lopa_while_launch")

    def iterations(self) -> int:
        n = _i32(0)
        torch.cuda.synchronize(self.device)
        _check(lib().lopa_while_iterations(self.h, ctypes.byref(n)), "lopa_while_iterations")
        return n.value

    def close(self):
        if getattr(self, "h", None):
            lib().lopa_while_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def syn_generate_dev(seed: int, block: int, vocab: int, branch_tokens, branch_mask, n_branches_dev,
                     out: torch.Tensor, extras: int = 0, branch_base: int = 0):
    """SYN-D2F logits for the branches present, the count read on the device (harness); the
    tables / out hold global branches [branch_base, branch_base + rows)."""
    mb, W = branch_mask.shape
    _check(lib().lopa_syn_generate_dev(seed & ((1 << 64) - 1), block, vocab, out.stride(-2), W, mb,
                                       _p(n_branches_dev), branch_base, _p(branch_tokens),
                                       _p(_u8(branch_mask)), extras, _p(out), _stream(out.device)),
           "lopa_syn_generate_dev")


class DecodeBlockGraph:
    """Alg. 1 over one window as ONE device-terminated CUDA graph (WhileGraph): each iteration is
    the harness forward of the present branches (syn_generate_dev, the model stand-in), one
    lopa_step and the device copy of the spawned tables; the loop ends on the device when the
    selected branch is complete (n_branches_next = 0, R21).  run(tokens0, mask0) -> tokens;
    forwards() = iterations of the last run."""

    def __init__(self, stepper: "Stepper", seed: int, block: int, extras: int = 0):
        st = stepper
        self.s, self.seed, self.block, self.extras = st, seed, block, extras
        d, W, mb = st.device, st.window, st.max_branches
        self.tok = torch.zeros((mb, W), dtype=torch.int32, device=d)
        self.msk = torch.zeros((mb, W), dtype=torch.uint8, device=d)
        self.nb = torch.ones(1, dtype=torch.int32, device=d)
        self.logits = torch.zeros((mb, W, st.ld), dtype=torch.bfloat16, device=d)
        self._args = st.args(self.logits, self.nb, self.tok, self.msk)
        # warm-up outside the capture (kernel attributes, lazy module loading), then restore
        self._body()
        torch.cuda.synchronize(d)
        self.graph = WhileGraph(self._body, st.out.n_next, until_zero=True, max_iters=4 * W + 4)

    def _body(self):
        st, o = self.s, self.s.out
        syn_generate_dev(self.seed, self.block, st.vocab, self.tok, self.msk, self.nb, self.logits, self.extras)
        _check(lib().lopa_step(ctypes.byref(self._args), _stream(st.device)), "lopa_step")
        k1 = o.next_tokens.shape[0]
        self.tok[:k1].copy_(o.next_tokens)
        self.msk[:k1].copy_(o.next_mask)
        self.nb.copy_(o.n_next)

    def run(self, tokens0: torch.Tensor, mask0: torch.Tensor, block: int | None = None) -> torch.Tensor:
        self.tok.zero_()
        self.msk.zero_()
        self.tok[0].copy_(tokens0.to(torch.int32))
        self.msk[0].copy_(_u8(mask0))
        self.nb.fill_(1)
        self.graph.launch()
        return self.tok[0]

    def forwards(self) -> int:
        return self.graph.iterations()


class DecodeBlockGraphBP:
    """DecodeBlockGraph branch-parallel: this rank's iteration = the harness forward of ITS OWN
    present branches (syn_generate_dev on global branches [lo, hi), count read on the device),
    lopa_bp_step (local reduction and record, the NCCL all-gather, the replicated select /
    anchor / spawn) and the table copies, in one device-terminated graph per block (every rank
    holds the same tables, so every rank's loop stops at the same iteration).  Either exchange:
    the NCCL all-gather is captured as a graph node, the peer-memory step keeps its epoch on the
    device."""

    def __init__(self, bp: "BranchParallel", seed: int, block: int, extras: int = 0):
        st = bp.s
        self.bp, self.s, self.seed, self.block, self.extras = bp, st, seed, block, extras
        d, W, mb = st.device, st.window, st.max_branches
        self.tok = torch.zeros((mb, W), dtype=torch.int32, device=d)
        self.msk = torch.zeros((mb, W), dtype=torch.uint8, device=d)
        self.nb = torch.ones(1, dtype=torch.int32, device=d)
        _, self.lo, self.hi, self.local = bp.ranks()[0]
        self._body()
        torch.cuda.synchronize(d)
        self.graph = WhileGraph(self._body, st.out.n_next, until_zero=True, max_iters=4 * W + 4)

    def _body(self):
        st, o = self.s, self.s.out
        if self.hi > self.lo:
            syn_generate_dev(self.seed, self.block, st.vocab, self.tok[self.lo:self.hi],
                             self.msk[self.lo:self.hi], self.nb, self.local[: self.hi - self.lo],
                             self.extras, branch_base=self.lo)
        self.bp.step(self.local, self.nb, self.tok, self.msk)
        k1 = o.next_tokens.shape[0]
        self.tok[:k1].copy_(o.next_tokens)
        self.msk[:k1].copy_(o.next_mask)
        self.nb.copy_(o.n_next)

    run = DecodeBlockGraph.run
    forwards = DecodeBlockGraph.forwards


# ----------------------------------------------------------------------------- measurement
def set_logits_prefetch(enabled: bool) -> bool:
    """lopa_set_logits_prefetch: allow (default) or forbid K1's first logits copy before the PDL
    wait (forbid it when the logits producer triggers its dependents early).  Returns the
    previous setting."""
    return bool(lib().lopa_set_logits_prefetch(1 if enabled else 0))


def profile_enable(max_records: int):
    """Record CUDA events around every K1 (vocabulary reduction) launch of the next calls."""
    _check(lib().lopa_profile_enable(max_records), "lopa_profile_enable")


def profile_read(max_records: int):
    """Synchronise and return the recorded K1 durations (ms); disables recording."""
    buf = (ctypes.c_float * max_records)()
    n = _i32(0)
    _check(lib().lopa_profile_read(buf, max_records, ctypes.byref(n)), "lopa_profile_read")
    return list(buf[: n.value])


# ----------------------------------------------------------------------------- harness
def syn_cv8(vocab: int) -> int:
    return 0 if vocab < 2 else int(round(8.0 * math.log(1.8 * (vocab - 1))))


def syn_generate(seed: int, block: int, vocab: int, branch_tokens, branch_mask, n_branches=None,
                 extras: int = 0, ld: int | None = None, out: torch.Tensor | None = None):
    """SYN-D2F logits (bf16 [n_branches][W][ld]) for the given branch states (harness only)."""
    _need_cuda(branch_tokens, branch_mask)
    nb_rows, W = branch_mask.shape
    n = nb_rows if n_branches is None else n_branches
    ld = ((vocab + 7) // 8) * 8 if ld is None else ld
    dev = branch_mask.device
    if out is None:
        out = torch.empty((n, W, ld), dtype=torch.bfloat16, device=dev)
    _check(lib().lopa_syn_generate(seed & ((1 << 64) - 1), block, vocab, ld, W, n,
                                   _p(branch_tokens.contiguous()), _p(_u8(branch_mask).contiguous()),
                                   extras, _p(out), _stream(dev)),
           "lopa_syn_generate")
    return out


# ----------------------------------------------------------------------------- BP (a5)
def bp_shard(max_branches: int, world: int, rank: int):
    """Branch-parallel partition: B_loc = ceil(max_branches / world); rank r owns
    global branches [r * B_loc, min((r + 1) * B_loc, max_branches))."""
    b_loc = -(-max_branches // world)
    lo = min(rank * b_loc, max_branches)
    hi = min(lo + b_loc, max_branches)
    return b_loc, lo, hi


def record_bytes(window: int, b_loc: int) -> int:
    return int(lib().lopa_bp_record_bytes(window, b_loc))


class BranchParallel:
    """One rank of a branch-parallel LoPA step over NCCL (one process per GPU).

    The NCCL unique id is created by rank 0 and shipped over the given torch process group."""

    def __init__(self, stepper: Stepper, rank: int, world: int, group=None, p2p: bool = False,
                 payload_bytes: int = 0):
        """p2p=True: exchange the records over peer memory (lopa_bp_step_p2p: CUDA IPC mappings
        of every rank's record buffer, NVLink stores + epoch flags) instead of ncclAllGather."""
        import torch.distributed as dist
        self.s, self.rank, self.world = stepper, rank, world
        self.b_loc, self.lo, self.hi = bp_shard(stepper.max_branches, world, rank)
        uid = torch.zeros(UNIQUE_ID_BYTES, dtype=torch.uint8)
        if rank == 0:
            buf = (ctypes.c_uint8 * UNIQUE_ID_BYTES)()
            _check(lib().lopa_bp_get_unique_id(buf), "lopa_bp_get_unique_id")
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        if world > 1:
            obj = [uid.tolist()]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = torch.tensor(obj[0], dtype=torch.uint8)
        raw = (ctypes.c_uint8 * UNIQUE_ID_BYTES)(*uid.tolist())
        h = ctypes.c_void_p()
        dev = stepper.device.index if stepper.device.index is not None else torch.cuda.current_device()
        _check(lib().lopa_bp_create(raw, rank, world, dev, ctypes.byref(h)), "lopa_bp_create")
        self.h = h
        W = stepper.window
        d = stepper.device
        self.rb = record_bytes(W, self.b_loc)
        self.records = torch.zeros(world * self.rb, dtype=torch.uint8, device=d)
        self.ws = new_workspace(self.b_loc * W, stepper.vocab, d)
        self.conf = torch.full((self.b_loc, W), float("nan"), dtype=torch.float32, device=d)
        self.argmax = torch.full((self.b_loc, W), -1, dtype=torch.int32, device=d)
        self.scores = torch.empty(world * self.b_loc, dtype=torch.float32, device=d)
        self.local = None  # this rank's logits buffer for decode_block_bp (allocated on first use)
        self.p2p = p2p
        self._payload_bytes = payload_bytes
        if p2p:
            hbuf = (ctypes.c_uint8 * IPC_HANDLE_BYTES)()
            _check(lib().lopa_bp_p2p_alloc(self.h, W, self.b_loc, payload_bytes, hbuf), "lopa_bp_p2p_alloc")
            mine = bytes(hbuf)
            if world > 1:
                allh = [None] * world
                dist.all_gather_object(allh, mine, group=group)
            else:
                allh = [mine]
            raw_all = (ctypes.c_uint8 * (IPC_HANDLE_BYTES * world))(*b"".join(allh))
            _check(lib().lopa_bp_p2p_open(self.h, raw_all), "lopa_bp_p2p_open")

    def ranks(self):
        """(rank, lo, hi, local logits buffer [b_loc][W][ld]) of this process's rank."""
        if self.local is None:
            self.local = torch.zeros((self.b_loc, self.s.window, self.s.ld), dtype=torch.bfloat16,
                                     device=self.s.device)
        return [(self.rank, self.lo, self.hi, self.local)]

    def step(self, *a) -> StepOutputs:
        """step(local_logits, n_branches, branch_tokens, branch_mask), or step(n_branches,
        branch_tokens, branch_mask) on the buffer of ranks().  local_logits: this rank's bf16
        [b_loc][W][ld]; the tables are the full replicated ones."""
        if len(a) == 3:
            self.ranks()
            a = (self.local, *a)
        local_logits, n_branches, branch_tokens, branch_mask = a
        s = self.s
        a = s.args(local_logits, n_branches, branch_tokens, branch_mask)
        a.conf, a.argmax = self.conf.data_ptr(), self.argmax.data_ptr()
        a.workspace, a.workspace_bytes = self.ws.data_ptr(), self.ws.numel()
        a.scores = self.scores.data_ptr()
        if self.p2p:
            _check(lib().lopa_bp_step_p2p(self.h, ctypes.byref(a), self.b_loc, _stream(s.device)),
                   "lopa_bp_step_p2p")
        else:
            _check(lib().lopa_bp_step(self.h, ctypes.byref(a), self.b_loc, _p(self.records),
                                      _stream(s.device)), "lopa_bp_step")
        return s.out

    def step_lmhead(self, hidden_local: torch.Tensor, weight: torch.Tensor, n_branches,
                    branch_tokens, branch_mask) -> StepOutputs:
        """The step from hidden states (lopa_bp_step_lmhead): this rank's [b_loc * W][K] bf16 hidden
        rows through the LM head + Conf, then the exchange and the global decisions; weight is the
        bf16 [V][K] output projection.  Same results as LMHead.step on one GPU."""
        _need_cuda(hidden_local, weight, n_branches, branch_tokens, branch_mask)
        s = self.s
        h = hidden_local.reshape(-1, hidden_local.shape[-1])
        if h.dtype != torch.bfloat16 or h.stride(1) != 1 or h.shape[0] != self.b_loc * s.window:
            raise LopaError("hidden_local must be bf16 [b_loc * window][K] with unit inner stride")
        if weight.dtype != torch.bfloat16 or weight.stride(1) != 1 or tuple(weight.shape) != (s.vocab, h.shape[1]):
            raise LopaError("weight must be bf16 [V][K] with unit inner stride")
        if getattr(self, "_lmh_ws", None) is None:
            self._lmh_ws = torch.empty(lib().lopa_lmhead_workspace_bytes(self.b_loc * s.window),
                                       dtype=torch.uint8, device=s.device)
        a = s.args(h, n_branches, branch_tokens, branch_mask)
        a.conf, a.argmax = self.conf.data_ptr(), self.argmax.data_ptr()
        a.workspace, a.workspace_bytes = self.ws.data_ptr(), self.ws.numel()
        a.scores = self.scores.data_ptr()
        _check(lib().lopa_bp_step_lmhead(self.h, ctypes.byref(a), self.b_loc, _p(h), h.stride(0),
                                         _p(weight), weight.stride(0), h.shape[1],
                                         None if self.p2p else _p(self.records), _p(self._lmh_ws),
                                         self._lmh_ws.numel(), _stream(s.device)), "lopa_bp_step_lmhead")
        return s.out

    def commit_winner(self, local_payloads: torch.Tensor, out: torch.Tensor | None = None,
                      winner: torch.Tensor | None = None) -> torch.Tensor:
        """NEXT-3 Commit-Winner-Cache: the selected branch's payload (this rank's
        [b_loc][bytes] buffer holds its own branches') on every rank, no host sync."""
        _need_cuda(local_payloads)
        flat = local_payloads.reshape(self.b_loc, -1)
        nbytes = flat.shape[1] * flat.element_size()
        if not flat.is_contiguous():
            raise LopaError("local_payloads must be contiguous [b_loc][...]")
        if out is None:
            out = torch.empty(nbytes, dtype=torch.uint8, device=flat.device)
        w = self.s.out.winner if winner is None else winner
        _check(lib().lopa_bp_commit_winner(self.h, _p(w), self.b_loc, _p(flat), nbytes, _p(out),
                                           _stream(flat.device)), "lopa_bp_commit_winner")
        return out

    def payload_slots(self, parity: int) -> int:
        """Device pointer of this rank's [b_loc][payload_bytes] payload slots of a parity
        (peer-memory mode with payload_bytes > 0), 0 if none."""
        return lib().lopa_bp_payload_slots(self.h, parity) or 0

    def payload_view(self, parity: int) -> torch.Tensor:
        """The payload slots of a parity as a uint8 tensor [b_loc][payload_bytes] (zero copy,
        through __cuda_array_interface__); the caller writes step e's payloads into parity
        e & 1 before that step."""
        ptr = self.payload_slots(parity)
        if not ptr:
            raise LopaError("no payload slots (p2p=True and payload_bytes > 0 needed)")
        nb = self._payload_bytes

        class _Slots:
            __cuda_array_interface__ = {"shape": (self.b_loc, nb), "typestr": "|u1", "data": (ptr, False),
                                        "version": 3, "strides": None}

        return torch.as_tensor(_Slots(), device=self.s.device)

    def commit_winner_p2p(self, out: torch.Tensor, winner: torch.Tensor | None = None) -> torch.Tensor:
        """NEXT-3 over peer memory: the last step's winner payload pulled from its owner."""
        _need_cuda(out)
        w = self.s.out.winner if winner is None else winner
        _check(lib().lopa_bp_commit_winner_p2p(self.h, _p(w), _p(out), _stream(out.device)),
               "lopa_bp_commit_winner_p2p")
        return out

    def check(self):
        _check(lib().lopa_bp_check(self.h), "lopa_bp_check")

    def close(self):
        if getattr(self, "h", None):
            lib().lopa_bp_destroy(self.h)
            self.h = None


class BPEmulator:
    """Single-GPU stand-in for ``world`` BranchParallel ranks (tests, and the bench's
    LOPA_BENCH_EMULATE_BP): every rank's local half (a1 + local a2 + its record,
    lopa_bp_local) runs on that rank's own logits buffer, then the global half (lopa_bp_finish)
    on the record array.  The NCCL all-gather is replaced by each rank writing its record in
    place into one contiguous array -- exactly the all-gather's result.  Same kernels as
    BranchParallel.step."""

    def __init__(self, stepper: Stepper, world: int):
        self.s, self.world = stepper, world
        W, d = stepper.window, stepper.device
        self.b_loc = bp_shard(stepper.max_branches, world, 0)[0]
        self.rb = record_bytes(W, self.b_loc)
        self.records = torch.zeros(world * self.rb, dtype=torch.uint8, device=d)
        self.scores = torch.empty(world * self.b_loc, dtype=torch.float32, device=d)
        self.ws = [new_workspace(self.b_loc * W, stepper.vocab, d) for _ in range(world)]
        self.conf = [torch.full((self.b_loc, W), float("nan"), dtype=torch.float32, device=d)
                     for _ in range(world)]
        self.argmax = [torch.full((self.b_loc, W), -1, dtype=torch.int32, device=d) for _ in range(world)]
        self.local = [torch.zeros((self.b_loc, W, stepper.ld), dtype=torch.bfloat16, device=d)
                      for _ in range(world)]

    def ranks(self):
        """(rank, lo, hi, local logits buffer) of every emulated rank."""
        return [(r, *bp_shard(self.s.max_branches, self.world, r)[1:], self.local[r])
                for r in range(self.world)]

    def step(self, n_branches, branch_tokens, branch_mask) -> StepOutputs:
        """One BP step on the ranks' local buffers (self.local[r] holds rank r's branches)."""
        st, d = self.s, self.s.device
        for r in range(self.world):
            a = st.args(self.local[r], n_branches, branch_tokens, branch_mask)
            a.conf, a.argmax = self.conf[r].data_ptr(), self.argmax[r].data_ptr()
            a.workspace, a.workspace_bytes = self.ws[r].data_ptr(), self.ws[r].numel()
            a.scores = self.scores.data_ptr()
            _check(lib().lopa_bp_local(ctypes.byref(a), r * self.b_loc, self.b_loc,
                                       ctypes.c_void_p(self.records.data_ptr() + r * self.rb), _stream(d)),
                   "lopa_bp_local")
        a = st.args(self.local[0], n_branches, branch_tokens, branch_mask)
        a.scores = self.scores.data_ptr()
        _check(lib().lopa_bp_finish(ctypes.byref(a), self.b_loc, self.world, _p(self.records), _stream(d)),
               "lopa_bp_finish")
        return st.out

    def gathered(self):
        """conf / argmax of every global branch [max_branches][W] (rank r's local branch jl is
        global branch r * b_loc + jl)."""
        mb = self.s.max_branches
        conf = torch.cat(self.conf)[:mb]
        amax = torch.cat(self.argmax)[:mb]
        return conf, amax


def bp_emulate_step(stepper: Stepper, world: int, logits, n_branches, branch_tokens, branch_mask):
    """One emulated `world`-rank BP step on full logits [max_branches][W][ld] (each rank gets
    its slice).  Returns (outputs, per-rank (conf, argmax) list, scores)."""
    emu = BPEmulator(stepper, world)
    for r, lo, hi, buf in emu.ranks():
        if hi > lo:
            buf[: hi - lo] = logits[lo:hi]
    out = emu.step(n_branches, branch_tokens, branch_mask)
    return out, list(zip(emu.conf, emu.argmax)), emu.scores


def decode_block_bp(bp, forward, tokens0: torch.Tensor, mask0: torch.Tensor,
                    max_forwards: int | None = None, on_step=None):
    """Alg. 1 over one window, branch-parallel (P:154-180 with BP): the branch tables are
    replicated; each rank runs the forward of ITS OWN present branches only (global branches
    [lo, min(hi, n)), into its local logits buffer) and reduces them, and the exchange selects the
    global winner.  ``bp`` is a BranchParallel (this process's rank) or a BPEmulator (every rank
    on one GPU).  ``forward(branch_tokens[m][W], branch_mask[m][W], out=logits[m][W][ld])`` as in
    decode_block.  ``on_step(outputs, n_branches_before)`` is called after every step (tests).
    Returns (tokens int32 [W] on the device, forwards); one host read per iteration."""
    st = bp.s
    k, W, dev = st.k, st.window, st.device
    tok = torch.zeros((k + 1, W), dtype=torch.int32, device=dev)
    msk = torch.zeros((k + 1, W), dtype=torch.uint8, device=dev)
    tok[0], msk[0] = tokens0.to(torch.int32), _u8(mask0)
    nb = torch.ones(1, dtype=torch.int32, device=dev)
    forwards, n = 0, 1
    while True:
        for _, lo, hi, buf in bp.ranks():
            m = max(0, min(hi, n) - lo)
            if m > 0:
                forward(tok[lo:lo + m], msk[lo:lo + m], out=buf[:m])
        out = bp.step(nb, tok, msk)
        forwards += 1
        if on_step is not None:
            on_step(out, n, tok, msk)
        n = int(out.n_next.item())
        if n == 0 or (max_forwards is not None and forwards >= max_forwards):
            return out.next_tokens[0].clone(), forwards
        tok.copy_(out.next_tokens)
        msk.copy_(out.next_mask)
        nb.copy_(out.n_next)
