// Branch parallelism (BP) across the GPUs of one box ("TP1+BP8"): each rank
// reduces and scores only its own branches, then ONE ncclAllGather of fixed-size records
// {local scores, local best (score, id), the best branch's tokens/mask/conf/argmax row}
// gives every rank what it needs to run the same deterministic select, anchor and spawn.
// The all-gather subsumes the (score, id) all-gather + winner-row broadcast of SURVEY §8(e):
// the broadcast root (the winner's owner) is device data, and a host-side root would force a
// device->host synchronisation every step.
#include <cstring>
#include <new>

#include <nccl.h>

#include "liblopa.h"
#include "lopa_internal.h"

struct lopa_bp {
  ncclComm_t comm;
  int32_t rank, world, device;
  // peer-memory exchange (lopa_bp_step_p2p)
  uint8_t* p2p_base = nullptr;      // local: [2 parities][world][rb] records, then [world] u32 flags
  size_t p2p_rb = 0, p2p_bytes = 0;
  int32_t p2p_b_loc = 0;
  size_t p2p_payload = 0;           // payload bytes per branch (0: none)
  size_t p2p_payload_off = 0;       // [2 parities][b_loc][payload] after the flags
  uint8_t* peer_base[32] = {};      // every rank's mapped base (own = p2p_base)
  uint8_t** d_peer_base = nullptr;  // device copy of peer_base
  bool p2p_open = false;
  uint32_t epoch = 0;
};

extern "C" int lopa_bp_get_unique_id(void* unique_id_out) {
  if (!unique_id_out) return LOPA_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == LOPA_BP_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return LOPA_ERR_NCCL;
  std::memcpy(unique_id_out, &id, sizeof(id));
  return LOPA_OK;
}

extern "C" int lopa_bp_create(const void* unique_id, int32_t rank, int32_t world, int32_t device,
                              lopa_bp_t** out) {
  if (!unique_id || !out || world < 1 || world > 32 || rank < 0 || rank >= world || device < 0)
    return LOPA_ERR_INVALID_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return LOPA_ERR_CUDA;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  lopa_bp* bp = new (std::nothrow) lopa_bp;
  if (!bp) return LOPA_ERR_CUDA;
  if (ncclCommInitRank(&bp->comm, world, id, rank) != ncclSuccess) {
    delete bp;
    return LOPA_ERR_NCCL;
  }
  bp->rank = rank;
  bp->world = world;
  bp->device = device;
  *out = bp;
  return LOPA_OK;
}

extern "C" int lopa_bp_step(lopa_bp_t* bp, const lopa_step_args_t* args, int32_t b_loc,
                            void* records, void* stream) {
  if (!bp || !args || !records || b_loc < 1) return LOPA_ERR_INVALID_ARG;
  if ((int64_t)b_loc * bp->world < args->max_branches) return LOPA_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t rb = lopa_bp_record_bytes(args->window, b_loc);
  uint8_t* mine = static_cast<uint8_t*>(records) + rb * bp->rank;
  int st = lopa::launch_bp_local(args, bp->rank * b_loc, b_loc, mine, s);
  if (st != LOPA_OK) return st;
  // in-place all-gather: rank r's send buffer is its own slot of the receive buffer
  if (ncclAllGather(mine, records, rb, ncclUint8, bp->comm, s) != ncclSuccess) return LOPA_ERR_NCCL;
  return lopa::launch_bp_finish(args, b_loc, bp->world, records, s);
}

// NEXT-3 Commit-Winner-Cache (Fig. 3 phase 2): every rank contributes the winner's
// payload if it owns the winner and zeros otherwise; a sum all-reduce over 32-bit words then
// leaves the owner's bytes on every rank (x + 0 = x exactly on integers).  The root is device
// data, so no host synchronisation is needed.
namespace {
__global__ void commit_select_kernel(const int32_t* winner, int32_t rank, int32_t b_loc,
                                     const uint4* local, size_t n16, uint4* out) {
  const int32_t w = *winner;
  const int32_t owner = w / b_loc;
  const uint4* src = local + (size_t)(w - owner * b_loc) * n16;
  const bool mine = owner == rank;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x)
    out[i] = mine ? src[i] : make_uint4(0u, 0u, 0u, 0u);
}
}  // namespace

extern "C" int lopa_bp_commit_winner(lopa_bp_t* bp, const int32_t* winner, int32_t b_loc,
                                     const void* local_payloads, size_t payload_bytes, void* out,
                                     void* stream) {
  if (!bp || !winner || !local_payloads || !out || b_loc < 1 || payload_bytes == 0 ||
      payload_bytes % 16 != 0)
    return LOPA_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(local_payloads) | reinterpret_cast<uintptr_t>(out)) & 15)
    return LOPA_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t n16 = payload_bytes / 16;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, bp->device);
  const size_t want = (n16 + 255) / 256;
  const int grid = (int)(want < (size_t)(4 * sms) ? (want ? want : 1) : (size_t)(4 * sms));
  commit_select_kernel<<<grid, 256, 0, s>>>(winner, bp->rank, b_loc,
                                            static_cast<const uint4*>(local_payloads), n16,
                                            static_cast<uint4*>(out));
  if (cudaGetLastError() != cudaSuccess) return LOPA_ERR_CUDA;
  if (ncclAllReduce(out, out, payload_bytes / 4, ncclUint32, ncclSum, bp->comm, s) != ncclSuccess)
    return LOPA_ERR_NCCL;
  return LOPA_OK;
}

extern "C" int lopa_bp_check(lopa_bp_t* bp) {
  if (!bp) return LOPA_ERR_INVALID_ARG;
  ncclResult_t async = ncclSuccess;
  if (ncclCommGetAsyncError(bp->comm, &async) != ncclSuccess || async != ncclSuccess)
    return LOPA_ERR_NCCL;
  return LOPA_OK;
}

extern "C" void lopa_bp_destroy(lopa_bp_t* bp) {
  if (!bp) return;
  if (bp->p2p_open)
    for (int q = 0; q < bp->world; ++q)
      if (q != bp->rank && bp->peer_base[q]) cudaIpcCloseMemHandle(bp->peer_base[q]);
  if (bp->d_peer_base) cudaFree(bp->d_peer_base);
  if (bp->p2p_base) cudaFree(bp->p2p_base);
  ncclCommDestroy(bp->comm);
  delete bp;
}

// ---- peer-memory exchange ---------------------------------------------------------------------
static_assert(sizeof(cudaIpcMemHandle_t) == LOPA_BP_IPC_HANDLE_BYTES, "IPC handle size");

#ifdef LOPA_BP_P2P_3K
namespace {
// One CTA: copy this rank's record (rb bytes, 16-byte units) into slot `rank` of the current
// parity of every peer, then, after a system-scope fence, raise this rank's flag to `epoch`
// in every peer's flag array (release).
__global__ void bp_publish_kernel(uint8_t* const* peer_base, int world, int rank, size_t rb,
                                  size_t flags_off, int parity, uint32_t epoch) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // K2 has written this rank's record
  asm volatile("griddepcontrol.launch_dependents;");
  const size_t slot = ((size_t)parity * world + rank) * rb;
  const uint4* src = reinterpret_cast<const uint4*>(peer_base[rank] + slot);
  const size_t n16 = rb / 16;
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    uint4* dst = reinterpret_cast<uint4*>(peer_base[q] + slot);
    for (size_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < world; ++q) {
      uint32_t* f = reinterpret_cast<uint32_t*>(peer_base[q] + flags_off) + rank;
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
    }
  }
}
}  // namespace
#endif

extern "C" int lopa_bp_p2p_alloc(lopa_bp_t* bp, int32_t window, int32_t b_loc, size_t payload_bytes,
                                 void* handle_out) {
  if (!bp || !handle_out || b_loc < 1 || window < 1 || window > LOPA_MAX_WINDOW || bp->p2p_base ||
      payload_bytes % 16 != 0)
    return LOPA_ERR_INVALID_ARG;
  if (cudaSetDevice(bp->device) != cudaSuccess) return LOPA_ERR_CUDA;
  bp->p2p_rb = lopa_bp_record_bytes(window, b_loc);
  bp->p2p_b_loc = b_loc;
  const size_t flags_off = 2 * (size_t)bp->world * bp->p2p_rb;
  bp->p2p_payload = payload_bytes;
  bp->p2p_payload_off = flags_off + 256;
  bp->p2p_bytes = bp->p2p_payload_off + 2 * (size_t)b_loc * payload_bytes;
  if (cudaMalloc(&bp->p2p_base, bp->p2p_bytes) != cudaSuccess) return LOPA_ERR_CUDA;
  if (cudaMemset(bp->p2p_base, 0, bp->p2p_bytes) != cudaSuccess) return LOPA_ERR_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, bp->p2p_base) != cudaSuccess) return LOPA_ERR_CUDA;
  std::memcpy(handle_out, &h, sizeof(h));
  return LOPA_OK;
}

extern "C" int lopa_bp_p2p_open(lopa_bp_t* bp, const void* all_handles) {
  if (!bp || !all_handles || !bp->p2p_base || bp->p2p_open) return LOPA_ERR_INVALID_ARG;
  if (cudaSetDevice(bp->device) != cudaSuccess) return LOPA_ERR_CUDA;
  const auto* hs = static_cast<const cudaIpcMemHandle_t*>(all_handles);
  for (int q = 0; q < bp->world; ++q) {
    if (q == bp->rank) {
      bp->peer_base[q] = bp->p2p_base;
      continue;
    }
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, hs[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return LOPA_ERR_CUDA;
    bp->peer_base[q] = static_cast<uint8_t*>(ptr);
  }
  if (cudaMalloc(&bp->d_peer_base, 32 * sizeof(uint8_t*)) != cudaSuccess) return LOPA_ERR_CUDA;
  if (cudaMemcpy(bp->d_peer_base, bp->peer_base, 32 * sizeof(uint8_t*), cudaMemcpyHostToDevice) !=
      cudaSuccess)
    return LOPA_ERR_CUDA;
  bp->p2p_open = true;
  return LOPA_OK;
}

extern "C" int lopa_bp_step_p2p(lopa_bp_t* bp, const lopa_step_args_t* args, int32_t b_loc,
                                void* stream) {
  if (!bp || !args || !bp->p2p_open || b_loc != bp->p2p_b_loc) return LOPA_ERR_INVALID_ARG;
  if ((int64_t)b_loc * bp->world < args->max_branches) return LOPA_ERR_INVALID_ARG;
  if (lopa_bp_record_bytes(args->window, b_loc) != bp->p2p_rb) return LOPA_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t epoch = ++bp->epoch;
  const int parity = (int)(epoch & 1u);
  const size_t rb = bp->p2p_rb;
  uint8_t* records = bp->p2p_base + (size_t)parity * bp->world * rb;
  uint8_t* mine = records + rb * bp->rank;
  const size_t flags_off = 2 * (size_t)bp->world * rb;
#ifndef LOPA_BP_P2P_3K
  // one fused kernel after K1: local half, NVLink stores + flags, wait, global half.  The kernel
  // keeps the exchange epoch on the device (graph safe); the host count above tracks it for
  // the payload slots of the Commit-Winner-Cache (lopa_bp_payload_slots / _commit_winner_p2p),
  // which therefore stay host-driven
  return lopa::launch_bp_fused(args, b_loc, mine, (uint8_t* const*)bp->d_peer_base, bp->world,
                               bp->rank, rb, flags_off, parity, epoch, s);
#else
  // round-1 form: K2 (local half), a publish kernel, the finishing kernel
  int st = lopa::launch_bp_local(args, bp->rank * b_loc, b_loc, mine, s);
  if (st != LOPA_OK) return st;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, bp_publish_kernel, (uint8_t* const*)bp->d_peer_base, (int)bp->world,
                           (int)bp->rank, rb, flags_off, parity, epoch) != cudaSuccess)
      return LOPA_ERR_CUDA;
  }
  return lopa::launch_bp_finish(args, b_loc, bp->world, records, s,
                                reinterpret_cast<const uint32_t*>(bp->p2p_base + flags_off), epoch);
#endif
}

// The branch-parallel step from hidden states (NEXT-4 x a5): each rank runs the LM head + Conf
// on its own branches' rows, then the same exchange as lopa_bp_step_p2p (peer memory, when
// opened) or lopa_bp_step (NCCL all-gather of `records`), the decision kernel reading the
// LM head's conf / argmax instead of K1's partials.
extern "C" int lopa_bp_step_lmhead(lopa_bp_t* bp, const lopa_step_args_t* args, int32_t b_loc,
                                   const void* hidden, int64_t ld_hidden, const void* weight,
                                   int64_t ld_weight, int32_t hidden_dim, void* records,
                                   void* lmh_workspace, size_t lmh_workspace_bytes, void* stream) {
  if (!bp || !args || b_loc < 1 || !hidden || !weight) return LOPA_ERR_INVALID_ARG;
  if ((int64_t)b_loc * bp->world < args->max_branches) return LOPA_ERR_INVALID_ARG;
  if (!bp->p2p_open && !records) return LOPA_ERR_INVALID_ARG;
  if (bp->p2p_open && (b_loc != bp->p2p_b_loc || lopa_bp_record_bytes(args->window, b_loc) != bp->p2p_rb))
    return LOPA_ERR_INVALID_ARG;
  if ((int64_t)b_loc * args->window > LOPA_MAX_ROWS) return LOPA_ERR_UNSUPPORTED;
  if (!args->conf || !args->argmax || !args->dev_status || !args->branch_mask) return LOPA_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int32_t W = args->window;
  const int32_t base = bp->rank * b_loc;
  // rows of this rank's branches: branch base + r / W; a row of an absent branch (or one past the
  // table) is not reduced (conf NaN, argmax -1) and its mask byte is never read
  int st = lopa::launch_lmhead_rows(hidden, ld_hidden, weight, ld_weight, b_loc * W, hidden_dim,
                                    args->vocab, args->branch_mask + (size_t)base * W,
                                    args->n_branches, W, base * W, args->conf, args->argmax,
                                    args->dev_status, lmh_workspace, lmh_workspace_bytes, stream,
                                    args->max_branches * W);
  if (st != LOPA_OK) return st;
  if (bp->p2p_open) {
    const uint32_t epoch = ++bp->epoch;
    const int parity = (int)(epoch & 1u);
    const size_t rb = bp->p2p_rb;
    uint8_t* mine = bp->p2p_base + (size_t)parity * bp->world * rb + rb * bp->rank;
    return lopa::launch_bp_fused(args, b_loc, mine, (uint8_t* const*)bp->d_peer_base, bp->world,
                                 bp->rank, rb, 2 * (size_t)bp->world * rb, parity, epoch, s, true);
  }
  const size_t rb = lopa_bp_record_bytes(W, b_loc);
  uint8_t* mine = static_cast<uint8_t*>(records) + rb * bp->rank;
  st = lopa::launch_bp_local(args, base, b_loc, mine, s, true);
  if (st != LOPA_OK) return st;
  if (ncclAllGather(mine, records, rb, ncclUint8, bp->comm, s) != ncclSuccess) return LOPA_ERR_NCCL;
  return lopa::launch_bp_finish(args, b_loc, bp->world, records, s);
}

// ---- Commit-Winner-Cache over peer memory ---------------------------------------------------------
namespace {
// Pull the winner's payload from its owner's mapped payload slots (parity of the last step).
__global__ void bp_pull_payload_kernel(uint8_t* const* peer_base, const int32_t* winner, int b_loc,
                                       size_t payload_off, size_t payload, int parity, uint4* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int w = *winner;
  const int owner = w / b_loc;
  const uint4* src = reinterpret_cast<const uint4*>(
      peer_base[owner] + payload_off + ((size_t)parity * b_loc + (w - owner * b_loc)) * payload);
  const size_t n16 = payload / 16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    out[i] = src[i];
}
}  // namespace

extern "C" void* lopa_bp_payload_slots(lopa_bp_t* bp, int32_t parity) {
  if (!bp || !bp->p2p_base || bp->p2p_payload == 0 || parity < 0 || parity > 1) return nullptr;
  return bp->p2p_base + bp->p2p_payload_off + (size_t)parity * bp->p2p_b_loc * bp->p2p_payload;
}

extern "C" int lopa_bp_commit_winner_p2p(lopa_bp_t* bp, const int32_t* winner, void* out, void* stream) {
  if (!bp || !winner || !out || !bp->p2p_open || bp->p2p_payload == 0 || bp->epoch == 0)
    return LOPA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(out) & 15) return LOPA_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, bp->device);
  const size_t want = (bp->p2p_payload / 16 + 255) / 256;
  const int grid = (int)(want < (size_t)(4 * sms) ? (want ? want : 1) : (size_t)(4 * sms));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int parity = (int)(bp->epoch & 1u);
  return cudaLaunchKernelEx(&cfg, bp_pull_payload_kernel, (uint8_t* const*)bp->d_peer_base, winner,
                            (int)bp->p2p_b_loc, bp->p2p_payload_off, bp->p2p_payload, parity,
                            static_cast<uint4*>(out)) == cudaSuccess
             ? LOPA_OK
             : LOPA_ERR_CUDA;
}
