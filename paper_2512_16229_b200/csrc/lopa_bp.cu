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
  ncclCommDestroy(bp->comm);
  delete bp;
}
