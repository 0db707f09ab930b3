// Host-side internals shared by the liblopa translation units (not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "liblopa.h"

namespace lopa {

// Canonical segmentation of a row: n_seg = ceil(V / 8192) segments of
// seg_len = 8 * ceil(ceil(V / n_seg) / 8) elements (the last one shorter).  Depends on V only.
#ifndef LOPA_SEG_ELEMS
#define LOPA_SEG_ELEMS 8192
#endif
constexpr int kSegElems = LOPA_SEG_ELEMS;          // max elements per canonical segment
constexpr int kChunksPerLane = kSegElems / 8 / 128;  // 16-byte chunks per lane per segment

inline void segmentation(int32_t vocab, int32_t* n_seg, int32_t* seg_len) {
  const int32_t ns = (vocab + kSegElems - 1) / kSegElems;
  const int32_t per = (vocab + ns - 1) / ns;
  *n_seg = ns;
  *seg_len = ((per + 7) / 8) * 8;
}

constexpr int kWarpsPerSeg = 4;  // warp partials per segment (one per consumer warp)
#ifndef LOPA_SEG_PER_ITEM
#define LOPA_SEG_PER_ITEM 2
#endif
constexpr int kSegPerItem = LOPA_SEG_PER_ITEM;  // canonical group = work item = one TMA copy

inline int32_t num_groups(int32_t n_seg) { return (n_seg + kSegPerItem - 1) / kSegPerItem; }

struct Workspace {
  uint32_t* ctrs;       // [0] work-item counter (zero between calls)
  float4* gpart;        // [n_groups][max_rows] group partials (group-major, raw row index)
};

size_t workspace_bytes(int32_t max_rows, int32_t vocab);
bool carve_workspace(void* ws, size_t bytes, int32_t max_rows, int32_t vocab, Workspace* out);

// Selects the device owning `stream` (or `ptr` for the legacy stream) in this library's
// runtime instance.  Returns false on failure.
bool bind_device(void* stream, const void* ptr, int* device);
int num_sms(int device);

// Records the runtime's message of a failed call (lopa_last_cuda_error) and maps it to a status.
void note_cuda_error(cudaError_t e);
inline int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return LOPA_OK;
  note_cuda_error(e);
  return LOPA_ERR_CUDA;
}

int launch_bp_finish(const lopa_step_args_t* a, int32_t b_loc, int32_t world, const void* records,
                     cudaStream_t s, const uint32_t* flags = nullptr, uint32_t epoch = 0);
int launch_bp_local(const lopa_step_args_t* a, int32_t branch_base, int32_t b_loc, void* record,
                    cudaStream_t s, bool conf_ready = false);
int launch_bp_fused(const lopa_step_args_t* a, int32_t b_loc, void* record, uint8_t* const* peer_base,
                    int32_t world, int32_t rank, size_t rb, size_t flags_off, int32_t parity,
                    uint32_t epoch, cudaStream_t s, bool conf_ready = false);
// The LM head + Conf over `rows` rows (chunks of 256); row_base = the global row index of row 0
// (the n_branches test of the fold), row_mask indexed by the local row.
int launch_lmhead_rows(const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                       int32_t rows, int32_t hidden_dim, int32_t vocab, const uint8_t* row_mask,
                       const int32_t* n_branches, int32_t window, int32_t row_base, float* conf,
                       int32_t* argmax, int32_t* dev_status, void* workspace, size_t workspace_bytes,
                       void* stream, int32_t kernel_rows);
int validate_step_args(const lopa_step_args_t* a, bool need_next, bool need_logits = true);
int launch_step_decide(const lopa_step_args_t* a, cudaStream_t s);

}  // namespace lopa
