// SYN-D2F synthetic logits on the device — the harness stand-in for the dLLM forward
// (SURVEY.md §8(d)).  It implements the counter-based definition of
// syngen/__init__.py independently (same integers, same bf16 bits) and holds none of LoPA's
// arithmetic.  tests/test_gpu_parity.py::test_syn_generate_matches_numpy checks the two agree bit for bit.
#include <cmath>
#include <cstdint>

#include "liblopa.h"
#include "lopa_internal.h"

namespace lopa {
namespace syn {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t H2(uint64_t seed, uint64_t a0, uint64_t a1) {
  return mix64(mix64(mix64(seed) ^ a0) ^ a1);
}
__device__ __forceinline__ uint64_t H3(uint64_t seed, uint64_t a0, uint64_t a1, uint64_t a2) {
  return mix64(H2(seed, a0, a1) ^ a2);
}
__device__ __forceinline__ uint64_t H4(uint64_t seed, uint64_t a0, uint64_t a1, uint64_t a2,
                                       uint64_t a3) {
  return mix64(H3(seed, a0, a1, a2) ^ a3);
}

// bf16 bits of (b - 128) / 64 for a byte b (exact: |value| < 2, multiple of 1/64).
__device__ __forceinline__ uint32_t noise_bits(uint32_t b) {
  const float f = (float)((int)b - 128) * (1.0f / 64.0f);
  return __float_as_uint(f) >> 16;
}

// One (branch, position) row of SYN-D2F logits, by one CTA of blockDim.x threads: position i of
// block `blk` whose state (W positions) is tok / msk.
__device__ __forceinline__ void syn_row(uint64_t seed, int blk, int V, long long ld, int W, int c8,
                                        const int32_t* __restrict__ tok,
                                        const uint8_t* __restrict__ msk, int i, int extras,
                                        uint16_t* __restrict__ row) {
  __shared__ unsigned long long s_hash;
  __shared__ int s_nb;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint64_t h = 0;
    for (int p = lane; p < W; p += 32)
      if (!msk[p]) h ^= H4(seed, 2, (uint64_t)blk, (uint64_t)p, (uint64_t)(int64_t)tok[p]);
    for (int off = 16; off > 0; off >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, off);
    int nb = 0;
    for (int d = 1; d <= 3; ++d) {
      const int q0 = i - d, q1 = i + d;
      nb += (q0 >= 0 && q0 < W && !msk[q0]) ? 1 : 0;
      nb += (q1 >= 0 && q1 < W && !msk[q1]) ? 1 : 0;
    }
    if (lane == 0) {
      s_hash = h;
      s_nb = nb;
    }
  }
  __syncthreads();
  const uint64_t rk = H4(seed, 1, (uint64_t)blk, (uint64_t)i, s_hash);
  const int t = (int)(H3(seed, 3, (uint64_t)blk, (uint64_t)i) % (uint64_t)V);
  const int h0 = c8 - 28 + (int)(H3(seed, 4, (uint64_t)blk, (uint64_t)i) % 49ull);
  const int jit = (int)(H2(seed, rk, 5) % 9ull) - 4;
  const int s8 = min(h0 + 16 * s_nb + jit, c8 + 60);
  int tie = -1;
  bool flat = false;
  if (extras & 1) {
    const int sel = (int)(H2(seed, rk, 6) % 16ull);
    if (sel == 0) {
      flat = true;
    } else if (sel == 1) {
      const int t2 = (int)(H3(seed, 7, (uint64_t)blk, (uint64_t)i) % (uint64_t)V);
      if (t2 != t) tie = t2;
    }
  }
  const uint32_t spike = __float_as_uint((float)s8 * 0.125f) >> 16;
  const int nq = (V + 7) / 8;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    uint32_t b[8];
    if (flat) {
#pragma unroll
      for (int r = 0; r < 8; ++r) b[r] = 0;
    } else {
      const uint64_t h = mix64(rk ^ (uint64_t)q);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int v = 8 * q + r;
        uint32_t bits = noise_bits((uint32_t)((h >> (8 * r)) & 0xFF));
        if (v == t || v == tie) bits = spike;
        b[r] = bits;
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (8 * q + r >= V) b[r] = 0;
    if (8 * q + 8 <= ld) {
      uint4 w = make_uint4(b[0] | (b[1] << 16), b[2] | (b[3] << 16), b[4] | (b[5] << 16),
                           b[6] | (b[7] << 16));
      *reinterpret_cast<uint4*>(row + 8 * (size_t)q) = w;
    } else {
      for (int r = 0; r < 8; ++r)
        if (8 * q + r < ld) row[8 * q + r] = (uint16_t)b[r];
    }
  }
  for (long long v = 8LL * nq + threadIdx.x; v < ld; v += blockDim.x) row[v] = 0;
}

// grid (W, n_branches), block 256: one CTA per (branch, position) row.
__global__ void syn_kernel(uint64_t seed, int blk, int V, long long ld, int W, int c8,
                           const int32_t* __restrict__ br_tok, const uint8_t* __restrict__ br_msk,
                           int extras, uint16_t* __restrict__ out) {
  const int i = blockIdx.x, j = blockIdx.y;
  syn_row(seed, blk, V, ld, W, c8, br_tok + (size_t)j * W, br_msk + (size_t)j * W, i, extras,
          out + ((size_t)j * W + i) * (size_t)ld);
}

// lopa_syn_generate with the branch count read on the device: grid (W, max_branches), rows of
// absent branches (j >= *n) skip.
__global__ void syn_dev_kernel(uint64_t seed, int blk, int V, long long ld, int W, int c8,
                               const int32_t* __restrict__ n_dev, int base,
                               const int32_t* __restrict__ br_tok,
                               const uint8_t* __restrict__ br_msk, int extras, uint16_t* __restrict__ out) {
  const int i = blockIdx.x, j = blockIdx.y;
  if (j >= *n_dev - base) return;  // branches [base, n) present: this shard's rows j < n - base
  syn_row(seed, blk, V, ld, W, c8, br_tok + (size_t)j * W, br_msk + (size_t)j * W, i, extras,
          out + ((size_t)j * W + i) * (size_t)ld);
}

// The D2F window's forward (lopa_d2f_syn_forward): grid (max_window, k + 1), one CTA per
// (branch, window position); the window (p0, W, n) is read on the device (sched).  Position
// c of the window is position i = (p0 + c) mod B of block b = (p0 + c) / B, generated from
// that block's columns of the branch's window row -- the same logits as SYN-D2F per block
// ("D2F loops").
__global__ void syn_window_kernel(uint64_t seed, int V, long long ld, int B, int c8,
                                  const int32_t* __restrict__ sched,
                                  const int32_t* __restrict__ br_tok,
                                  const uint8_t* __restrict__ br_msk, int extras,
                                  uint16_t* __restrict__ out) {
  const int p0 = sched[0], W = sched[1], n = sched[2], done = sched[3];
  const int c = blockIdx.x, j = blockIdx.y;
  if (done || c >= W || j >= n) return;
  const int p = p0 + c, b = p / B, i = p - b * B;
  const int cb = b * B - p0;
  syn_row(seed, b, V, ld, B, c8, br_tok + (size_t)j * W + cb, br_msk + (size_t)j * W + cb, i,
          extras, out + ((size_t)j * W + c) * (size_t)ld);
}

}  // namespace syn
}  // namespace lopa

extern "C" int lopa_syn_generate(uint64_t seed, int32_t block, int32_t vocab, int64_t ld,
                                 int32_t window, int32_t n_branches, const int32_t* branch_tokens,
                                 const uint8_t* branch_mask, int32_t extras, void* out,
                                 void* stream) {
  if (vocab < 1 || ld < vocab || ld % 8 != 0 || window < 1 || n_branches < 0 || block < 0)
    return LOPA_ERR_INVALID_ARG;
  if (!branch_tokens || !branch_mask || !out || (reinterpret_cast<uintptr_t>(out) & 15))
    return LOPA_ERR_INVALID_ARG;
  if (n_branches == 0) return LOPA_OK;
  if (n_branches > 65535) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!lopa::bind_device(stream, out, &dev)) return LOPA_ERR_CUDA;
  const int c8 = vocab < 2 ? 0 : (int)std::lround(8.0 * std::log(1.8 * (double)(vocab - 1)));
  dim3 grid(window, n_branches);
  lopa::syn::syn_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, block, vocab, ld, window, c8, branch_tokens, branch_mask, extras,
      static_cast<uint16_t*>(out));
  return lopa::cuda_status(cudaGetLastError());
}

extern "C" int lopa_d2f_syn_forward(uint64_t seed, int32_t vocab, int64_t ld, int32_t extras,
                                    const lopa_d2f_t* d, void* logits, void* stream) {
  if (!d || !logits || vocab < 1 || ld < vocab || ld % 8 != 0 || d->block_size < 1 ||
      d->max_window < 1 || d->max_window > LOPA_MAX_WINDOW || d->k < 0 ||
      d->k + 1 > LOPA_MAX_BRANCHES || !d->sched || !d->branch_tokens || !d->branch_mask ||
      (reinterpret_cast<uintptr_t>(logits) & 15))
    return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!lopa::bind_device(stream, logits, &dev)) return LOPA_ERR_CUDA;
  const int c8 = vocab < 2 ? 0 : (int)std::lround(8.0 * std::log(1.8 * (double)(vocab - 1)));
  dim3 grid(d->max_window, d->k + 1);
  lopa::syn::syn_window_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, vocab, ld, d->block_size, c8, d->sched, d->branch_tokens, d->branch_mask, extras,
      static_cast<uint16_t*>(logits));
  return lopa::cuda_status(cudaGetLastError());
}

extern "C" int lopa_syn_generate_dev(uint64_t seed, int32_t block, int32_t vocab, int64_t ld,
                                     int32_t window, int32_t max_branches, const int32_t* n_branches_dev,
                                     int32_t branch_base, const int32_t* branch_tokens,
                                     const uint8_t* branch_mask, int32_t extras, void* out, void* stream) {
  if (vocab < 1 || ld < vocab || ld % 8 != 0 || window < 1 || max_branches < 1 || block < 0 ||
      branch_base < 0)
    return LOPA_ERR_INVALID_ARG;
  if (!n_branches_dev || !branch_tokens || !branch_mask || !out || (reinterpret_cast<uintptr_t>(out) & 15))
    return LOPA_ERR_INVALID_ARG;
  if (max_branches > 65535) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!lopa::bind_device(stream, out, &dev)) return LOPA_ERR_CUDA;
  const int c8 = vocab < 2 ? 0 : (int)std::lround(8.0 * std::log(1.8 * (double)(vocab - 1)));
  dim3 grid(window, max_branches);
  lopa::syn::syn_dev_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      seed, block, vocab, ld, window, c8, n_branches_dev, branch_base, branch_tokens, branch_mask,
      extras, static_cast<uint16_t*>(out));
  return lopa::cuda_status(cudaGetLastError());
}
