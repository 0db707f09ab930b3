// Warp-level LoPA decisions (one warp owns a window of W <= 64 positions and <= 32 branches):
//   Eq. 2 branch scores + select, Eq. 1 anchor,
//   top-k lookahead spawn.
// Lane l owns positions l and l + 32.  All decisions are exact functions of the fp32 conf
// bits: ordered integer keys, ballots and rank counting — no floating-point reassociation.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lopa_ptx.cuh"

namespace lopa {

constexpr int kDevEmptyMask = 1;
constexpr int kDevNonfinite = 2;

// Position state of one window held in registers: lane owns slots 0 (i = lane) and 1
// (i = lane + 32).
struct WinRegs {
  float conf[2];
  int32_t amax[2];
  int32_t tok[2];
  uint32_t msk[2];  // 1 = masked
};

// Order-preserving map of a float to uint32 (for non-NaN values; -inf is smallest).
__device__ __forceinline__ uint32_t ordered_bits(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Load the window row of branch state (tok/msk) and conf/argmax.  conf / msk may point to shared
// memory (generic loads); amax is global and read L2-coherently (written by other CTAs).
__device__ __forceinline__ void load_window(WinRegs& r, const float* conf, const int32_t* amax,
                                            const int32_t* tok, const uint8_t* msk, int W,
                                            int lane) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int i = lane + 32 * s;
    const bool in = i < W;
    r.msk[s] = in ? (uint32_t)(msk[i] != 0) : 0u;
    r.tok[s] = in ? tok[i] : 0;
    r.conf[s] = (in && r.msk[s]) ? conf[i] : 0.f;
    r.amax[s] = (in && r.msk[s]) ? __ldcg(amax + i) : -1;
  }
}

// Eq. 2: lane j < n_br scores branch j: sum of conf over its masked positions in
// position order (fp64), divided by the count, rounded once to fp32; 1.0 if none (R8).
// Absent branches (n_br <= j < max_br) score -inf.  Returns the branch's score in lane j.
// conf / mask are generic pointers (shared memory in the fused tail).
__device__ __forceinline__ float warp_branch_score(const float* conf, const uint8_t* mask,
                                                   int n_br, int max_br, int W, int lane) {
  float score = -INFINITY;
  if (lane < n_br) {
    const float* c = conf + (size_t)lane * W;
    const uint8_t* m = mask + (size_t)lane * W;
    double sum = 0.0;
    int cnt = 0;
    for (int i = 0; i < W; ++i) {
      if (m[i]) {
        sum += (double)c[i];
        ++cnt;
      }
    }
    score = cnt ? (float)(sum / (double)cnt) : 1.0f;
  }
  (void)max_br;
  return score;
}

// Branch-confidence metrics.
constexpr int kMetricMean = 0;            // Eq. 2: mean over M_Bj
constexpr int kMetricSlidingMin = 1;      // min over length-w windows (position order) of the mean
constexpr int kMetricBottomFraction = 2;  // mean of the ceil(eta * |M_Bj|) lowest confidences

// C(B_j) of one branch with a full warp (lane owns positions lane and lane + 32).  conf / mask are
// generic pointers; dscr (64 doubles) and fscr (64 floats) are per-warp shared scratch.  Every sum
// is an exact fp64 sum (each conf lies in [2^-23, 1], at most 64 terms), so the value equals the
// oracle's fp64 value whatever the summation order, rounded once to fp32.  1.0 if M_Bj is empty.
__device__ __forceinline__ float warp_metric_score(const float* conf, const uint8_t* mask, int W,
                                                   int metric, float param, double* dscr,
                                                   float* fscr, int lane) {
  bool m[2];
  double v[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    m[h] = i < W && mask[i] != 0;
    v[h] = m[h] ? (double)conf[i] : 0.0;
  }
  const uint32_t b0 = __ballot_sync(0xffffffffu, m[0]), b1 = __ballot_sync(0xffffffffu, m[1]);
  const int n = __popc(b0) + __popc(b1);
  if (n == 0) return 1.0f;
  if (metric == kMetricMean) {
    double s = v[0] + v[1];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return (float)(s / (double)n);
  }
  const uint32_t lt = (1u << lane) - 1u;
  const int idx[2] = {__popc(b0 & lt), __popc(b0) + __popc(b1 & lt)};
  float result;
  if (metric == kMetricSlidingMin) {
    const int w = min(max((int)param, 1), n);
    // inclusive prefix sums in position (= compacted) order, stored by compacted index
    double P[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double x = v[h];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      P[h] = x;
    }
    P[1] += __shfl_sync(0xffffffffu, P[0], 31);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (m[h]) dscr[idx[h]] = P[h];
    __syncwarp();
    double best = INFINITY;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (m[h] && idx[h] >= w - 1) {
        const double lo = idx[h] - w >= 0 ? dscr[idx[h] - w] : 0.0;
        best = fmin(best, (P[h] - lo) / (double)w);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, off));
    result = (float)best;
  } else {  // kMetricBottomFraction
    const int b = (int)ceil((double)param * (double)n);
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (m[h]) fscr[idx[h]] = (float)v[h];
    __syncwarp();
    double s = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (m[h]) {
        const float x = (float)v[h];
        int r = 0;
        for (int q = 0; q < n; ++q) r += (fscr[q] < x || (fscr[q] == x && q < idx[h])) ? 1 : 0;
        if (r < b) s += v[h];
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    result = (float)(s / (double)b);
  }
  __syncwarp();
  return result;
}

// Select (R9): smallest j with the largest fp32 score.  Scores are never NaN-free
// guaranteed (a NONFINITE row poisons its branch); NaN scores lose (treated as -inf).
__device__ __forceinline__ int warp_select(float score, int lane, int n_lanes_valid) {
  const float s = (lane < n_lanes_valid && !isnan(score)) ? score : -INFINITY;
  const uint32_t key = ordered_bits(s);
  const uint32_t best = __reduce_max_sync(0xffffffffu, key);
  const uint32_t cand = (key == best && lane < n_lanes_valid) ? (uint32_t)lane : 0xffffffffu;
  const uint32_t w = __reduce_min_sync(0xffffffffu, cand);
  return (w == 0xffffffffu) ? 0 : (int)w;
}

// Eq. 1 + Alg. 1 step 1 on the window in registers: fills I_fill in place (r becomes B0).
// Returns LOPA_DEV_EMPTY_MASK if nothing is masked (state unchanged), else 0.
__device__ __forceinline__ int warp_anchor(WinRegs& r, float tau, int lane) {
  bool high[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) high[s] = r.msk[s] && (r.conf[s] > tau);
  const uint32_t any_masked = __ballot_sync(0xffffffffu, r.msk[0] | r.msk[1]);
  if (!any_masked) return kDevEmptyMask;
  const uint32_t any_high = __ballot_sync(0xffffffffu, high[0] | high[1]);
  if (any_high) {
#pragma unroll
    for (int s = 0; s < 2; ++s)
      if (high[s]) {
        r.tok[s] = r.amax[s];
        r.msk[s] = 0;
      }
    return 0;
  }
  // Fallback (Eq. 1 "otherwise"): argmax conf over M_t, lowest position on ties (R5).
  uint32_t k0 = r.msk[0] ? ordered_bits(r.conf[0]) : 0u;
  uint32_t k1 = r.msk[1] ? ordered_bits(r.conf[1]) : 0u;
  const uint32_t best = __reduce_max_sync(0xffffffffu, max(k0, k1));
  uint32_t cand = 0xffffffffu;
  if (r.msk[1] && k1 == best) cand = (uint32_t)(lane + 32);
  if (r.msk[0] && k0 == best) cand = (uint32_t)lane;
  const uint32_t istar = __reduce_min_sync(0xffffffffu, cand);
#pragma unroll
  for (int s = 0; s < 2; ++s)
    if ((uint32_t)(lane + 32 * s) == istar) {
      r.tok[s] = r.amax[s];
      r.msk[s] = 0;
    }
  return 0;
}

// Alg. 1 step 2: rank of every position of M_B0 under (conf desc, position asc)
// by counting, n = min(k, |M_B0|).  `keys` is a 64-entry per-warp shared scratch.
// Writes branch tables rows 0..n, lookahead_pos[0..k), *n_branches = n + 1.
__device__ __forceinline__ void warp_spawn(const WinRegs& b0, int W, int k, uint64_t* keys,
                                           int32_t* br_tok, uint8_t* br_msk, int32_t* look,
                                           int32_t* n_branches, int lane) {
  // key = ordered conf bits << 32 | (63 - i): larger key = earlier in the order.
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int i = lane + 32 * s;
    keys[i] = b0.msk[s] ? (((uint64_t)ordered_bits(b0.conf[s]) << 32) | (uint64_t)(63 - i))
                        : 0ull;
  }
  __syncwarp();
  const int n_mb0 = __popc(__ballot_sync(0xffffffffu, b0.msk[0])) +
                    __popc(__ballot_sync(0xffffffffu, b0.msk[1]));
  const int n = min(k, n_mb0);
  int rank[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const uint64_t mine = keys[lane + 32 * s];
    int cnt = 0;
#pragma unroll 8
    for (int q = 0; q < 64; ++q) cnt += (keys[q] > mine) ? 1 : 0;
    rank[s] = b0.msk[s] ? cnt : 1 << 20;
  }
  __syncwarp();
#ifdef TL
  if (lane == 0) TL(12);
#endif
  // Branch j (1..n) fills p_j = the position of rank j - 1.
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int i = lane + 32 * s;
    if (rank[s] < n && look) look[rank[s]] = i;
  }
  if (look)
    for (int q = n + lane; q < k; q += 32) look[q] = -1;
  for (int j = 0; j <= n; ++j) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int i = lane + 32 * s;
      if (i < W) {
        const bool fill = (j >= 1) && (rank[s] == j - 1);
        br_tok[(size_t)j * W + i] = fill ? b0.amax[s] : b0.tok[s];
        br_msk[(size_t)j * W + i] = fill ? 0 : (uint8_t)b0.msk[s];
      }
    }
  }
  if (lane == 0) *n_branches = n + 1;
#ifdef TL
  if (lane == 0) TL(13);
#endif
}

// Store the window registers to a table row.
__device__ __forceinline__ void store_window(const WinRegs& r, int32_t* tok, uint8_t* msk, int W,
                                             int lane) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int i = lane + 32 * s;
    if (i < W) {
      tok[i] = r.tok[s];
      msk[i] = (uint8_t)r.msk[s];
    }
  }
}

}  // namespace lopa
