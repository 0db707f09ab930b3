// Warp-level LoPA decisions over a window of W <= 32*S positions (S = 2 for W <= 64, S = 8 for
// the D2F multi-block window up to 256) and <= 32 branches:
//   Eq. 2 branch scores (+ the P:204 variants) and select, Eq. 1 anchor
//    with a per-position threshold (D2F), top-k lookahead spawn
//   (P:167-171).
// Lane l owns positions l + 32 h, h < S.  All decisions are exact functions of the fp32 conf bits:
// ordered integer keys, ballots and rank counting — no floating-point reassociation.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lopa_ptx.cuh"

namespace lopa {

constexpr int kDevEmptyMask = 1;
constexpr int kDevNonfinite = 2;
constexpr int kDevPeerTimeout = 4;
constexpr int kDevInternal = 8;   // LOPA_DEV_INTERNAL: a K1 partial never arrived (bounded poll)

// Position state of one window held in registers.
template <int S>
struct WinRegs {
  float conf[S];
  int32_t amax[S];
  int32_t tok[S];
  uint32_t msk[S];  // 1 = masked
};

// Order-preserving map of a float to uint32 (for non-NaN values; -inf is smallest).
__device__ __forceinline__ uint32_t ordered_bits(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Load the window row of branch state (tok/msk) and conf/argmax.  conf / msk may point to shared
// memory (generic loads); amax is read L2-coherently.
template <int S>
__device__ __forceinline__ void load_window(WinRegs<S>& r, const float* conf, const int32_t* amax,
                                            const int32_t* tok, const uint8_t* msk, int W,
                                            int lane) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    const bool in = i < W;
    r.msk[s] = in ? (uint32_t)(msk[i] != 0) : 0u;
    r.tok[s] = in ? tok[i] : 0;
    r.conf[s] = (in && r.msk[s]) ? conf[i] : 0.f;
    r.amax[s] = (in && r.msk[s]) ? __ldcg(amax + i) : -1;
  }
}

// Eq. 2: lane j < n_br scores branch j (mean of conf over its masked positions, fp64,
// rounded once to fp32; 1.0 if none, R8).  Absent branches score -inf.
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

// C(B_j) of one branch with a full warp.  conf / mask are generic pointers; dscr (32 S doubles) and
// fscr (32 S floats) are per-warp shared scratch.  Every sum is an exact fp64 sum (reading R24:
// each conf is an fp32 value >= 1/V, so its lowest significant bit is >= 2^-(23 + ceil(log2 V));
// with <= W terms the sum stays below 2^ceil(log2 W); the host enforces
// ceil(log2 W) + 23 + ceil(log2 V) <= 53), so the value equals the oracle's fp64 value whatever
// the order, rounded once to fp32.  1.0 if M_Bj is empty.
#ifndef LOPA_SCORE_MARK
#define LOPA_SCORE_MARK(s) ((void)0)
#endif
template <int S>
__device__ __forceinline__ float warp_metric_score(const float* conf, const uint8_t* mask, int W,
                                                   int metric, float param, double* dscr,
                                                   float* fscr, int lane) {
  bool m[S];
  double v[S];
  uint32_t b[S];
  int n = 0;
#pragma unroll
  for (int h = 0; h < S; ++h) {
    const int i = lane + 32 * h;
    m[h] = i < W && mask[i] != 0;
    v[h] = m[h] ? (double)conf[i] : 0.0;
    b[h] = __ballot_sync(0xffffffffu, m[h]);
    n += __popc(b[h]);
  }
  if (n == 0) return 1.0f;
  LOPA_SCORE_MARK(12);
  if (metric == kMetricMean) {
    double s = 0.0;
#pragma unroll
    for (int h = 0; h < S; ++h) s += v[h];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    LOPA_SCORE_MARK(13);
    const float r = (float)(s / (double)n);
    LOPA_SCORE_MARK(14);
    return r;
  }
  const uint32_t lt = (1u << lane) - 1u;
  int idx[S];
  {
    int base = 0;
#pragma unroll
    for (int h = 0; h < S; ++h) {
      idx[h] = base + __popc(b[h] & lt);
      base += __popc(b[h]);
    }
  }
  float result;
  if (metric == kMetricSlidingMin) {
    const int w = min(max((int)param, 1), n);
    // inclusive prefix sums in position (= compacted) order, stored by compacted index
    double P[S];
    double carry = 0.0;
#pragma unroll
    for (int h = 0; h < S; ++h) {
      double x = v[h];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
      }
      P[h] = x + carry;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
#pragma unroll
    for (int h = 0; h < S; ++h)
      if (m[h]) dscr[idx[h]] = P[h];
    __syncwarp();
    double best = INFINITY;
#pragma unroll
    for (int h = 0; h < S; ++h) {
      if (m[h] && idx[h] >= w - 1) {
        const double lo = idx[h] - w >= 0 ? dscr[idx[h] - w] : 0.0;
        best = fmin(best, (P[h] - lo) / (double)w);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, off));
    result = (float)best;
  } else {  // kMetricBottomFraction
    const int bcnt = (int)ceil((double)param * (double)n);
#pragma unroll
    for (int h = 0; h < S; ++h)
      if (m[h]) fscr[idx[h]] = (float)v[h];
    __syncwarp();
    double s = 0.0;
#pragma unroll
    for (int h = 0; h < S; ++h) {
      if (m[h]) {
        const float x = (float)v[h];
        int r = 0;
        for (int q = 0; q < n; ++q) r += (fscr[q] < x || (fscr[q] == x && q < idx[h])) ? 1 : 0;
        if (r < bcnt) s += v[h];
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    result = (float)(s / (double)bcnt);
  }
  __syncwarp();
  return result;
}

// Select (R9): smallest j with the largest fp32 score (NaN scores lose).
__device__ __forceinline__ int warp_select(float score, int lane, int n_lanes_valid) {
  const float s = (lane < n_lanes_valid && !isnan(score)) ? score : -INFINITY;
  const uint32_t key = ordered_bits(s);
  const uint32_t best = __reduce_max_sync(0xffffffffu, key);
  const uint32_t cand = (key == best && lane < n_lanes_valid) ? (uint32_t)lane : 0xffffffffu;
  const uint32_t w = __reduce_min_sync(0xffffffffu, cand);
  return (w == 0xffffffffu) ? 0 : (int)w;
}

// Eq. 1 + Alg. 1 step 1 on the window in registers: fills I_fill in place (r becomes B0).
// tau_pos (nullable): per-position thresholds (D2F window: tau_act / tau_conf per block).
// Returns LOPA_DEV_EMPTY_MASK if nothing is masked (state unchanged), else 0.
template <int S>
__device__ __forceinline__ int warp_anchor(WinRegs<S>& r, float tau, const float* tau_pos, int W,
                                           int lane) {
  bool high[S];
  bool anym = false, anyh = false;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    const float t = (tau_pos && i < W) ? tau_pos[i] : tau;
    high[s] = r.msk[s] && (r.conf[s] > t);
    anym |= r.msk[s] != 0;
    anyh |= high[s];
  }
  if (!__any_sync(0xffffffffu, anym)) return kDevEmptyMask;
  if (__any_sync(0xffffffffu, anyh)) {
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (high[s]) {
        r.tok[s] = r.amax[s];
        r.msk[s] = 0;
      }
    return 0;
  }
  // Fallback (Eq. 1 "otherwise"): argmax conf over M_t, lowest position on ties (R5).
  uint32_t kmax = 0u;
#pragma unroll
  for (int s = 0; s < S; ++s) kmax = max(kmax, r.msk[s] ? ordered_bits(r.conf[s]) : 0u);
  const uint32_t best = __reduce_max_sync(0xffffffffu, kmax);
  uint32_t cand = 0xffffffffu;
#pragma unroll
  for (int s = S - 1; s >= 0; --s)
    if (r.msk[s] && ordered_bits(r.conf[s]) == best) cand = (uint32_t)(lane + 32 * s);
  const uint32_t istar = __reduce_min_sync(0xffffffffu, cand);
#pragma unroll
  for (int s = 0; s < S; ++s)
    if ((uint32_t)(lane + 32 * s) == istar) {
      r.tok[s] = r.amax[s];
      r.msk[s] = 0;
    }
  return 0;
}

// Alg. 1 step 2 with one warp: rank of every position of M_B0 under (conf desc,
// position asc) by counting, n = min(k, |M_B0|).  `keys` is 32 S entries of shared scratch.
// Writes branch tables rows 0..n, lookahead_pos[0..k), *n_branches = n + 1.
template <int S>
__device__ __forceinline__ void warp_spawn(const WinRegs<S>& b0, int W, int k, uint64_t* keys,
                                           int32_t* br_tok, uint8_t* br_msk, int32_t* look,
                                           int32_t* n_branches, int lane) {
  // key = ordered conf bits << 32 | (32 S - 1 - i): larger key = earlier in the order.
  int n_mb0 = 0;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    keys[i] = b0.msk[s] ? (((uint64_t)ordered_bits(b0.conf[s]) << 32) | (uint64_t)(32 * S - 1 - i))
                        : 0ull;
    n_mb0 += __popc(__ballot_sync(0xffffffffu, b0.msk[s]));
  }
  __syncwarp();
  const int n = min(k, n_mb0);
  int rank[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const uint64_t mine = keys[lane + 32 * s];
    int cnt = 0;
#pragma unroll 8
    for (int q = 0; q < 32 * S; ++q) cnt += (keys[q] > mine) ? 1 : 0;
    rank[s] = b0.msk[s] ? cnt : 1 << 20;
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    if (rank[s] < n && look) look[rank[s]] = i;
  }
  if (look)
    for (int q = n + lane; q < k; q += 32) look[q] = -1;
  for (int j = 0; j <= n; ++j) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane + 32 * s;
      if (i < W) {
        const bool fill = (j >= 1) && (rank[s] == j - 1);
        br_tok[(size_t)j * W + i] = fill ? b0.amax[s] : b0.tok[s];
        br_msk[(size_t)j * W + i] = fill ? 0 : (uint8_t)b0.msk[s];
      }
    }
  }
  if (lane == 0) *n_branches = n + 1;
}

// Store the window registers to a table row.
template <int S>
__device__ __forceinline__ void store_window(const WinRegs<S>& r, int32_t* tok, uint8_t* msk, int W,
                                             int lane) {
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int i = lane + 32 * s;
    if (i < W) {
      tok[i] = r.tok[s];
      msk[i] = (uint8_t)r.msk[s];
    }
  }
}

}  // namespace lopa
