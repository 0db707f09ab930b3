// liblopa core: the fused vocabulary reduction (a1) with its in-kernel tails (a2-a4), the
// standalone decision kernels and the C-ABI entry points.
//
// Kernel design:
//   * A persistent grid of one CTA per SM.  Work units are (masked row, canonical segment)
//     pairs, compacted in-kernel from the masks (no host sync) and split into contiguous runs
//     per CTA, so every SM streams the same number of bytes whatever the row count.
//   * Warp 0 lane 0 is the TMA producer: one cp.async.bulk of <= 16 KB per unit into an
//     8-stage shared-memory ring, completion tracked by mbarrier transaction bytes, L2
//     evict-first (each logit is read exactly once).
//   * Two consumer warpgroups take alternate stages.  Each of the 4 warps of a group reduces a
//     fixed interleaved quarter of the segment from shared memory with 128-bit loads: exact
//     max (max.bf16x2), sum of exp2((x - m) * log2 e) in a fixed tree/sequence, exact first
//     argmax.  The warp's partial (m, s, argmax) goes to the workspace.
//   * The warp that completes a row's last partial folds the row's partials in a fixed order
//     (conf bits depend only on the row's bytes), and the warp that completes the last row
//     runs the tail: Eq. 2 + select, Eq. 1 anchor, top-k spawn (MODE_STEP) or the local
//     branch-parallel record (MODE_BP_LOCAL).
#include <cstdio>
#include <cstring>
#include <mutex>

#include "liblopa.h"
#include "lopa_decide.cuh"
#include "lopa_internal.h"
#include "lopa_ptx.cuh"

namespace lopa {

constexpr int kStages = 8;
constexpr int kConsumerWGs = 2;
constexpr int kThreads = 32 + 128 * kConsumerWGs;
constexpr int kWarps = kThreads / 32;
constexpr int kStageBytes = 16384;
constexpr int kMaxGroups = LOPA_MAX_ROWS / 32;

enum Mode : int { MODE_CONF = 0, MODE_STEP = 1, MODE_BP_LOCAL = 2 };

struct Params {
  const uint16_t* logits;
  int64_t ld;
  int32_t vocab, n_seg, seg_len;
  int32_t n_cand;              // candidate rows (logits rows)
  const uint8_t* row_mask;     // nullable
  const int32_t* n_branches;   // nullable (MODE_CONF)
  int32_t window;
  int32_t branch_base;         // global id of logits branch 0 (BP local)
  int32_t cap;                 // branch capacity of the logits / conf tables
  float* conf;
  int32_t* argmax;
  int32_t* dev_status;
  uint32_t* done_cnt;
  uint32_t* row_cnt;
  float4* partials;
  int mode;
  // tails
  const int32_t* branch_tokens;  // global tables [.. ][W]
  const uint8_t* branch_mask;
  int32_t k;
  float tau;
  float* scores;
  int32_t* winner;
  int32_t* next_tokens;
  uint8_t* next_mask;
  int32_t* lookahead;
  int32_t* n_next;
  uint8_t* record;
};

// ------------------------------------------------------------------ BP record layout
// {f32 best_score, i32 best_id, i32 n_present, i32 b_loc} {f32 scores[round4(b_loc)]}
// {i32 tokens[64]} {f32 conf[64]} {i32 argmax[64]} {u8 mask[64]}
struct RecordView {
  float* best_score;
  int32_t* best_id;
  int32_t* n_present;
  int32_t* b_loc;
  float* scores;
  int32_t* tokens;
  float* conf;
  int32_t* argmax;
  uint8_t* mask;
};
__host__ __device__ inline size_t record_bytes(int32_t b_loc) {
  const size_t b4 = (size_t)((b_loc + 3) / 4) * 4;
  return 16 + 4 * b4 + 3 * 4 * LOPA_MAX_WINDOW + LOPA_MAX_WINDOW;
}
__host__ __device__ inline RecordView record_view(void* base, int32_t b_loc) {
  uint8_t* p = static_cast<uint8_t*>(base);
  const size_t b4 = (size_t)((b_loc + 3) / 4) * 4;
  RecordView v;
  v.best_score = reinterpret_cast<float*>(p);
  v.best_id = reinterpret_cast<int32_t*>(p + 4);
  v.n_present = reinterpret_cast<int32_t*>(p + 8);
  v.b_loc = reinterpret_cast<int32_t*>(p + 12);
  v.scores = reinterpret_cast<float*>(p + 16);
  v.tokens = reinterpret_cast<int32_t*>(p + 16 + 4 * b4);
  v.conf = reinterpret_cast<float*>(p + 16 + 4 * b4 + 4 * LOPA_MAX_WINDOW);
  v.argmax = reinterpret_cast<int32_t*>(p + 16 + 4 * b4 + 8 * LOPA_MAX_WINDOW);
  v.mask = p + 16 + 4 * b4 + 12 * LOPA_MAX_WINDOW;
  return v;
}

// ------------------------------------------------------------------ segment slice reduce
struct Partial {
  float m, s;
  uint32_t a;
};

__device__ __forceinline__ void mask_tail(uint4& v, int nvalid) {
  uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (2 * j >= nvalid) w[j] = (w[j] & 0xFFFF0000u) | 0xFF80u;
    if (2 * j + 1 >= nvalid) w[j] = (w[j] & 0x0000FFFFu) | 0xFF800000u;
  }
  v = make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ float chunk_exp_sum(const uint4& v, float m) {
  // Element order within a 16-byte chunk: e0 = lo(x), e1 = hi(x), e2 = lo(y), ...
  const float e0 = ex2((bf16lo(v.x) - m) * kLog2e);
  const float e1 = ex2((bf16hi(v.x) - m) * kLog2e);
  const float e2 = ex2((bf16lo(v.y) - m) * kLog2e);
  const float e3 = ex2((bf16hi(v.y) - m) * kLog2e);
  const float e4 = ex2((bf16lo(v.z) - m) * kLog2e);
  const float e5 = ex2((bf16hi(v.z) - m) * kLog2e);
  const float e6 = ex2((bf16lo(v.w) - m) * kLog2e);
  const float e7 = ex2((bf16hi(v.w) - m) * kLog2e);
  return ((e0 + e1) + (e2 + e3)) + ((e4 + e5) + (e6 + e7));
}

__device__ __forceinline__ bool chunk_has_nan(const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  bool bad = false;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bad |= isnan(bf16lo(w[j])) | isnan(bf16hi(w[j]));
  }
  return bad;
}

// Warp `wq` (0..3) reduces chunks c = 128 t + 32 wq + lane (t = 0..7) of the stage buffer.
// e0: row element index of the segment's first element.
__device__ __forceinline__ Partial reduce_slice(const uint8_t* stage, int nchunks, int e0,
                                                int vocab, int wq, int lane) {
  const uint4* buf = reinterpret_cast<const uint4*>(stage);
  uint4 v[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int c = 128 * t + 32 * wq + lane;
    v[t] = (c < nchunks) ? lds128(buf + c)
                         : make_uint4(kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2);
  }
  if ((vocab & 7) != 0) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int c = 128 * t + 32 * wq + lane;
      const int nvalid = vocab - (e0 + 8 * c);
      if (c < nchunks && nvalid < 8) mask_tail(v[t], nvalid);
    }
  }
  // exact max: per-chunk bf16x2 max, then across chunks and lanes
  uint32_t cm[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) cm[t] = bmax2(bmax2(v[t].x, v[t].y), bmax2(v[t].z, v[t].w));
  uint32_t mm = cm[0];
#pragma unroll
  for (int t = 1; t < 8; ++t) mm = bmax2(mm, cm[t]);
  const float ml = fmaxf(bf16lo(mm), bf16hi(mm));
  const uint32_t okey = __reduce_max_sync(0xffffffffu, ordered_bits(ml));
  const float m = __uint_as_float((okey & 0x80000000u) ? (okey & 0x7FFFFFFFu) : ~okey);

  Partial p;
  p.m = m;
  if (m == -INFINITY) {  // warp-uniform: every element is -inf (or NaN)
    bool bad = false;
#pragma unroll
    for (int t = 0; t < 8; ++t) bad |= chunk_has_nan(v[t]);
    p.s = __any_sync(0xffffffffu, bad) ? __int_as_float(0x7FC00000) : 0.f;
    p.a = 0xFFFFFFFFu;
    return p;
  }
  // sum of exp in a fixed order: tree inside a chunk, chunks in t order, butterfly over lanes
  float ls = 0.f;
#pragma unroll
  for (int t = 0; t < 8; ++t) ls += chunk_exp_sum(v[t], m);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
  p.s = ls;
  // exact first argmax: only lanes holding the max search their registers
  uint32_t cand = 0xFFFFFFFFu;
  if (ml == m) {
    int tf = 7;
#pragma unroll
    for (int t = 7; t >= 0; --t)
      if (fmaxf(bf16lo(cm[t]), bf16hi(cm[t])) == m) tf = t;
    uint4 w = v[0];
#pragma unroll
    for (int t = 1; t < 8; ++t)
      if (tf == t) w = v[t];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    int ef = 7;
#pragma unroll
    for (int e = 7; e >= 0; --e) {
      const float x = (e & 1) ? bf16hi(ws[e >> 1]) : bf16lo(ws[e >> 1]);
      if (x == m) ef = e;
    }
    cand = (uint32_t)(e0 + 8 * (128 * tf + 32 * wq + lane) + ef);
  }
  p.a = __reduce_min_sync(0xffffffffu, cand);
  return p;
}

// Fold a row's partials (fixed order: lane-sequential over p = lane, lane + 32, ..., then a
// butterfly) -> conf, argmax.  Returns true if the row is not a distribution (R20).
__device__ __forceinline__ bool fold_row(const float4* P, int n_part, int lane, float* conf_out,
                                         int32_t* amax_out) {
  float ml = -INFINITY;
  for (int p = lane; p < n_part; p += 32) ml = fmaxf(ml, __ldcg(P + p).x);
  const uint32_t okey = __reduce_max_sync(0xffffffffu, ordered_bits(ml));
  const float M = __uint_as_float((okey & 0x80000000u) ? (okey & 0x7FFFFFFFu) : ~okey);
  float S = 0.f;
  uint32_t a = 0xFFFFFFFFu;
  for (int p = lane; p < n_part; p += 32) {
    const float4 q = __ldcg(P + p);
    S += q.y * ex2((q.x - M) * kLog2e);
    if (q.x == M) a = min(a, __float_as_uint(q.z));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
  a = __reduce_min_sync(0xffffffffu, a);
  *conf_out = __fdiv_rn(1.0f, S);
  *amax_out = (int32_t)a;
  return !(S >= 1.0f);
}

// ------------------------------------------------------------------ tails (one warp)
__device__ void tail_step(const Params& P, uint64_t* keys, int lane) {
  __threadfence();
  const int W = P.window;
  const int nb = max(0, min(*P.n_branches, P.cap));
  const float score = warp_branch_score(P.conf, P.branch_mask, nb, P.cap, W, lane);
  if (lane < P.cap) P.scores[lane] = score;
  const int w = warp_select(score, lane, nb);
  if (lane == 0) *P.winner = w;
  WinRegs r;
  load_window(r, P.conf + (size_t)w * W, P.argmax + (size_t)w * W,
              P.branch_tokens + (size_t)w * W, P.branch_mask + (size_t)w * W, W, lane);
  const bool any = __ballot_sync(0xffffffffu, r.msk[0] | r.msk[1]) != 0;
  if (!any) {  // R21: the winner is complete
    store_window(r, P.next_tokens, P.next_mask, W, lane);
    if (P.lookahead)
      for (int q = lane; q < P.k; q += 32) P.lookahead[q] = -1;
    if (lane == 0) *P.n_next = 0;
    return;
  }
  warp_anchor(r, P.tau, lane);
  warp_spawn(r, W, P.k, keys, P.next_tokens, P.next_mask, P.lookahead, P.n_next, lane);
}

__device__ void tail_bp_local(const Params& P, int lane) {
  __threadfence();
  const int W = P.window;
  const int nb = max(0, min(*P.n_branches - P.branch_base, P.cap));
  const uint8_t* bmask = P.branch_mask + (size_t)P.branch_base * W;
  const float score = warp_branch_score(P.conf, bmask, nb, P.cap, W, lane);
  RecordView rv = record_view(P.record, P.cap);
  if (lane < P.cap) rv.scores[lane] = score;
  const int w = warp_select(score, lane, nb);
  const float best = __shfl_sync(0xffffffffu, score, w);
  if (lane == 0) {
    *rv.best_score = nb > 0 ? best : -INFINITY;
    *rv.best_id = nb > 0 ? P.branch_base + w : 0x7FFFFFFF;
    *rv.n_present = nb;
    *rv.b_loc = P.cap;
  }
  if (nb == 0) return;
  WinRegs r;
  load_window(r, P.conf + (size_t)w * W, P.argmax + (size_t)w * W,
              P.branch_tokens + (size_t)(P.branch_base + w) * W, bmask + (size_t)w * W, W, lane);
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int i = lane + 32 * s;
    rv.tokens[i] = r.tok[s];
    rv.conf[i] = r.conf[s];
    rv.argmax[i] = r.amax[s];
    rv.mask[i] = (uint8_t)r.msk[s];
  }
}

// ------------------------------------------------------------------ the fused kernel
__global__ void __launch_bounds__(kThreads, 1) lopa_reduce_kernel(const Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint32_t* gbits = reinterpret_cast<uint32_t*>(empty + kStages);
  uint32_t* goff = gbits + kMaxGroups;
  uint32_t* misc = goff + kMaxGroups;  // [0] = n_masked
  uint16_t* row_list = reinterpret_cast<uint16_t*>(misc + 4);
  uint64_t* keys = reinterpret_cast<uint64_t*>(row_list + LOPA_MAX_ROWS);  // [kWarps][64]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarpsPerSeg);
    }
    fence_mbar_init();
  }
  // ---- in-kernel row compaction: rows with mask = 1 of present branches
  const int W = P.window;
  int nb_eff = 0x7FFFFFFF;
  if (P.n_branches) nb_eff = *P.n_branches - P.branch_base;
  const int n_groups = (P.n_cand + 31) >> 5;
  for (int g = warp; g < n_groups; g += kWarps) {
    const int r = g * 32 + lane;
    bool v = r < P.n_cand;
    if (v && P.row_mask) v = P.row_mask[r] != 0;
    if (v && P.n_branches) v = (r / W) < nb_eff;
    const uint32_t bits = __ballot_sync(0xffffffffu, v);
    if (lane == 0) gbits[g] = bits;
  }
  __syncthreads();
  if (warp == 0) {
    // exclusive scan of group popcounts: lane owns groups 4 lane .. 4 lane + 3
    uint32_t c[4], tot = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int g = 4 * lane + q;
      c[q] = g < n_groups ? __popc(gbits[g]) : 0u;
      tot += c[q];
    }
    uint32_t incl = tot;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    uint32_t run = incl - tot;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int g = 4 * lane + q;
      if (g < n_groups) goff[g] = run;
      run += c[q];
    }
    if (lane == 31) misc[0] = incl;
  }
  __syncthreads();
  for (int g = warp; g < n_groups; g += kWarps) {
    const uint32_t bits = gbits[g];
    if ((bits >> lane) & 1u)
      row_list[goff[g] + __popc(bits & ((1u << lane) - 1u))] = (uint16_t)(g * 32 + lane);
  }
  __syncthreads();

  const int n_masked = (int)misc[0];
  if (n_masked == 0) {
    if (blockIdx.x == 0 && warp == 1) {
      if (P.mode == MODE_STEP) tail_step(P, keys + 64 * warp, lane);
      if (P.mode == MODE_BP_LOCAL) tail_bp_local(P, lane);
    }
    return;
  }
  const int n_seg = P.n_seg;
  const int n_part = n_seg * kWarpsPerSeg;
  const long long U = (long long)n_masked * n_seg;
  const long long u0 = U * blockIdx.x / gridDim.x;
  const long long u1 = U * (blockIdx.x + 1) / gridDim.x;
  const int n_local = (int)(u1 - u0);

  if (warp == 0) {
    // ---- TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < n_local; ++i) {
        const long long u = u0 + i;
        const int rc = (int)(u / n_seg);
        const int seg = (int)(u - (long long)rc * n_seg);
        const int row = row_list[rc];
        const int s = i % kStages;
        if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        const int e0 = seg * P.seg_len;
        const int e1 = min(P.vocab, e0 + P.seg_len);
        const uint32_t bytes = (uint32_t)(((e1 - e0 + 7) >> 3) << 4);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(stages + (size_t)s * kStageBytes, P.logits + (size_t)row * P.ld + e0, bytes,
                 &full[s], pol);
      }
    }
    return;
  }
  // ---- consumers
  const int wg = (warp - 1) >> 2;
  const int wq = (warp - 1) & 3;
  for (int i = wg; i < n_local; i += kConsumerWGs) {
    const int s = i % kStages;
    mbar_wait(&full[s], (i / kStages) & 1);
    const long long u = u0 + i;
    const int rc = (int)(u / n_seg);
    const int seg = (int)(u - (long long)rc * n_seg);
    const int row = row_list[rc];
    const int e0 = seg * P.seg_len;
    const int e1 = min(P.vocab, e0 + P.seg_len);
    const int nchunks = (e1 - e0 + 7) >> 3;
    const Partial pr = reduce_slice(stages + (size_t)s * kStageBytes, nchunks, e0, P.vocab, wq, lane);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);

    uint32_t last = 0;
    if (lane == 0) {
      P.partials[(size_t)row * n_part + seg * kWarpsPerSeg + wq] =
          make_float4(pr.m, pr.s, __uint_as_float(pr.a), 0.f);
      __threadfence();
      last = (atomicAdd(&P.row_cnt[row], 1u) == (uint32_t)(n_part - 1)) ? 1u : 0u;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) continue;
    // ---- this warp completed row `row`: fold it
    __threadfence();
    float c;
    int32_t a;
    const bool bad = fold_row(P.partials + (size_t)row * n_part, n_part, lane, &c, &a);
    uint32_t tail = 0;
    if (lane == 0) {
      P.conf[row] = c;
      P.argmax[row] = a;
      if (bad) atomicOr(P.dev_status, kDevNonfinite);
      P.row_cnt[row] = 0;
      if (P.mode != MODE_CONF) {
        __threadfence();
        tail = (atomicAdd(P.done_cnt, 1u) == (uint32_t)(n_masked - 1)) ? 1u : 0u;
      }
    }
    tail = __shfl_sync(0xffffffffu, tail, 0);
    if (!tail) continue;
    if (P.mode == MODE_STEP) tail_step(P, keys + 64 * warp, lane);
    if (P.mode == MODE_BP_LOCAL) tail_bp_local(P, lane);
    if (lane == 0) *P.done_cnt = 0;
  }
}

constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 2 * kStages * 8 +
                              2 * kMaxGroups * 4 + 16 + LOPA_MAX_ROWS * 2 + kWarps * 64 * 8;

// ------------------------------------------------------------------ small decision kernels
__global__ void anchor_kernel(const float* conf, const int32_t* argmax, const int32_t* tokens,
                              const uint8_t* mask, int W, float tau, int32_t* tok_out,
                              uint8_t* msk_out, int32_t* dev_status) {
  const int lane = threadIdx.x;
  WinRegs r;
  load_window(r, conf, argmax, tokens, mask, W, lane);
  const int st = warp_anchor(r, tau, lane);
  if (st && lane == 0) atomicOr(dev_status, st);
  store_window(r, tok_out, msk_out, W, lane);
}

__global__ void spawn_kernel(const float* conf, const int32_t* argmax, const int32_t* tok_b0,
                             const uint8_t* msk_b0, int W, int k, int32_t* br_tok,
                             uint8_t* br_msk, int32_t* look, int32_t* n_branches) {
  __shared__ uint64_t keys[64];
  const int lane = threadIdx.x;
  WinRegs r;
  load_window(r, conf, argmax, tok_b0, msk_b0, W, lane);
  warp_spawn(r, W, k, keys, br_tok, br_msk, look, n_branches, lane);
}

__global__ void verify_kernel(const float* conf, const uint8_t* mask, const int32_t* n_branches,
                              int max_br, int W, float* scores, int32_t* winner) {
  const int lane = threadIdx.x;
  const int nb = max(0, min(*n_branches, max_br));
  const float score = warp_branch_score(conf, mask, nb, max_br, W, lane);
  if (lane < max_br) scores[lane] = score;
  const int w = warp_select(score, lane, nb);
  if (lane == 0) *winner = w;
}

// Global half of a BP step: one warp; lane r reads record r's header.
__global__ void bp_finish_kernel(const Params P, const uint8_t* records, int world, int b_loc,
                                 int n_scores) {
  __shared__ uint64_t keys[64];
  const int lane = threadIdx.x;
  const size_t rb = record_bytes(b_loc);
  float bs = -INFINITY;
  int bid = 0x7FFFFFFF;
  if (lane < world) {
    RecordView rv = record_view(const_cast<uint8_t*>(records) + rb * lane, b_loc);
    bs = *rv.best_score;
    bid = *rv.best_id;
    if (isnan(bs)) bs = -INFINITY;
  }
  // largest score, then smallest global id (R9)
  const uint32_t kb = __reduce_max_sync(0xffffffffu, ordered_bits(bs));
  const uint32_t cand = (ordered_bits(bs) == kb && lane < world) ? (uint32_t)bid : 0xFFFFFFFFu;
  const uint32_t wid = __reduce_min_sync(0xffffffffu, cand);
  // the owner rank of the winner: the lane whose best id is wid
  const uint32_t owner_ballot = __ballot_sync(0xffffffffu, lane < world && (uint32_t)bid == wid);
  const int owner = owner_ballot ? __ffs(owner_ballot) - 1 : 0;
  for (int j = lane; j < n_scores; j += 32) {
    const int r = j / b_loc, jl = j - r * b_loc;
    float v = -INFINITY;
    if (r < world) {
      RecordView rv = record_view(const_cast<uint8_t*>(records) + rb * r, b_loc);
      if (jl < *rv.n_present) v = rv.scores[jl];
    }
    P.scores[j] = v;
  }
  const int W = P.window;
  const bool none = (wid == 0xFFFFFFFFu) || (wid == 0x7FFFFFFFu);
  if (lane == 0) *P.winner = none ? 0 : (int)wid;
  WinRegs r;
  if (none) {  // no branch present anywhere: pass branch 0 through as complete
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int i = lane + 32 * s;
      r.msk[s] = 0;
      r.tok[s] = i < W ? P.branch_tokens[i] : 0;
      r.conf[s] = 0.f;
      r.amax[s] = -1;
    }
  } else {
    RecordView rv = record_view(const_cast<uint8_t*>(records) + rb * owner, b_loc);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int i = lane + 32 * s;
      const bool in = i < W;
      r.msk[s] = in ? (uint32_t)(rv.mask[i] != 0) : 0u;
      r.tok[s] = in ? rv.tokens[i] : 0;
      r.conf[s] = (in && r.msk[s]) ? rv.conf[i] : 0.f;
      r.amax[s] = (in && r.msk[s]) ? rv.argmax[i] : -1;
    }
  }
  const bool any = __ballot_sync(0xffffffffu, r.msk[0] | r.msk[1]) != 0;
  if (!any) {
    store_window(r, P.next_tokens, P.next_mask, W, lane);
    if (P.lookahead)
      for (int q = lane; q < P.k; q += 32) P.lookahead[q] = -1;
    if (lane == 0) *P.n_next = 0;
    return;
  }
  warp_anchor(r, P.tau, lane);
  warp_spawn(r, W, P.k, keys, P.next_tokens, P.next_mask, P.lookahead, P.n_next, lane);
}

// ------------------------------------------------------------------ host helpers
static std::mutex g_mu;
static int g_sms[64];
static bool g_attr[64];

int num_sms(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (device < 0 || device >= 64) return 0;
  if (!g_sms[device]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    g_sms[device] = n;
  }
  return g_sms[device];
}

static int ensure_kernel_attrs(int device) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (device >= 0 && device < 64 && g_attr[device]) return LOPA_OK;
  }
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess)
    return LOPA_ERR_CUDA;
  if (major != 10 || minor != 0) return LOPA_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(lopa_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kSmemBytes) != cudaSuccess)
    return LOPA_ERR_CUDA;
  std::lock_guard<std::mutex> lk(g_mu);
  if (device >= 0 && device < 64) g_attr[device] = true;
  return LOPA_OK;
}

bool bind_device(void* stream, const void* ptr, int* device) {
  int dev = -1;
  if (stream != nullptr) {
    if (cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &dev) != cudaSuccess) dev = -1;
  }
  if (dev < 0 && ptr != nullptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeDevice)
      dev = at.device;
  }
  if (dev < 0) {
    cudaGetLastError();
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
  }
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != dev && cudaSetDevice(dev) != cudaSuccess) return false;
  *device = dev;
  return true;
}

size_t workspace_bytes(int32_t max_rows, int32_t vocab) {
  if (max_rows < 1 || vocab < 1) return 256;
  int32_t ns, sl;
  segmentation(vocab, &ns, &sl);
  const size_t rc = (((size_t)max_rows * 4) + 255) / 256 * 256;
  return 256 + rc + (size_t)max_rows * ns * kWarpsPerSeg * sizeof(float4);
}

bool carve_workspace(void* ws, size_t bytes, int32_t max_rows, int32_t vocab, Workspace* out) {
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255) != 0) return false;
  if (bytes < workspace_bytes(max_rows, vocab)) return false;
  uint8_t* p = static_cast<uint8_t*>(ws);
  const size_t rc = (((size_t)max_rows * 4) + 255) / 256 * 256;
  out->done_cnt = reinterpret_cast<uint32_t*>(p);
  out->row_cnt = reinterpret_cast<uint32_t*>(p + 256);
  out->partials = reinterpret_cast<float4*>(p + 256 + rc);
  return true;
}

static int launch_reduce(const Params& P, int device, cudaStream_t s) {
  int st = ensure_kernel_attrs(device);
  if (st != LOPA_OK) return st;
  const int grid = num_sms(device);
  if (grid <= 0) return LOPA_ERR_CUDA;
  lopa_reduce_kernel<<<grid, kThreads, kSmemBytes, s>>>(P);
  return cuda_status(cudaGetLastError());
}

static bool logits_ok(const void* logits, int64_t ld, int32_t vocab) {
  return logits && vocab >= 1 && ld >= vocab && (ld % 8) == 0 &&
         (reinterpret_cast<uintptr_t>(logits) & 15) == 0;
}

int validate_step_args(const lopa_step_args_t* a, bool need_next) {
  if (!a) return LOPA_ERR_INVALID_ARG;
  if (!logits_ok(a->logits, a->ld, a->vocab)) return LOPA_ERR_INVALID_ARG;
  if (a->window < 1 || a->max_branches < 1 || a->k < 0) return LOPA_ERR_INVALID_ARG;
  if (!(a->tau > 0.f && a->tau <= 1.f)) return LOPA_ERR_INVALID_ARG;
  if (!a->n_branches || !a->branch_tokens || !a->branch_mask || !a->conf || !a->argmax ||
      !a->dev_status || !a->workspace)
    return LOPA_ERR_INVALID_ARG;
  if (need_next && (!a->scores || !a->winner || !a->next_tokens || !a->next_mask ||
                    !a->n_branches_next || (a->k > 0 && !a->lookahead_pos)))
    return LOPA_ERR_INVALID_ARG;
  if (a->window > LOPA_MAX_WINDOW) return LOPA_ERR_UNSUPPORTED;
  if (a->max_branches > LOPA_MAX_BRANCHES || a->k + 1 > LOPA_MAX_BRANCHES)
    return LOPA_ERR_UNSUPPORTED;
  return LOPA_OK;
}

static Params base_params(const lopa_step_args_t* a, const Workspace& ws) {
  Params P;
  memset(&P, 0, sizeof(P));
  P.logits = static_cast<const uint16_t*>(a->logits);
  P.ld = a->ld;
  P.vocab = a->vocab;
  segmentation(a->vocab, &P.n_seg, &P.seg_len);
  P.window = a->window;
  P.n_branches = a->n_branches;
  P.conf = a->conf;
  P.argmax = a->argmax;
  P.dev_status = a->dev_status;
  P.done_cnt = ws.done_cnt;
  P.row_cnt = ws.row_cnt;
  P.partials = ws.partials;
  P.branch_tokens = a->branch_tokens;
  P.branch_mask = a->branch_mask;
  P.k = a->k;
  P.tau = a->tau;
  P.scores = a->scores;
  P.winner = a->winner;
  P.next_tokens = a->next_tokens;
  P.next_mask = a->next_mask;
  P.lookahead = a->lookahead_pos;
  P.n_next = a->n_branches_next;
  return P;
}

int launch_bp_local(const lopa_step_args_t* a, int32_t branch_base, int32_t b_loc, void* record,
                    cudaStream_t s) {
  int st = validate_step_args(a, false);
  if (st != LOPA_OK) return st;
  if (!record || b_loc < 1 || branch_base < 0) return LOPA_ERR_INVALID_ARG;
  if (b_loc > LOPA_MAX_BRANCHES || (int64_t)b_loc * a->window > LOPA_MAX_ROWS)
    return LOPA_ERR_UNSUPPORTED;
  Workspace ws;
  if (!carve_workspace(a->workspace, a->workspace_bytes, b_loc * a->window, a->vocab, &ws))
    return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!bind_device(s, a->logits, &dev)) return LOPA_ERR_CUDA;
  Params P = base_params(a, ws);
  P.mode = MODE_BP_LOCAL;
  P.branch_base = branch_base;
  P.cap = b_loc;
  P.n_cand = b_loc * a->window;
  P.row_mask = a->branch_mask + (size_t)branch_base * a->window;
  P.record = static_cast<uint8_t*>(record);
  return launch_reduce(P, dev, s);
}

int launch_bp_finish(const lopa_step_args_t* a, int32_t b_loc, int32_t world, const void* records,
                     cudaStream_t s) {
  if (!a || !records || b_loc < 1 || world < 1 || world > 32) return LOPA_ERR_INVALID_ARG;
  if (a->window < 1 || a->k < 0 || !(a->tau > 0.f && a->tau <= 1.f)) return LOPA_ERR_INVALID_ARG;
  if (!a->scores || !a->winner || !a->next_tokens || !a->next_mask || !a->n_branches_next ||
      !a->branch_tokens || !a->branch_mask || (a->k > 0 && !a->lookahead_pos))
    return LOPA_ERR_INVALID_ARG;
  if (a->window > LOPA_MAX_WINDOW || a->k + 1 > LOPA_MAX_BRANCHES) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!bind_device(s, records, &dev)) return LOPA_ERR_CUDA;
  Workspace ws{};
  Params P = base_params(a, ws);
  const int n_scores = a->max_branches;
  bp_finish_kernel<<<1, 32, 0, s>>>(P, static_cast<const uint8_t*>(records), world, b_loc,
                                    n_scores);
  return cuda_status(cudaGetLastError());
}

}  // namespace lopa

// =================================================================== C ABI
using namespace lopa;

extern "C" int lopa_version(void) { return LOPA_VERSION; }

extern "C" const char* lopa_status_string(int status) {
  switch (status) {
    case LOPA_OK: return "ok";
    case LOPA_ERR_INVALID_ARG: return "invalid argument";
    case LOPA_ERR_UNSUPPORTED: return "unsupported (size limit or device is not sm_100)";
    case LOPA_ERR_CUDA: return "CUDA error";
    case LOPA_ERR_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

extern "C" size_t lopa_workspace_bytes(int32_t max_rows, int32_t vocab) {
  return lopa::workspace_bytes(max_rows, vocab);
}

extern "C" int32_t lopa_num_segments(int32_t vocab) {
  if (vocab < 1) return 0;
  int32_t ns, sl;
  segmentation(vocab, &ns, &sl);
  return ns;
}

extern "C" int lopa_confidence(const void* logits, int64_t ld, int32_t n_rows, int32_t vocab,
                               const uint8_t* row_mask, float* conf, int32_t* argmax,
                               int32_t* dev_status, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (n_rows < 0) return LOPA_ERR_INVALID_ARG;
  if (!logits_ok(logits, ld, vocab) || !conf || !argmax || !dev_status || !workspace)
    return LOPA_ERR_INVALID_ARG;
  if (n_rows > LOPA_MAX_ROWS) return LOPA_ERR_UNSUPPORTED;
  if (n_rows == 0) return LOPA_OK;
  Workspace ws;
  if (!carve_workspace(workspace, workspace_bytes, n_rows, vocab, &ws)) return LOPA_ERR_INVALID_ARG;
  int dev;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!bind_device(stream, logits, &dev)) return LOPA_ERR_CUDA;
  Params P;
  memset(&P, 0, sizeof(P));
  P.logits = static_cast<const uint16_t*>(logits);
  P.ld = ld;
  P.vocab = vocab;
  segmentation(vocab, &P.n_seg, &P.seg_len);
  P.n_cand = n_rows;
  P.row_mask = row_mask;
  P.window = 1;
  P.conf = conf;
  P.argmax = argmax;
  P.dev_status = dev_status;
  P.done_cnt = ws.done_cnt;
  P.row_cnt = ws.row_cnt;
  P.partials = ws.partials;
  P.mode = MODE_CONF;
  return launch_reduce(P, dev, s);
}

extern "C" int lopa_anchor_fill(const float* conf, const int32_t* argmax, const int32_t* tokens,
                                const uint8_t* mask, int32_t window, float tau,
                                int32_t* tokens_out, uint8_t* mask_out, int32_t* dev_status,
                                void* stream) {
  if (!conf || !argmax || !tokens || !mask || !tokens_out || !mask_out || !dev_status)
    return LOPA_ERR_INVALID_ARG;
  if (window < 1 || !(tau > 0.f && tau <= 1.f)) return LOPA_ERR_INVALID_ARG;
  if (window > LOPA_MAX_WINDOW) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!bind_device(stream, conf, &dev)) return LOPA_ERR_CUDA;
  anchor_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(conf, argmax, tokens, mask, window,
                                                                  tau, tokens_out, mask_out,
                                                                  dev_status);
  return cuda_status(cudaGetLastError());
}

extern "C" int lopa_spawn_branches(const float* conf, const int32_t* argmax,
                                   const int32_t* tokens_b0, const uint8_t* mask_b0,
                                   int32_t window, int32_t k, int32_t* branch_tokens,
                                   uint8_t* branch_mask, int32_t* lookahead_pos,
                                   int32_t* n_branches, void* stream) {
  if (!conf || !argmax || !tokens_b0 || !mask_b0 || !branch_tokens || !branch_mask ||
      !n_branches || (k > 0 && !lookahead_pos))
    return LOPA_ERR_INVALID_ARG;
  if (window < 1 || k < 0) return LOPA_ERR_INVALID_ARG;
  if (window > LOPA_MAX_WINDOW || k + 1 > LOPA_MAX_BRANCHES) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!bind_device(stream, conf, &dev)) return LOPA_ERR_CUDA;
  spawn_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      conf, argmax, tokens_b0, mask_b0, window, k, branch_tokens, branch_mask, lookahead_pos,
      n_branches);
  return cuda_status(cudaGetLastError());
}

extern "C" int lopa_verify_select(const float* conf, const uint8_t* branch_mask,
                                  const int32_t* n_branches, int32_t max_branches,
                                  int32_t window, float* scores, int32_t* winner, void* stream) {
  if (!conf || !branch_mask || !n_branches || !scores || !winner) return LOPA_ERR_INVALID_ARG;
  if (window < 1 || max_branches < 1) return LOPA_ERR_INVALID_ARG;
  if (window > LOPA_MAX_WINDOW || max_branches > LOPA_MAX_BRANCHES) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!bind_device(stream, conf, &dev)) return LOPA_ERR_CUDA;
  verify_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(conf, branch_mask, n_branches,
                                                                  max_branches, window, scores,
                                                                  winner);
  return cuda_status(cudaGetLastError());
}

extern "C" int lopa_step(const lopa_step_args_t* a, void* stream) {
  int st = validate_step_args(a, true);
  if (st != LOPA_OK) return st;
  const int32_t rows = a->max_branches * a->window;
  if (rows > LOPA_MAX_ROWS) return LOPA_ERR_UNSUPPORTED;
  Workspace ws;
  if (!carve_workspace(a->workspace, a->workspace_bytes, rows, a->vocab, &ws))
    return LOPA_ERR_INVALID_ARG;
  int dev;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!bind_device(stream, a->logits, &dev)) return LOPA_ERR_CUDA;
  Params P = base_params(a, ws);
  P.mode = MODE_STEP;
  P.cap = a->max_branches;
  P.n_cand = rows;
  P.row_mask = a->branch_mask;
  return launch_reduce(P, dev, s);
}

extern "C" size_t lopa_bp_record_bytes(int32_t window, int32_t b_loc) {
  (void)window;
  return lopa::record_bytes(b_loc < 1 ? 1 : b_loc);
}

extern "C" int lopa_bp_local(const lopa_step_args_t* args, int32_t branch_base, int32_t b_loc,
                             void* record, void* stream) {
  return launch_bp_local(args, branch_base, b_loc, record, static_cast<cudaStream_t>(stream));
}

extern "C" int lopa_bp_finish(const lopa_step_args_t* args, int32_t b_loc, int32_t world,
                              const void* records, void* stream) {
  return launch_bp_finish(args, b_loc, world, records, static_cast<cudaStream_t>(stream));
}
