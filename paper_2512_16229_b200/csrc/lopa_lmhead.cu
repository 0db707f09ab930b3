// NEXT-4: the LM-head GEMM with the confidence reduction fused into its
// epilogue, so the logits never touch HBM.
//
//   logits[r][v] = sum_k hidden[r][k] * weight[v][k]          (the model's output projection)
//   conf[r]      = 1 / sum_v exp(logits[r][v] - max_v logits[r][v])   (Conf; R1, R2)
//   argmax[r]    = lowest v with logits[r][v] = max                    (R3, R4)
//
// On tcgen05 (sm_100a): one persistent CTA per SM owns a contiguous vocabulary range and
// streams its weight rows once (TMA, SWIZZLE_128B, L2 evict_first); the hidden states (all
// rows, <= 256) are re-read per tile from L2 (evict_last).  Accumulators live in TMEM:
// rows = MMA M (two 128-row halves), vocab = MMA N (<= 256 per tile), K in steps of 16.
// Warp roles: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (one elected lane),
// warps 2..9 epilogue (tcgen05.ld, one thread per row: an online max / exp-sum / argmax over
// the tile's columns, carried across the CTA's tiles).  Each CTA writes one (m, s, argmax)
// partial per row; lopa_lmhead_fold_kernel folds the per-CTA partials of a row in fixed order.
//
// Precision: bf16 inputs, fp32 accumulation in TMEM (the logits are never rounded to bf16);
// the tolerance against the fp64 oracle is derived in DESIGN.md §4 (reading R27).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "liblopa.h"
#include "lopa_internal.h"
#include "lopa_ptx.cuh"

namespace lopa {
namespace lmh {

constexpr int kBK = 64;                    // K elements per stage (= one 128-byte swizzle row)
constexpr int kMaxRows = 256;              // two M = 128 halves
constexpr int kMaxN = 256;                 // vocabulary columns per tile
constexpr int kStages = 3;
constexpr int kHalfBytes = 128 * kBK * 2;  // 16 KB: one 128-row half of A per stage
constexpr int kABytes = 2 * kHalfBytes;
constexpr int kBBytes = kMaxN * kBK * 2;   // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kTmemCols = 512;
constexpr int kMaxGrid = 256;
constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 1024 /*align*/ + 256 +
                              kMaxRows * 16 /*row exchange*/;

// ---- tcgen05 / TMA PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] . B[smem]^T, both K-major, bf16 -> fp32, M = 128, N from idesc.
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on `bar` once every tcgen05 operation issued so far by this thread has completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B (8 rows x 128 B atoms, 1024 B apart).
//   bits [0,14) start >> 4 | [16,30) LBO >> 4 (1: unused for swizzled K-major)
//   [32,46) SBO >> 4 = 64 (1024 B) | [46,48) version = 1 | [61,64) layout = 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t start = (smem_u32(p) >> 4) & 0x3FFFu;
  return start | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor, kind::f16: D fp32 (bits [4,6) = 1), A and B bf16 ([7,10) = [10,13) = 1),
// both K-major, N >> 3 at [17,23), M >> 4 at [24,29).
__device__ __forceinline__ uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// 32 lanes x 32 columns of fp32 from TMEM: thread t of the warp gets row (lane base + t),
// columns [col, col + 32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Optional wait-time accounting (-DLOPA_LMH_PROF): clock64 cycles each role spends waiting,
// per CTA, read back with lopa_debug_lmhead_prof().  Compiled out of the product build.
#ifdef LOPA_LMH_PROF
__device__ unsigned long long g_lmh_prof[kMaxGrid * 8];
#define LMH_T0() const long long _t0 = clock64()
#define LMH_ACC(slot) atomicAdd(&g_lmh_prof[blockIdx.x * 8 + (slot)], (unsigned long long)(clock64() - _t0))
#else
#define LMH_T0() ((void)0)
#define LMH_ACC(slot) ((void)0)
#endif

struct Args {
  int32_t M, K, V;
  int32_t n_half;     // ceil(M / 128)
  int32_t n_units;    // ceil(V / 16): 16-column vocabulary units
  float4* gpart;      // [grid][kMaxRows] per-CTA partials (m, s, argmax bits, -)
  float* conf;
  int32_t* argmax;
  int32_t* dev_status;
  const uint8_t* row_mask;     // nullable: rows with row_mask[r] == 0 are not reported
  const int32_t* n_branches;   // nullable: rows r with r / window >= *n_branches are not reported
  int32_t window;
  int32_t row_base;            // global index of this launch's row 0 (rows > 256 run in chunks)
};

// The vocabulary units of CTA b: [u0, u1) with u = floor(b * n_units / G).
__device__ __forceinline__ void cta_range(int b, int G, int n_units, int* u0, int* u1) {
  *u0 = (int)(((long long)b * n_units) / G);
  *u1 = (int)(((long long)(b + 1) * n_units) / G);
}

// Tile t of a CTA's n_units units (default: 256-column tiles and one narrow remainder).  With
// LOPA_LMH_BALANCED (measured +9 us on the Dream LM head, rejected) the ceil(n_units / 16) tiles get
// near-equal widths (65 units -> 5 x 13, i.e. 208 columns each) instead of full 256-column tiles
// plus one narrow remainder tile whose hidden-state reloads dominate its time.
#ifndef LOPA_LMH_BALANCED
#define LOPA_LMH_BALANCED 0
#endif
__device__ __forceinline__ void tile_cols(int u0, int n_units, int n_tiles, int t, int* v0, int* N) {
#if LOPA_LMH_BALANCED
  const int a = (t * n_units) / n_tiles, e = ((t + 1) * n_units) / n_tiles;
#else
  const int a = 16 * t, e = min(n_units, 16 * t + 16);
#endif
  *v0 = (u0 + a) * 16;
  *N = (e - a) * 16;
}

__global__ void __launch_bounds__(kThreads, 1)
    lopa_lmhead_kernel(const __grid_constant__ CUtensorMap map_a,
                       const __grid_constant__ CUtensorMap map_b256,
                       const __grid_constant__ CUtensorMap map_b16, const Args A) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float4* xch = reinterpret_cast<float4*>(smem + kStages * kStageBytes + 256);  // [kMaxRows]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int n_half = A.n_half;
  const int n_acc = n_half == 1 ? 2 : 1;  // accumulator buffers (512 TMEM columns in total)
  int u0, u1;
  cta_range(b, G, A.n_units, &u0, &u1);
  const int n_tiles = (u1 - u0 + 15) / 16;
  const int nk = A.K / kBK;
#ifdef LOPA_LMH_PROF
  if (tid == 0) g_lmh_prof[blockIdx.x * 8 + 6] = (unsigned long long)clock64();
#endif

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      const uint64_t pol_a = policy_evict_last(), pol_b = policy_evict_first();
      uint32_t it = 0;
      for (int t = 0; t < n_tiles; ++t) {
        int v0, N;
        tile_cols(u0, u1 - u0, n_tiles, t, &v0, &N);
        const uint32_t bytes = (uint32_t)(n_half * kHalfBytes + N * kBK * 2);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = (int)(it % kStages);
          {
            LMH_T0();
            if (it >= (uint32_t)kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
            LMH_ACC(0);
          }
          uint8_t* sa = smem + (size_t)s * kStageBytes;
          uint8_t* sb = sa + kABytes;
          mbar_arrive_expect_tx(&full[s], bytes);
          for (int h = 0; h < n_half; ++h)
            tma_load_2d(sa + h * kHalfBytes, &map_a, kb * kBK, h * 128, &full[s], pol_a);
          if (N == kMaxN) {
            tma_load_2d(sb, &map_b256, kb * kBK, v0, &full[s], pol_b);
          } else {
            for (int j = 0; j < N / 16; ++j)
              tma_load_2d(sb + j * 16 * kBK * 2, &map_b16, kb * kBK, v0 + 16 * j, &full[s], pol_b);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    uint32_t it = 0;
    for (int t = 0; t < n_tiles; ++t) {
      int v0_unused, N;
      tile_cols(u0, u1 - u0, n_tiles, t, &v0_unused, &N);
      const int a = t % n_acc;
      {
        LMH_T0();
        if (t >= n_acc) mbar_wait(&tempty[a], ((t / n_acc) - 1) & 1);
        if (lane == 0) LMH_ACC(1);
      }
      tc_fence_after();
      const uint32_t idesc = idesc_bf16(128, N);
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = (int)(it % kStages);
        {
          LMH_T0();
          mbar_wait(&full[s], (it / kStages) & 1);
          if (lane == 0) LMH_ACC(2);
        }
        tc_fence_after();
        if (lane == 0) {
          const uint8_t* sa = smem + (size_t)s * kStageBytes;
          const uint8_t* sb = sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t bdesc = smem_desc_sw128(sb + kk * 32);
            for (int h = 0; h < n_half; ++h) {
              const uint64_t adesc = smem_desc_sw128(sa + h * kHalfBytes + kk * 32);
              mma_bf16(tmem + (uint32_t)((a * n_half + h) * kMaxN), adesc, bdesc, idesc,
                       (kb | kk) != 0 ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(&tfull[a]);  // accumulator complete
      __syncwarp();
    }
  } else {
    // ---- epilogue: 16 warps; warp w reads TMEM lanes 32 (w % 4) .. +31 (hardware rule).
    // ew = w - 2: bits 0-1 lane quarter (via w % 4), bit 2 = M half, bit 3 = column parity:
    // a thread owns one row and the 32-column chunks of its parity of every tile.
    const int ew = warp - 2;
    const int half = (ew >> 2) & 1;
    const int par = ew >> 3;
    const int q = warp & 3;
    const int row = half * 128 + q * 32 + lane;
    const bool active = half < n_half;
    float m = -INFINITY, ssum = 0.f;
    int am = 0x7FFFFFFF;
    for (int t = 0; t < n_tiles; ++t) {
      int v0, N;
      tile_cols(u0, u1 - u0, n_tiles, t, &v0, &N);
      const int a = t % n_acc;
      {
        LMH_T0();
        mbar_wait(&tfull[a], (t / n_acc) & 1);
        if (lane == 0 && ew == 0) LMH_ACC(3);
      }
#ifdef LOPA_LMH_PROF
      const long long _te = clock64();
#endif
      tc_fence_after();
      if (active) {
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((a * n_half + half) * kMaxN);
        for (int c0 = 32 * par; c0 < N; c0 += 64) {
          float v[32];
          tmem_ld32(base + (uint32_t)c0, v);
          // columns past the tile (N % 32 == 16) or past V are not logits: exp(-inf) = 0
          const int nv = min(min(32, N - c0), A.V - (v0 + c0));
          if (nv < 32) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = i < nv ? v[i] : -INFINITY;
          }
          float cm = v[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) cm = fmax_nan(cm, v[i]);
          if (cm == -INFINITY) continue;  // every term exp(-inf) = 0
          if (cm > m) {  // new running maximum: its first column, and rescale the sum
            int ci = 31;
#pragma unroll
            for (int i = 31; i >= 0; --i) ci = v[i] == cm ? i : ci;
            ssum = (m == -INFINITY) ? 0.f : ssum * ex2((m - cm) * kLog2e);
            m = cm;
            am = v0 + c0 + ci;
          } else if (cm != cm) {
            m = cm;  // NaN: the row is not a distribution (propagates into the sum)
          }
          float2 acc = make_float2(0.f, 0.f);
          const float2 nm = make_float2(-m, -m), l2 = make_float2(kLog2e, kLog2e);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 d = __fmul2_rn(__fadd2_rn(make_float2(v[2 * i], v[2 * i + 1]), nm), l2);
            acc = __fadd2_rn(acc, make_float2(ex2(d.x), ex2(d.y)));
          }
          ssum += acc.x + acc.y;
        }
      }
      tc_fence_before();
      __syncwarp();
#ifdef LOPA_LMH_PROF
      if (lane == 0 && ew == 0) atomicAdd(&g_lmh_prof[blockIdx.x * 8 + 4], (unsigned long long)(clock64() - _te));
#endif
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    // combine the two column parities of each row (fixed order: parity 0 folds parity 1 in)
    if (par == 1) xch[row] = make_float4(m, ssum, __int_as_float(am), 0.f);
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps) : "memory");
    if (par == 0 && active && row < A.M) {
      const float4 o = xch[row];
      const float M = fmax_nan(m, o.x);
      float S = 0.f;
      if (M == -INFINITY || M != M) {
        S = (M != M) ? M : 0.f;
      } else {
        S = ssum * ex2((m - M) * kLog2e) + o.y * ex2((o.x - M) * kLog2e);
      }
      int best = 0x7FFFFFFF;
      if (m == M) best = am;
      if (o.x == M) best = min(best, __float_as_int(o.z));
      A.gpart[(size_t)b * kMaxRows + row] = make_float4(M, S, __int_as_float(best), 0.f);
    }
  }
#ifdef LOPA_LMH_PROF
  if (tid == 0) g_lmh_prof[blockIdx.x * 8 + 5] = (unsigned long long)clock64();
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
  }
  asm volatile("griddepcontrol.launch_dependents;");
}


// ---- CTA-pair form (cta_group::2), rows 129..256 ---------------------------------------------
// A cluster of two CTAs on one TPC computes each 256-row x N-column tile with one
// tcgen05.mma.cta_group::2 (M = 256): CTA rank r holds rows [128 r, 128 r + 128) of the hidden
// states and columns [N/2 r, N/2 (r + 1)) of the tile's weight rows in its shared memory, and
// its TMEM receives its 128 rows x N columns.  So each CTA needs 256 TMEM columns per tile and
// the accumulator is double-buffered (the MMA of tile t + 1 overlaps the epilogue of tile t),
// and every MMA reads half of its operands from each SM's shared memory.  The leader (rank 0)
// issues the MMAs; both CTAs' TMA loads complete on the leader's stage barriers; the commits
// multicast to both CTAs; both epilogues release an accumulator on the leader's barrier.
namespace pair {
#ifndef LOPA_LMH2_STAGES
#define LOPA_LMH2_STAGES 6
#endif
constexpr int kStages = LOPA_LMH2_STAGES;
constexpr int kABytes = 128 * kBK * 2;   // 16 KB: this CTA's 128 rows
constexpr int kBBytes = 128 * kBK * 2;   // 16 KB: this CTA's <= 128 weight rows
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kEpiWarps = 16;            // 4 lane quarters x 4 column groups
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kTmemCols = 512;
constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + 1024 /*align*/ + 256 +
                              3 * 128 * 16 /*column-group exchange*/;
constexpr uint32_t kWaitLimit = 1u << 24;  // bounded waits: a lost arrival traps instead of hanging

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(saddr), "r"(rank));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (uint32_t n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(addr), "r"(parity), "r"(1000u) : "memory");
    if (ok) return;
    if (n == kWaitLimit) asm volatile("trap;");
  }
}
// 2-D tile load into this CTA's shared memory, completing on the leader's barrier (cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t bar_cluster, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` (same offset) in both CTAs of the pair once the issued MMAs completed
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// Tile t of a pair's nu units: ceil(nu / 16) tiles of near-equal width (multiples of 16 columns,
// <= 256), so no tile is a narrow remainder whose hidden-state reloads would not hide under MMA.
// The pair MMA needs N % 32 == 0 (16 weight rows per CTA; measured: N = 16·odd gives wrong
// columns), so an odd-unit tile is computed 16 columns wider (Nm) and the epilogue ignores them.
__device__ __forceinline__ void tile_cols_pair(int u0, int nu, int nt, int t, int* v0, int* N, int* Nm) {
  const int a = (t * nu) / nt, e = ((t + 1) * nu) / nt;
  *v0 = (u0 + a) * 16;
  *N = (e - a) * 16;
  *Nm = (*N + 31) & ~31;
}

// maps: A (box 128 rows); B boxes of 128, 64, 32 and 16 rows (Nm/2 rows = sum of set bits)
struct BMaps {
  CUtensorMap b[4];
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    lopa_lmhead_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                            const __grid_constant__ BMaps maps_b, const Args A) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [2]
  uint64_t* tempty = tfull + 2;        // [2] (the leader's are used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float4* xch = reinterpret_cast<float4*>(smem + kStages * kStageBytes + 256);  // [3][128]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int P = (int)gridDim.x / 2, p = (int)blockIdx.x / 2;
  int u0, u1;
  cta_range(p, P, A.n_units, &u0, &u1);
  const int nu = u1 - u0;
  const int n_tiles = (nu + 15) / 16;
  const int nk = A.K / kBK;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // The weights are constant model parameters: the first stages' weight rows are requested
  // BEFORE the PDL wait, so they stream while the previous kernel (e.g. the previous step's
  // decisions) finishes; the hidden states (a previous kernel's output) and the workspace are
  // touched only after it.
  const uint64_t pol_a = policy_evict_last(), pol_b = policy_evict_first();
  auto load_b = [&](int s, int kb, int vb, int nh, uint32_t bar) {
    uint8_t* sb = smem + (size_t)s * kStageBytes + kABytes;
    int r = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int box = 128 >> i;
      if (nh & box) {
        tma_load_2d_pair(sb + r * kBK * 2, &maps_b.b[i], kb * kBK, vb + r, bar, pol_b);
        r += box;
      }
    }
  };
#ifndef LOPA_LMH_NO_PREWAIT
  const int n_pre = n_tiles > 0 ? min(kStages, nk) : 0;  // stages of tile 0 requested early
#else
  const int n_pre = 0;  // A/B: every load after the wait
#endif
  if (warp == 0 && lane == 0 && n_pre > 0) {
    int v0, N, Nm;
    tile_cols_pair(u0, nu, n_tiles, 0, &v0, &N, &Nm);
    for (int kb = 0; kb < n_pre; ++kb) {
      if (rank == 0) mbar_arrive_expect_tx(&full[kb], (uint32_t)(2 * kABytes + Nm * kBK * 2));
      load_b(kb, kb, v0 + (int)rank * (Nm / 2), Nm / 2, map_to_rank(smem_u32(&full[kb]), 0));
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): this CTA's rows of A and half of the tile's weight rows
      uint32_t it = 0;
      for (int t = 0; t < n_tiles; ++t) {
        int v0, N, Nm;
        tile_cols_pair(u0, nu, n_tiles, t, &v0, &N, &Nm);
        const int nh = Nm / 2;  // weight rows per CTA (multiple of 16)
        const int vb = v0 + (int)rank * nh;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = (int)(it % kStages);
          if (it >= (uint32_t)kStages) wait_bounded(&empty[s], ((it / kStages) - 1) & 1);
          uint8_t* sa = smem + (size_t)s * kStageBytes;
          const uint32_t bar = map_to_rank(smem_u32(&full[s]), 0);
          const bool pre = it < (uint32_t)n_pre;  // weights already requested before the wait
          if (rank == 0 && !pre) mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * kABytes + Nm * kBK * 2));
          tma_load_2d_pair(sa, &map_a, kb * kBK, (int)rank * 128, bar, pol_a);
          if (!pre) load_b(s, kb, vb, nh, bar);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---- MMA issuer (leader only): M = 256 across the pair, N = the tile's columns
      uint32_t it = 0;
      for (int t = 0; t < n_tiles; ++t) {
        int v0_unused, N, Nm;
        tile_cols_pair(u0, nu, n_tiles, t, &v0_unused, &N, &Nm);
        const int a = t & 1;
        if (t >= 2) wait_bounded(&tempty[a], ((t >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t idesc = idesc_bf16(256, Nm);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = (int)(it % kStages);
          wait_bounded(&full[s], (it / kStages) & 1);
          tc_fence_after();
          if (lane == 0) {
            const uint8_t* sa = smem + (size_t)s * kStageBytes;
            const uint8_t* sb = sa + kABytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              mma_bf16_pair(tmem + (uint32_t)(a * 256), smem_desc_sw128(sa + kk * 32),
                            smem_desc_sw128(sb + kk * 32), idesc, (kb | kk) != 0 ? 1u : 0u);
            mma_commit_pair(&empty[s]);  // frees the stage in both CTAs
          }
          __syncwarp();
        }
        if (lane == 0) mma_commit_pair(&tfull[a]);  // accumulator complete in both CTAs
        __syncwarp();
      }
    }
  } else {
    // ---- epilogue: 16 warps; warp w reads TMEM lanes 32 (w % 4) .. +31 (hardware rule);
    // column group g = (w - 2) >> 2 takes the 32-column chunks g, g + 4 of every tile.
    const int ew = warp - 2;
    const int g = ew >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + lane;                 // this CTA's row (TMEM lane)
    const uint32_t tempty_leader = map_to_rank(smem_u32(&tempty[0]), 0);
    float m = -INFINITY, ssum = 0.f;
    int am = 0x7FFFFFFF;
    for (int t = 0; t < n_tiles; ++t) {
      int v0, N, Nm;
      tile_cols_pair(u0, nu, n_tiles, t, &v0, &N, &Nm);
      const int a = t & 1;
      wait_bounded(&tfull[a], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * 256);
      for (int c0 = 32 * g; c0 < N; c0 += 128) {
        float v[32];
        tmem_ld32(base + (uint32_t)c0, v);
        const int nv = min(min(32, N - c0), A.V - (v0 + c0));  // past the tile or V: not logits
        if (nv < 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = i < nv ? v[i] : -INFINITY;
        }
        float cm = v[0];
#pragma unroll
        for (int i = 1; i < 32; ++i) cm = fmax_nan(cm, v[i]);
        if (cm == -INFINITY) continue;
        if (cm > m) {
          int ci = 31;
#pragma unroll
          for (int i = 31; i >= 0; --i) ci = v[i] == cm ? i : ci;
          ssum = (m == -INFINITY) ? 0.f : ssum * ex2((m - cm) * kLog2e);
          m = cm;
          am = v0 + c0 + ci;
        } else if (cm != cm) {
          m = cm;
        }
        float2 acc = make_float2(0.f, 0.f);
        const float2 nm = make_float2(-m, -m), l2 = make_float2(kLog2e, kLog2e);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 d = __fmul2_rn(__fadd2_rn(make_float2(v[2 * i], v[2 * i + 1]), nm), l2);
          acc = __fadd2_rn(acc, make_float2(ex2(d.x), ex2(d.y)));
        }
        ssum += acc.x + acc.y;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_cluster(tempty_leader + (uint32_t)(a * 8));
    }
    // combine the four column groups of each row in fixed order 0, 1, 2, 3
    if (g > 0) xch[(g - 1) * 128 + lrow] = make_float4(m, ssum, __int_as_float(am), 0.f);
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps) : "memory");
    const int row = (int)rank * 128 + lrow;
    if (g == 0 && row < A.M) {
      float4 o[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) o[j] = xch[j * 128 + lrow];
      float M = m;
#pragma unroll
      for (int j = 0; j < 3; ++j) M = fmax_nan(M, o[j].x);
      float S = 0.f;
      int best = 0x7FFFFFFF;
      if (M == -INFINITY || M != M) {
        S = (M != M) ? M : 0.f;
      } else {
        S = ssum * ex2((m - M) * kLog2e);
#pragma unroll
        for (int j = 0; j < 3; ++j) S += o[j].y * ex2((o[j].x - M) * kLog2e);
      }
      if (m == M) best = am;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (o[j].x == M) best = min(best, __float_as_int(o[j].z));
      A.gpart[(size_t)p * kMaxRows + row] = make_float4(M, S, __int_as_float(best), 0.f);
    }
  }
  tc_fence_before();
  cluster_sync_all();  // every MMA, commit and remote arrival of the pair is done
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols)
                 : "memory");
  }
  asm volatile("griddepcontrol.launch_dependents;");
}
}  // namespace pair

// One warp per row: lane l folds the partials l, l + 32, ... in order, then a fixed butterfly.
__global__ void __launch_bounds__(256) lopa_lmhead_fold_kernel(const Args A, int G) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int row = (int)(blockIdx.x * 8 + (threadIdx.x >> 5));
  const int lane = threadIdx.x & 31;
  if (row >= A.M) return;
  // the branch test first: a row of an absent branch never reads the mask (a shard's rows can
  // run past the table's last branch)
  const bool valid = (!A.n_branches || (A.row_base + row) / A.window < *A.n_branches) &&
                     (!A.row_mask || A.row_mask[row] != 0);
  if (!valid) {  // not a row of the step: untouched semantics of a1 (conf NaN, argmax -1)
    if (lane == 0) {
      A.conf[row] = NAN;
      A.argmax[row] = -1;
    }
    return;
  }
  float M = -INFINITY;
  for (int p = lane; p < G; p += 32) M = fmax_nan(M, __ldcg(&A.gpart[(size_t)p * kMaxRows + row]).x);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) M = fmax_nan(M, __shfl_xor_sync(0xffffffffu, M, off));
  float S = 0.f;
  int am = 0x7FFFFFFF;
  for (int p = lane; p < G; p += 32) {
    const float4 q = __ldcg(&A.gpart[(size_t)p * kMaxRows + row]);
    if (q.x == -INFINITY && M == -INFINITY) continue;  // empty range
    S += q.y * ex2((q.x - M) * kLog2e);
    if (q.x == M) am = min(am, __float_as_int(q.z));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    S += __shfl_xor_sync(0xffffffffu, S, off);
    am = min(am, __shfl_xor_sync(0xffffffffu, am, off));
  }
  if (lane == 0) {
    const bool ok = (S >= 1.0f) && !isnan(M);
    A.conf[row] = ok ? __fdiv_rn(1.0f, S) : NAN;
    A.argmax[row] = ok ? am : -1;
    if (!ok) atomicOr(A.dev_status, LOPA_DEV_NONFINITE);
  }
}

// ---- host ------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static std::once_flag once;
  static EncodeTiledFn fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 map over [rows][cols] (row pitch ld elements), box = 64 columns x box_rows rows.
static bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld,
                     int box_rows) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int grid_for(int device) {
  const int n = num_sms(device);
  return n < kMaxGrid ? n : kMaxGrid;
}

// The CTA-pair kernel serves rows 129..256 unless LOPA_LMH_SINGLE=1 (A/B switch).
static bool use_pair_kernel() {
  static const bool on = [] {
    const char* v = getenv("LOPA_LMH_SINGLE");
    return !(v && v[0] == '1');
  }();
  return on;
}

// CTA pairs that can be resident at once (one pair per TPC; an SM without a free partner on its
// TPC stays idle), cached per device.
static int pair_grid_for(int device) {
  static std::mutex mu;
  static int cached[64];
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) return 0;
  if (cached[device] == 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (num_sms(device) / 2));
    cfg.blockDim = dim3(pair::kThreads);
    cfg.dynamicSmemBytes = pair::kSmemBytes;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, pair::lopa_lmhead_pair_kernel, &cfg) != cudaSuccess || n < 1)
      n = num_sms(device) / 2;
    cached[device] = n < kMaxGrid ? n : kMaxGrid;
  }
  return cached[device];
}

}  // namespace lmh
}  // namespace lopa

using namespace lopa;

#ifdef LOPA_LMH_PROF
extern "C" __attribute__((visibility("default"))) int lopa_debug_lmhead_prof(unsigned long long* out, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, lmh::g_lmh_prof, sizeof(unsigned long long) * n * 8);
  static unsigned long long zeros[lmh::kMaxGrid * 8];
  cudaMemcpyToSymbol(lmh::g_lmh_prof, zeros, sizeof(zeros));
  return 0;
}
#endif

extern "C" size_t lopa_lmhead_workspace_bytes(int32_t rows) {
  (void)rows;
  return (size_t)lmh::kMaxGrid * lmh::kMaxRows * sizeof(float4);
}

static int launch_lmhead_chunk(const void* hidden, int64_t ld_hidden, const void* weight,
                               int64_t ld_weight, int32_t rows, int32_t hidden_dim, int32_t vocab,
                               const uint8_t* row_mask, const int32_t* n_branches, int32_t window,
                               int32_t row_base, float* conf, int32_t* argmax, int32_t* dev_status,
                               void* workspace, size_t workspace_bytes, void* stream, bool pair) {
  if (!hidden || !weight || !conf || !argmax || !dev_status || !workspace) return LOPA_ERR_INVALID_ARG;
  if (rows < 1 || rows > lmh::kMaxRows || vocab < 1 || vocab > LOPA_MAX_VOCAB || hidden_dim < lmh::kBK ||
      hidden_dim % lmh::kBK != 0)
    return LOPA_ERR_INVALID_ARG;
  if (ld_hidden < hidden_dim || ld_weight < hidden_dim || ld_hidden % 8 || ld_weight % 8)
    return LOPA_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(hidden) | reinterpret_cast<uintptr_t>(weight)) & 15)
    return LOPA_ERR_INVALID_ARG;
  if (workspace_bytes < lopa_lmhead_workspace_bytes(rows)) return LOPA_ERR_INVALID_ARG;
  int device = -1;
  if (!bind_device(stream, hidden, &device)) return LOPA_ERR_CUDA;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10 || minor != 0) return LOPA_ERR_UNSUPPORTED;
  CUtensorMap ma, mb256, mb16;
  if (!lmh::make_map(&ma, hidden, rows, hidden_dim, ld_hidden, 128) ||
      !lmh::make_map(&mb256, weight, vocab, hidden_dim, ld_weight, 256) ||
      !lmh::make_map(&mb16, weight, vocab, hidden_dim, ld_weight, 16))
    return LOPA_ERR_CUDA;
  // the kernel's shared-memory opt-in is per device context: set once per device
  static std::mutex attr_mu;
  static bool attr_done[64];
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    if (device < 0 || device >= 64) return LOPA_ERR_UNSUPPORTED;
    if (!attr_done[device]) {
      cudaError_t e = cudaFuncSetAttribute(lmh::lopa_lmhead_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)lmh::kSmemBytes);
      if (e != cudaSuccess) return cuda_status(e);
      e = cudaFuncSetAttribute(lmh::pair::lopa_lmhead_pair_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lmh::pair::kSmemBytes);
      if (e != cudaSuccess) return cuda_status(e);
      attr_done[device] = true;
    }
  }
  lmh::Args a;
  a.M = rows;
  a.K = hidden_dim;
  a.V = vocab;
  a.n_half = (rows + 127) / 128;
  a.n_units = (vocab + 15) / 16;
  a.gpart = static_cast<float4*>(workspace);
  a.conf = conf;
  a.argmax = argmax;
  a.dev_status = dev_status;
  a.row_mask = row_mask;
  a.n_branches = n_branches;
  a.window = window < 1 ? 1 : window;
  a.row_base = row_base;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int G = 0;  // partials per row (CTAs, or CTA pairs)
  cudaError_t e = cudaSuccess;
  if (pair) {
    lmh::pair::BMaps mb;
    for (int i = 0; i < 4; ++i)
      if (!lmh::make_map(&mb.b[i], weight, vocab, hidden_dim, ld_weight, 128 >> i)) return LOPA_ERR_CUDA;
    const int pairs = lmh::pair_grid_for(device);
    if (pairs < 1) return LOPA_ERR_CUDA;
    G = pairs;
    // programmatic dependent launch: the CTA pairs become resident and request their first
    // weight stages while the previous kernel on the stream finishes (see the kernel)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(lmh::pair::kThreads);
    cfg.dynamicSmemBytes = lmh::pair::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, lmh::pair::lopa_lmhead_pair_kernel, ma, mb, a);
    if (e != cudaSuccess) return LOPA_ERR_CUDA;
  } else {
    G = lmh::grid_for(device);
    lmh::lopa_lmhead_kernel<<<G, lmh::kThreads, lmh::kSmemBytes, s>>>(ma, mb256, mb16, a);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return LOPA_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((rows + 7) / 8);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, lmh::lopa_lmhead_fold_kernel, a, G);
  return e == cudaSuccess ? LOPA_OK : LOPA_ERR_CUDA;
}

// Rows beyond 256 (e.g. k = 14: 15 branches x 32 positions) run in chunks of 256 rows, each a
// full pass over the weights (stream-ordered; the workspace is reused).
namespace lopa {
int launch_lmhead_rows(const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                       int32_t rows, int32_t hidden_dim, int32_t vocab, const uint8_t* row_mask,
                       const int32_t* n_branches, int32_t window, int32_t row_base, float* conf,
                       int32_t* argmax, int32_t* dev_status, void* workspace, size_t workspace_bytes,
                       void* stream, int32_t kernel_rows) {
  if (rows < 1 || rows > LOPA_MAX_ROWS || !hidden || row_base < 0) return LOPA_ERR_INVALID_ARG;
  // The kernel form (and so the per-row fold structure, i.e. the conf bits) follows
  // kernel_rows -- the whole step's rows -- not this call's: a branch-parallel shard reduces its
  // rows exactly as the one-GPU step does (the CTA pairs serve every pass once the step has more
  // than 128 rows).
  const bool pair = (kernel_rows > 128 || rows > 128) && lmh::use_pair_kernel();
  for (int32_t r0 = 0; r0 < rows; r0 += lmh::kMaxRows) {
    const int32_t rc = rows - r0 < lmh::kMaxRows ? rows - r0 : lmh::kMaxRows;
    const int st = launch_lmhead_chunk(
        static_cast<const uint16_t*>(hidden) + (size_t)r0 * ld_hidden, ld_hidden, weight, ld_weight,
        rc, hidden_dim, vocab, row_mask ? row_mask + r0 : nullptr, n_branches, window, row_base + r0,
        conf ? conf + r0 : nullptr, argmax ? argmax + r0 : nullptr, dev_status, workspace,
        workspace_bytes, stream, pair);
    if (st != LOPA_OK) return st;
  }
  return LOPA_OK;
}
}  // namespace lopa

static int launch_lmhead(const void* hidden, int64_t ld_hidden, const void* weight, int64_t ld_weight,
                         int32_t rows, int32_t hidden_dim, int32_t vocab, const uint8_t* row_mask,
                         const int32_t* n_branches, int32_t window, float* conf, int32_t* argmax,
                         int32_t* dev_status, void* workspace, size_t workspace_bytes, void* stream) {
  return lopa::launch_lmhead_rows(hidden, ld_hidden, weight, ld_weight, rows, hidden_dim, vocab,
                                  row_mask, n_branches, window, 0, conf, argmax, dev_status,
                                  workspace, workspace_bytes, stream, rows);
}

extern "C" int lopa_lmhead_confidence(const void* hidden, int64_t ld_hidden, const void* weight,
                                      int64_t ld_weight, int32_t rows, int32_t hidden_dim,
                                      int32_t vocab, const uint8_t* row_mask, float* conf,
                                      int32_t* argmax, int32_t* dev_status, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  return launch_lmhead(hidden, ld_hidden, weight, ld_weight, rows, hidden_dim, vocab, row_mask,
                       nullptr, 1, conf, argmax, dev_status, workspace, workspace_bytes, stream);
}

extern "C" int lopa_step_lmhead(const lopa_step_args_t* a, const void* hidden, int64_t ld_hidden,
                                const void* weight, int64_t ld_weight, int32_t hidden_dim,
                                void* lmh_workspace, size_t lmh_workspace_bytes, void* stream) {
  if (!a) return LOPA_ERR_INVALID_ARG;
  int st = validate_step_args(a, true, false);
  if (st != LOPA_OK) return st;
  const int64_t rows = (int64_t)a->max_branches * a->window;
  if (rows > LOPA_MAX_ROWS) return LOPA_ERR_UNSUPPORTED;
  st = launch_lmhead(hidden, ld_hidden, weight, ld_weight, (int32_t)rows, hidden_dim, a->vocab,
                     a->branch_mask, a->n_branches, a->window, a->conf, a->argmax, a->dev_status,
                     lmh_workspace, lmh_workspace_bytes, stream);
  if (st != LOPA_OK) return st;
  return launch_step_decide(a, static_cast<cudaStream_t>(stream));
}
