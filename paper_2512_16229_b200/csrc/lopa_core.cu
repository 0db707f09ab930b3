// liblopa core: the vocabulary reduction K1 (a1), the fold + decision kernel K2 (a1 fold,
// a2-a4), the standalone decision kernels and the C-ABI entry points.  DESIGN.md §5.
//
// K1 lopa_reduce_kernel (persistent, one CTA per SM but one left to K2):
//   * A row of V logits is cut into canonical segments (<= 8192 elements, 16 KB) and segments
//     into groups of kSegPerItem = 2; a work item is one (group, row) = ONE cp.async.bulk of
//     <= 32 KB into a kStages-deep ring, mbarrier transaction bytes, L2 evict-first.  Items are
//     numbered group-major so the short last group of every row streams at the very end.
//   * CTA b issues its first item (group 0 of row b) before the row masks arrive, then works
//     over items numbered on the valid (masked, present) rows only: item b, then claims from a
//     global counter, two claims in flight (the first two sent before the masks arrive).  K1
//     resets the counter itself (the last producer done claiming zeroes it).
//   * kConsumerWGs consumer warpgroups share the stages (warpgroup w: segment w % 2 of the
//     stages of phase w / 2); each warp reduces an interleaved quarter of its segment with
//     128-bit shared loads: exact max (max.NaN.bf16x2), sum of exp2((x - m) log2 e) with x - m
//     formed exactly by fma.f32.bf16 and packed f32x2 multiplies/adds in a fixed order, exact
//     first argmax; the stage is released once the registers hold it.
//   * The warp completing an item folds its warp partials (fixed order) into one group partial
//     in the workspace ([n_grp][n_cand], group-major).  No atomics per row or segment.
// K2 lopa_tail_kernel<MODE, S> (one CTA, programmatic dependent launch on K1's free SM): stages
//   the tables and builds the masked-row list while K1 streams; after griddepcontrol.wait it
//   bulk-copies the group partials into shared memory, folds each row in a fixed 16-slot tree
//   (conf bits depend only on the row's bytes), then Eq. 2 + select, Eq. 1 anchor and the
//   top-k spawn (MODE_STEP / MODE_DECIDE) or the branch-parallel record (MODE_BP_LOCAL).
//
// Compile-time knobs (A/B builds via build.py --variant; defaults are the measured best):
//   LOPA_STAGES, LOPA_WGS, LOPA_CTAS_PER_SM, LOPA_NO_COMPACT (raw item numbering only),
//   LOPA_SEG_ELEMS,
//   LOPA_SEG_PER_ITEM, LOPA_MBAR_SUSPEND_NS, LOPA_TAIL_THREADS, LOPA_POLY_WORDS (exp2 on the FMA
//   pipe), LOPA_LATE_ARGMAX; experiments only: LOPA_NOCOMPUTE (streaming without arithmetic),
//   LOPA_EXP_NOARGMAX, LOPA_NO_PDL, LOPA_NO_TLB_WARM; LOPA_TIMELINE (per-CTA %globaltimer
//   stamps read by scripts/timeline.py).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>

#include <cuda_bf16.h>

#include "liblopa.h"
#include "lopa_ptx.cuh"
namespace lopa {
// Optional per-CTA timeline (-DLOPA_TIMELINE): %globaltimer stamps of the kernel's phases,
// read back with lopa_debug_timeline().  Compiled out of the product build.
#ifdef LOPA_TIMELINE
constexpr int kTlSlots = 24;
__device__ unsigned long long g_timeline[256 * kTlSlots];
__device__ __forceinline__ void tl_stamp(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_timeline[blockIdx.x * kTlSlots + slot] = t;
}
#define TL(slot) tl_stamp(slot)
__device__ __forceinline__ void tl_max(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMax(&g_timeline[blockIdx.x * kTlSlots + slot], t);
}
#define TLMAX(slot) tl_max(slot)
__device__ __forceinline__ void tl_clk(int slot) { g_timeline[blockIdx.x * kTlSlots + slot] = clock64(); }
// clock64 read issued only once `dep` is available: the store waits for it (scoreboard) and
// the clock read follows in program order
__device__ __forceinline__ void tl_clk_dep(int slot, float dep) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(&g_timeline[blockIdx.x * kTlSlots + slot]),
               "r"(__float_as_uint(dep))
               : "memory");
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  g_timeline[blockIdx.x * kTlSlots + slot] = (unsigned long long)t;
}

#define TLC(slot) tl_clk(slot)
#else
#define TL(slot) ((void)0)
#define TLMAX(slot) ((void)0)
#define TLC(slot) ((void)0)
#endif
// Checked builds (-DLOPA_CHECKED, the library's own sanitizer tier: compute-sanitizer is not
// available on this pool): every global access of the step's kernels is tested against the
// bounds the C ABI's contract implies (liblopa.h), K1's stage ring asserts that a consumer reads
// the stage use it waited for, and K2 / the fold kernel assert that every partial they fold was
// written by THIS launch's K1 (a per-launch epoch stamped into the partial's unused 4th word).
// Violations are counted in device globals read by lopa_debug_check_read().
#ifdef LOPA_CHECKED
__device__ unsigned int g_chk_count;
__device__ unsigned int g_chk_first;
__device__ unsigned int g_chk_sites;
__device__ __noinline__ void chk_fail(int site) {
  if (atomicAdd(&g_chk_count, 1u) == 0) g_chk_first = (unsigned)site;
  atomicOr(&g_chk_sites, 1u << (site & 31));
}
#define LOPA_CHK(cond, site) \
  do {                       \
    if (!(cond)) chk_fail(site); \
  } while (0)
#else
#define LOPA_CHK(cond, site) ((void)0)
#endif
#ifdef LOPA_CHAIN_TL
// experiment: per-step %globaltimer marks of chained steps, indexed by the partial epoch:
// [epoch % 64][0 K1 first CTA start, 1 K1 last CTA end, 2 K2 start, 3 K2 rows folded,
//  4 K2 decisions done, 5 K2 final wait returned, 6 K1 first CTA after its wait]
__device__ unsigned long long g_chain[64][12];
__device__ __forceinline__ unsigned long long ch_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CHMIN(e, s) atomicMin(&g_chain[(e) & 63][(s)], ch_now())
#define CHMAX(e, s) atomicMax(&g_chain[(e) & 63][(s)], ch_now())
#define CHSET(e, s) (g_chain[(e) & 63][(s)] = ch_now())
#elif defined(LOPA_K2_CYC)
// experiment: K2's phase boundaries in SM clock cycles (thread 0 only, no K1 marks;
// scripts/k2_cycles.py)
__device__ unsigned long long g_chain[64][16];
#define CHMIN(e, s) ((void)0)
#define CHMAX(e, s) ((void)0)
#define CHSET(e, s) (g_chain[(e) & 63][(s)] = (unsigned long long)clock64())
__device__ uint32_t g_k2cur;  // the step being marked (set by K2 before its decisions)
#define LOPA_SCORE_MARK(s) \
  do { if (threadIdx.x == 0) g_chain[g_k2cur & 63][(s)] = (unsigned long long)clock64(); } while (0)
#else
#define CHMIN(e, s) ((void)0)
#define CHMAX(e, s) ((void)0)
#define CHSET(e, s) ((void)0)
#endif
}  // namespace lopa
#include "lopa_decide.cuh"
#include "lopa_internal.h"

namespace lopa {

#ifndef LOPA_STAGES
#define LOPA_STAGES 3
#endif
#ifndef LOPA_WGS
#define LOPA_WGS 6
#endif
#ifndef LOPA_CTAS_PER_SM
#define LOPA_CTAS_PER_SM 1
#endif

constexpr int kStages = LOPA_STAGES;      // TMA ring depth (one <= 32 KB work item per stage)
constexpr int kConsumerWGs = LOPA_WGS;    // consumer warpgroups per CTA
constexpr int kThreads = 32 + 128 * kConsumerWGs;
constexpr int kWarps = kThreads / 32;
constexpr int kStageBytes = kSegPerItem * 2 * kSegElems;  // one work item per stage
constexpr int kMaxGroups = LOPA_MAX_ROWS / 32;
#ifdef LOPA_NO_VLIST_SMEM
constexpr int kVlistBytes = 0;
#else
constexpr int kVlistBytes = LOPA_MAX_ROWS * 2;  // K1's valid-row list (uint16)
#endif
constexpr int kPartPerItem = kSegPerItem * kWarpsPerSeg;  // warp partials per work item
constexpr int kItemSlots = 2 * kStages;                   // item partial slots per CTA
constexpr int kWgStride = kConsumerWGs / kSegPerItem;     // stages consumed in parallel
static_assert(kConsumerWGs % kSegPerItem == 0, "warpgroups cover the segments of a stage");
// A warpgroup must consume every use of its stages in order (mbarrier parity waits can only
// tell consecutive phases apart), so each stage belongs to exactly one consumer phase.
static_assert(kStages % kWgStride == 0, "stages must divide evenly among consumer phases");

enum Mode : int { MODE_CONF = 0, MODE_STEP = 1, MODE_BP_LOCAL = 2, MODE_DECIDE = 3, MODE_BP_FUSED = 4 };
// MODE_BP_FUSED: MODE_BP_LOCAL, then the peer-memory exchange and the global select / anchor /
// spawn in the same kernel (lopa_bp_step_p2p: K2 stores its record into every peer over NVLink,
// raises its epoch flag there, waits for every peer's, and finishes the step).
// MODE_DECIDE: conf / argmax already in P.conf / P.argmax (the fused LM-head path); K2 only decides.

struct Params {
  const uint16_t* logits;
  int64_t ld;
  int32_t vocab, n_seg, seg_len, n_grp;  // canonical segmentation (lopa_internal.h)
  int32_t n_cand;              // candidate rows (logits rows)
  const uint8_t* row_mask;     // nullable
  const int32_t* n_branches;   // nullable (MODE_CONF)
  int32_t window;
  int32_t branch_base;         // global id of logits branch 0 (BP local)
  int32_t cap;                 // branch capacity of the logits / conf tables
  int32_t table_rows;          // rows of the replicated branch tables (max_branches; n_rows / 1 for a1 alone)
  int32_t k1_alone;            // K1 launched without a consumer (lopa_debug_reduce_only)
  int32_t prefetch;            // K1 may copy its first item before the PDL wait (lopa_set_logits_prefetch)
  int32_t conf_ready;          // K2 without K1: conf / argmax already in P.conf / P.argmax (the
                               // branch-parallel step from hidden states, lopa_bp_step_lmhead)
  // MODE_BP_FUSED: the peer-memory exchange (lopa_bp_step_p2p)
  uint8_t* const* peer_base;   // device array: every rank's mapped exchange buffer
  int32_t bp_world, bp_rank, bp_b_loc, bp_parity;
  uint32_t bp_epoch;
  int64_t bp_rb, bp_flags_off;
  const int32_t* window_dev;   // nullable: the window read on the device (lopa_d2f_* loop);
                               // n_cand = cap * window then (see with_device_window)
  float* conf;
  int32_t* argmax;
  int32_t* dev_status;
  uint32_t* ctrs;              // [0] work-item counter, [1] producers done (K1 self-reset)
  float4* gpart;               // [n_grp][n_cand] group partials (m, s, argmax bits, -), group-major
  int mode;
  // tails
  const int32_t* branch_tokens;  // global tables [.. ][W]
  const uint8_t* branch_mask;
  int32_t k;
  float tau;
  const float* tau_pos;        // nullable: per-position Eq. 1 thresholds of the window (D2F)
  int32_t metric;              // branch-confidence metric (kMetric*)
  float metric_param;          // window w (sliding) or eta (bottom fraction)
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

// Programmatic dependent launch (PDL): the next kernel in the stream may launch early; its
// griddepcontrol.wait returns once this grid's memory operations are visible.
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// A discarded L2 load: warms the address translation (and L2) for a page used later.
__device__ __forceinline__ void touch_global(const void* p) {
  uint32_t d;
  asm volatile("ld.global.cg.u8 %0, [%1];" : "=r"(d) : "l"(p) : "memory");
  asm volatile("" ::"r"(d));
}
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;"); }

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

// (lo - m, hi - m) of a bf16x2 word, each formed exactly as one fp32 rounding of x - m:
// fma.rn.f32.bf16 reads the bf16 halves in place (FHFMA.BF16: no unpack instructions).
__device__ __forceinline__ float2 minus_m(uint32_t w, float negm) {
#ifdef LOPA_MINUS_M_UNPACK
  // experiment: unpack the halves on the integer pipe, one packed fp32 add (the same single
  // rounding of x - m, so the same bits)
  return __fadd2_rn(make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u)),
                    make_float2(negm, negm));
#endif
  float lo, hi;
  asm("{\n.reg .b16 l, h, one;\n"
      "mov.b32 {l, h}, %2;\n"
      "mov.b16 one, 0x3F80;\n"
      "fma.rn.f32.bf16 %0, l, one, %3;\n"
      "fma.rn.f32.bf16 %1, h, one, %3;\n}"
      : "=f"(lo), "=f"(hi)
      : "r"(w), "f"(negm));
  return make_float2(lo, hi);
}

__device__ __forceinline__ float2 ex2x2(float2 d) {
  const float2 z = __fmul2_rn(d, make_float2(kLog2e, kLog2e));
  return make_float2(ex2(z.x), ex2(z.y));
}

// 2^x on the FMA pipe (the "FA4 trick": relieves the MUFU/XU pipe): x = j + f, j = rint(x),
// f in [-0.5, 0.5]; 2^f by a degree-5 fit (max rel. error 3e-7 in fp32, like ex2.approx);
// 2^j added to the exponent field.  x is clamped at -126 (the term is then < 2^-125, far below
// one ulp of the sum S >= 1).  NaN inputs need no care: a NaN in a slice makes its max NaN
// (max.NaN.bf16x2), which poisons the whole slice through the MUFU path.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  const float2 xc = make_float2(fmaxf(x.x, -126.f), fmaxf(x.y, -126.f));
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 r = __fadd2_rn(xc, magic);
  const float2 jf = __fadd2_rn(r, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(xc, make_float2(-jf.x, -jf.y));
  float2 p = make_float2(0.0013260914711281657f, 0.0013260914711281657f);
  p = __ffma2_rn(p, f, make_float2(0.009670180268585682f, 0.009670180268585682f));
  p = __ffma2_rn(p, f, make_float2(0.055507123470306396f, 0.055507123470306396f));
  p = __ffma2_rn(p, f, make_float2(0.2402222454547882f, 0.2402222454547882f));
  p = __ffma2_rn(p, f, make_float2(0.6931470036506653f, 0.6931470036506653f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  const int jx = __float_as_int(r.x) - 0x4B400000, jy = __float_as_int(r.y) - 0x4B400000;
  return make_float2(__int_as_float(__float_as_int(p.x) + (jx << 23)),
                     __int_as_float(__float_as_int(p.y) + (jy << 23)));
}

#ifndef LOPA_POLY_WORDS
#define LOPA_POLY_WORDS 0  // words (of 4 per chunk) whose two exps use ex2_poly2
#endif

// Sum of exp(x - m) over one 16-byte chunk (8 elements), in the fixed packed order
// ((e0,e1) + (e2,e3)) + ((e4,e5) + (e6,e7)) as float2 pairs.  Which words take the polynomial
// is fixed by position, so the result is still a function of the chunk's bytes only.
__device__ __forceinline__ float2 chunk_exp_sum2(const uint4& v, float negm) {
  const float2 L2 = make_float2(kLog2e, kLog2e);
  const float2 p0 = ex2x2(minus_m(v.x, negm));
  const float2 p1 = LOPA_POLY_WORDS >= 3 ? ex2_poly2(__fmul2_rn(minus_m(v.y, negm), L2)) : ex2x2(minus_m(v.y, negm));
  const float2 p2 = LOPA_POLY_WORDS >= 2 ? ex2_poly2(__fmul2_rn(minus_m(v.z, negm), L2)) : ex2x2(minus_m(v.z, negm));
  const float2 p3 = LOPA_POLY_WORDS >= 1 ? ex2_poly2(__fmul2_rn(minus_m(v.w, negm), L2)) : ex2x2(minus_m(v.w, negm));
  return __fadd2_rn(__fadd2_rn(p0, p1), __fadd2_rn(p2, p3));
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

__device__ __forceinline__ float unordered(uint32_t key) {
  return __uint_as_float((key & 0x80000000u) ? (key & 0x7FFFFFFFu) : ~key);
}

// Warp `wq` (0..3) reduces chunks c = 128 t + 32 wq + lane (t = 0..7) of the stage buffer and
// releases the stage (empty_bar) once its shared-memory reads are done.
// e0: row element index of the segment's first element.
__device__ __forceinline__ Partial reduce_slice(const uint8_t* stage, int nchunks, int e0,
                                                int vocab, int wq, int lane, uint64_t* empty_bar) {
  const uint4* buf = reinterpret_cast<const uint4*>(stage);
  uint4 v[kChunksPerLane];
  if (nchunks >= 128 * (kChunksPerLane - 1)) {
    // common case (a full-size segment): only the last chunk of a lane can fall outside
#pragma unroll
    for (int t = 0; t < kChunksPerLane - 1; ++t) v[t] = lds128(buf + 128 * t + 32 * wq + lane);
    const int c = 128 * (kChunksPerLane - 1) + 32 * wq + lane;
    v[kChunksPerLane - 1] = lds128(buf + min(c, nchunks - 1));
    if (c >= nchunks)
      v[kChunksPerLane - 1] = make_uint4(kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2);
  } else {
#pragma unroll
    for (int t = 0; t < kChunksPerLane; ++t) {
      const int c = 128 * t + 32 * wq + lane;
      v[t] = (c < nchunks) ? lds128(buf + c)
                           : make_uint4(kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2);
    }
  }
#ifdef LOPA_NOCOMPUTE
  // streaming experiment: consume the stage and return a dummy partial
  {
    uint32_t acc = 0;
#pragma unroll
    for (int t = 0; t < kChunksPerLane; ++t) acc ^= v[t].x ^ v[t].y ^ v[t].z ^ v[t].w;
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar);
    Partial d;
    d.m = 0.f;
    d.s = 1.0f + (acc == 0x12345678u ? 1.f : 0.f);
    d.a = 0;
    return d;
  }
#endif
  const bool ragged = (vocab & 7) != 0;
  if (ragged) {
#pragma unroll
    for (int t = 0; t < kChunksPerLane; ++t) {
      const int c = 128 * t + 32 * wq + lane;
      const int nvalid = vocab - (e0 + 8 * c);
      if (c < nchunks && nvalid < 8) mask_tail(v[t], nvalid);
    }
  }
  // exact max: per-chunk bf16x2 max, then across chunks and lanes
  uint32_t cm[kChunksPerLane];
#pragma unroll
  for (int t = 0; t < kChunksPerLane; ++t) cm[t] = bmax2(bmax2(v[t].x, v[t].y), bmax2(v[t].z, v[t].w));
  uint32_t mm = cm[0];
#pragma unroll
  for (int t = 1; t < kChunksPerLane; ++t) mm = bmax2(mm, cm[t]);
  const float ml = fmax_nan(bf16lo(mm), bf16hi(mm));  // NaN-propagating, like bmax2
  const float m = unordered(__reduce_max_sync(0xffffffffu, ordered_bits(ml)));

  Partial p;
  p.m = m;
  if (m == -INFINITY) {  // warp-uniform: every element is -inf (or NaN)
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_bar);
    bool bad = false;
#pragma unroll
    for (int t = 0; t < kChunksPerLane; ++t) bad |= chunk_has_nan(v[t]);
    p.s = __any_sync(0xffffffffu, bad) ? __int_as_float(0x7FC00000) : 0.f;
    p.a = 0xFFFFFFFFu;
    return p;
  }
  // exact first argmax: a lane holding the max finds its first chunk containing it and re-reads
  // that chunk from shared memory (the stage is released only afterwards).
  auto argmax_cand = [&]() -> uint32_t {
    uint32_t cand = 0xFFFFFFFFu;
#ifndef LOPA_EXP_NOARGMAX
    if (ml == m) {
      // packed bf16x2 compares against (m, m): m is a bf16 value, and -0 == +0 as in IEEE
      const __nv_bfloat162 m2 = __floats2bfloat162_rn(m, m);
      int tf = kChunksPerLane - 1;
#pragma unroll
      for (int t = kChunksPerLane - 1; t >= 0; --t)
        if (!__hbne2(*reinterpret_cast<const __nv_bfloat162*>(&cm[t]), m2)) tf = t;
      const int c = 128 * tf + 32 * wq + lane;
      uint4 w = lds128(buf + c);
      if (ragged) {
        const int nvalid = vocab - (e0 + 8 * c);
        if (nvalid < 8) mask_tail(w, nvalid);
      }
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      int ef = 7;
#pragma unroll
      for (int j = 3; j >= 0; --j) {
        const unsigned eq = __heq2_mask(*reinterpret_cast<const __nv_bfloat162*>(&ws[j]), m2);
        if (eq) ef = 2 * j + ((eq & 0xFFFFu) ? 0 : 1);
      }
      cand = (uint32_t)(e0 + 8 * c + ef);
    }
#endif
    return cand;
  };
  // sum of exp(x - m) in a fixed order: packed tree inside a chunk, chunks in t order, then
  // (.x + .y), then a butterfly over lanes (identical bits in every lane)
  auto exp_sum = [&]() -> float {
    const float negm = -m;
    float2 acc = chunk_exp_sum2(v[0], negm);
#pragma unroll
    for (int t = 1; t < kChunksPerLane; ++t) acc = __fadd2_rn(acc, chunk_exp_sum2(v[t], negm));
    return acc.x + acc.y;
  };
#ifdef LOPA_LATE_ARGMAX
  float ls = exp_sum();
  const uint32_t cand = argmax_cand();
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_bar);
#else
  const uint32_t cand = argmax_cand();
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_bar);
  float ls = exp_sum();
#endif
  p.a = __reduce_min_sync(0xffffffffu, cand);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
  p.s = ls;
  return p;
}

// ------------------------------------------------------------------ canonical folds
// Fold of partials q[0..n) in index order: M = max m; S = sum_p s_p * 2^((m_p - M) log2 e) in p
// order; argmax = the smallest index among partials with m_p = M.  A partial with m = -inf
// contributes s * 0 = 0 (NaN if it saw a NaN); when M = -inf (every element -inf) the factor is 1,
// so S = sum s = 0 (or NaN) and a row fold reports it as non-finite (R20).
struct FoldAcc {
  float M, S;
  uint32_t a;
};
template <typename Get>
__device__ __forceinline__ FoldAcc fold_seq(int n, Get get) {
  float M = -INFINITY;
#pragma unroll 1
  for (int p = 0; p < n; ++p) M = fmaxf(M, get(p).x);
  FoldAcc r{M, 0.f, 0xFFFFFFFFu};
#pragma unroll 1
  for (int p = 0; p < n; ++p) {
    const float4 q = get(p);
    r.S += q.y * (M == -INFINITY ? 1.f : ex2((q.x - M) * kLog2e));
    if (q.x == M) r.a = min(r.a, __float_as_uint(q.z));
  }
  return r;
}

// Row fold over <= 16 group partials held in registers: M = max (order-free); the terms are
// summed in a fixed 16-slot pairwise tree (slots >= n hold +0, which leaves every sum exact),
// so the result depends only on the partials; argmax = smallest index among partials with m = M.
__device__ __forceinline__ FoldAcc fold_tree16(int n, const float4 (&q)[16]) {
  float M = -INFINITY;
#pragma unroll
  for (int p = 0; p < 16; ++p) M = fmaxf(M, p < n ? q[p].x : -INFINITY);
  float t[16];
  uint32_t a = 0xFFFFFFFFu;
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    // explicit _rn operations: no FMA contraction, so every instantiation (runtime or
    // compile-time n) rounds identically
    t[p] = p < n ? __fmul_rn(q[p].y, M == -INFINITY ? 1.f : ex2(__fmul_rn(__fsub_rn(q[p].x, M), kLog2e)))
                 : 0.f;
    a = (p < n && q[p].x == M) ? min(a, __float_as_uint(q[p].z)) : a;
  }
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
    for (int p = 0; p < w; ++p) t[p] = __fadd_rn(t[2 * p], t[2 * p + 1]);
  return FoldAcc{M, t[0], a};
}

// A step on a device-resident window (lopa_step_args_t.window_dev): the kernel's view of the
// window and candidate rows (cap x W) comes from the device; every other field is unchanged.
__device__ __forceinline__ Params with_device_window(const Params& P0) {
  Params P = P0;
  if (P0.window_dev) {
    const int W = *P0.window_dev;
    P.window = W;
    P.n_cand = P0.cap * W;
  }
  return P;
}

// ------------------------------------------------------------------ group partials
// A group partial (the fold of one (group, row) work item) occupies one 16-byte workspace slot
// as TWO 64-bit words, each single-copy atomic and each stamped with the launch's epoch
// (workspace counter ctrs[2] + 1), so that a reader can tell a partial of THIS launch from a
// stale one without any fence on the writer's side:
//   A = S bits | (M's bf16 bits << 32) | (stamp & 0xFFFF) << 48    (M is a max of bf16 logits:
//       its low 16 bits are zero, so the bf16 bits are lossless)
//   B = argmax | stamp << 32
// K2 therefore folds each row as soon as its partials have landed, while K1 still streams, and
// waits for K1's grid only at its very end (LOPA_NO_K2_POLL: the round-1 hand-off, K2 waits for
// K1's grid before reading the partials).  Epoch protocol: K1 reads e = ctrs[2] after its grid
// dependency wait and stamps e + 1; the launch's consumer (K2, the fold kernel, or K1 itself
// when launched alone) stores ctrs[2] = e + 1 once K1 has completed, so every K1 launch stamps
// a fresh epoch, also across CUDA-graph replays.
__device__ __forceinline__ void store_partial(float4* slot, const FoldAcc& f, uint32_t stamp) {
  const uint64_t A = (uint64_t)__float_as_uint(f.S) | ((uint64_t)(__float_as_uint(f.M) >> 16) << 32) |
                     ((uint64_t)(stamp & 0xFFFFu) << 48);
  const uint64_t B = (uint64_t)f.a | ((uint64_t)stamp << 32);
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(slot), "l"(A), "l"(B) : "memory");
}
__device__ __forceinline__ float4 decode_partial(uint64_t A, uint64_t B) {
  return make_float4(__uint_as_float(((uint32_t)(A >> 32) & 0xFFFFu) << 16), __uint_as_float((uint32_t)A),
                     __uint_as_float((uint32_t)B), 0.f);
}
__device__ __forceinline__ bool stamped(uint64_t A, uint64_t B, uint32_t stamp) {
  return (uint32_t)(B >> 32) == stamp && (uint32_t)(A >> 48) == (stamp & 0xFFFFu);
}
__device__ __forceinline__ void load_stamp_half(const float4* slot, uint64_t* B) {
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(*B) : "l"(reinterpret_cast<const char*>(slot) + 8) : "memory");
}
__device__ __forceinline__ void load_partial_raw(const float4* slot, uint64_t* A, uint64_t* B) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(*A), "=l"(*B) : "l"(slot) : "memory");
}
// A slot staged in shared memory (bulk copy after K1 completed) -> (M, S, argmax bits, -).
__device__ __forceinline__ float4 decode_slot(const float4& q, uint32_t* stamp) {
  const uint64_t A = (uint64_t)__float_as_uint(q.x) | ((uint64_t)__float_as_uint(q.y) << 32);
  const uint64_t B = (uint64_t)__float_as_uint(q.z) | ((uint64_t)__float_as_uint(q.w) << 32);
  *stamp = (uint32_t)(B >> 32);
  return decode_partial(A, B);
}
constexpr uint32_t kPollSpins = 1u << 22;  // ~0.5 s at 100 ns: a K1 that never arrives is an error

// ------------------------------------------------------------------ K2's decision tail
// Everything the decision tail needs, staged in K2's shared memory.
constexpr int kScoreWarps = 8;  // warps scoring branches in the tail
struct TailSmem {
  float conf[LOPA_MAX_ROWS];
  int32_t amax[LOPA_MAX_ROWS];
  int32_t tok[LOPA_MAX_ROWS];
  uint8_t msk[LOPA_MAX_ROWS];
  float scores[LOPA_MAX_BRANCHES];
  uint64_t keys[LOPA_MAX_WINDOW];
  int32_t b0_tok[LOPA_MAX_WINDOW];
  int32_t b0_amax[LOPA_MAX_WINDOW];
  uint8_t b0_msk[LOPA_MAX_WINDOW];
  int32_t rank[LOPA_MAX_WINDOW];
  float taus[LOPA_MAX_WINDOW];  // per-position thresholds (staged from P.tau_pos, if any)
  int32_t n;       // lookahead count, -1 = winner complete
  int32_t best;    // (BP) local best
  uint32_t stamp;  // this launch's partial epoch (timeline builds' marks)
  double dscr[kScoreWarps][LOPA_MAX_WINDOW];  // per-warp metric scratch
  float fscr[kScoreWarps][LOPA_MAX_WINDOW];
};
constexpr size_t kTailBytes = (sizeof(TailSmem) + 127) / 128 * 128;

// Eq. 2 (or a variant) for branches [0, cap) of the staged table (nb present): warp w
// scores branches w, w + NT/32, ... (warp_metric_score: exact fp64 sums).
template <int NT, int S>
__device__ __forceinline__ void cta_scores(TailSmem& T, const Params& P, int nb, int W, int warp,
                                           int lane, float* out) {
  static_assert(NT / 32 >= kScoreWarps, "scoring warps");
  if (warp >= kScoreWarps) return;
  for (int j = warp; j < P.cap; j += kScoreWarps) {
    float sc = -INFINITY;
    if (j < nb)
      sc = warp_metric_score<S>(T.conf + j * W, T.msk + j * W, W, P.metric, P.metric_param,
                                T.dscr[warp], T.fscr[warp], lane);
    if (lane == 0) {
      T.scores[j] = sc;
      if (out) out[j] = sc;
    }
  }
}

// a2 -> a3 -> a4 with the tail CTA (T.conf / T.amax hold the folded rows).  After the scores,
// warps 0..S-1 (32 S threads = one per window position) finish with a named barrier.
template <int NT, int S>
__device__ void cta_tail_step(const Params& P, TailSmem& T, int tid, int nb) {
  // nb = branches present, read by the kernel's prologue (no global load on the tail's path)
  const int warp = tid >> 5, lane = tid & 31;
  const int W = P.window;
  if (nb == 0) {  // no branch (the block was already complete, R21): pass row 0 through
    if (tid < W) {
      P.next_tokens[tid] = P.branch_tokens[tid];
      P.next_mask[tid] = P.branch_mask[tid];
    }
    if (P.lookahead)
      for (int q = tid; q < P.k; q += NT) P.lookahead[q] = -1;
    for (int j = tid; j < P.cap; j += NT) P.scores[j] = -INFINITY;
    if (tid == 0) {
      *P.winner = 0;
      *P.n_next = 0;
    }
    return;
  }
#ifdef LOPA_K2_DEFER_STORES
  // experiment: the scores / winner reach global memory only after the decisions
  cta_scores<NT, S>(T, P, nb, W, warp, lane, nullptr);
#else
  cta_scores<NT, S>(T, P, nb, W, warp, lane, P.scores);
#endif
  if (tid == 0) CHSET(T.stamp, 0);
  __syncthreads();
  if (tid == 0) TLC(22);
  if (tid == 0) CHSET(T.stamp, 7);
  TL(7);
  if (warp >= S) return;
  constexpr int kPos = 32 * S;
  if (warp == 0) {
    const float sc = lane < P.cap ? T.scores[lane] : -INFINITY;
    const int w = warp_select(sc, lane, nb);
    if (lane == 0) CHSET(T.stamp, 1);
    WinRegs<S> r;
#pragma unroll
    for (int h = 0; h < S; ++h) {
      const int i = lane + 32 * h;
      const bool in = i < W;
      r.msk[h] = in ? (uint32_t)T.msk[w * W + i] : 0u;
      r.tok[h] = in ? T.tok[w * W + i] : 0;
      r.conf[h] = in ? T.conf[w * W + i] : 0.f;
      r.amax[h] = in ? T.amax[w * W + i] : -1;
    }
    bool anym = false;
#pragma unroll
    for (int h = 0; h < S; ++h) anym |= r.msk[h] != 0;
    const bool any = __any_sync(0xffffffffu, anym);
    if (any) warp_anchor<S>(r, P.tau, P.tau_pos ? T.taus : nullptr, W, lane);
    if (lane == 0) CHSET(T.stamp, 6);
    int n_mb0 = 0;
#pragma unroll
    for (int h = 0; h < S; ++h) {
      const int i = lane + 32 * h;
      T.b0_tok[i] = r.tok[h];
      T.b0_amax[i] = r.amax[h];
      T.b0_msk[i] = (uint8_t)r.msk[h];
      T.keys[i] = r.msk[h] ? (((uint64_t)ordered_bits(r.conf[h]) << 32) | (uint64_t)(kPos - 1 - i))
                           : 0ull;
      n_mb0 += __popc(__ballot_sync(0xffffffffu, r.msk[h]));
    }
    if (lane == 0) CHSET(T.stamp, 11);
    if (lane == 0) {
#ifdef LOPA_K2_DEFER_STORES
      T.best = w;
#else
      *P.winner = w;
#endif
      T.n = any ? min(P.k, n_mb0) : -1;
    }
  }
  named_bar_sync(1, kPos);
  if (tid == 0) CHSET(T.stamp, 8);
  TL(9);
  const int nl = T.n;
  if (nl < 0) {  // R21: the winner is complete -> pass it through, no branches
    if (tid < W) {
      P.next_tokens[tid] = T.b0_tok[tid];
      P.next_mask[tid] = T.b0_msk[tid];
    }
    if (P.lookahead)
      for (int q = tid; q < P.k; q += kPos) P.lookahead[q] = -1;
    if (tid == 0) *P.n_next = 0;
    return;
  }
  // Alg. 1 step 2: rank of each position of M_B0 under (conf desc, position asc), one thread
  // per position counting the larger keys (broadcast shared-memory reads)
  {
    const int pos = tid;
    const uint64_t mine = T.keys[pos];
    int cnt = 0;
#pragma unroll 16
    for (int q = 0; q < kPos; ++q) cnt += (T.keys[q] > mine) ? 1 : 0;
    const int rk = T.b0_msk[pos] ? cnt : (1 << 20);
    T.rank[pos] = rk;
    LOPA_CHK(rk >= nl || rk < P.k, 8);
    if (rk < nl && P.lookahead) P.lookahead[rk] = pos;
    if (P.lookahead)
      for (int q = nl + tid; q < P.k; q += kPos) P.lookahead[q] = -1;
  }
  named_bar_sync(1, kPos);
  if (tid == 0) CHSET(T.stamp, 9);
  TL(12);
  // next tables: thread = position i, rows j = 0..nl
  if (tid < W) {
    const int i = tid;
    const int32_t tb = T.b0_tok[i], ta = T.b0_amax[i];
    const uint8_t mb = T.b0_msk[i];
    const int rk = T.rank[i];
    for (int j = 0; j <= nl; ++j) {
      const bool fill = (j >= 1) && (rk == j - 1);
      LOPA_CHK(j <= P.k && i < W, 8);
      P.next_tokens[(size_t)j * W + i] = fill ? ta : tb;
      P.next_mask[(size_t)j * W + i] = fill ? (uint8_t)0 : mb;
    }
  }
  if (tid == 0) *P.n_next = nl + 1;
#ifdef LOPA_K2_DEFER_STORES
  if (tid == 0) *P.winner = T.best;
  for (int j = tid; j < P.cap; j += kPos) P.scores[j] = T.scores[j];
#endif
  if (tid == 0) CHSET(T.stamp, 10);
  TL(13);
}

// Local half of a BP step with all threads of K2: local Eq. 2 scores, local best
// (smallest local j with the largest score), and the exchange record.
template <int NT, int S>
__device__ void cta_tail_bp_local(const Params& P, TailSmem& T, int tid, int nb,
                                  uint8_t* record = nullptr) {
  const int warp = tid >> 5, lane = tid & 31;
  const int W = P.window;
  RecordView rv = record_view(record ? record : P.record, P.cap);
  cta_scores<NT, S>(T, P, nb, W, warp, lane, rv.scores);
  __syncthreads();
  if (warp == 0) {
    const float sc = lane < P.cap ? T.scores[lane] : -INFINITY;
    const int w = warp_select(sc, lane, nb);
    if (lane == 0) {
      *rv.best_score = nb > 0 ? T.scores[w] : -INFINITY;
      *rv.best_id = nb > 0 ? P.branch_base + w : 0x7FFFFFFF;
      *rv.n_present = nb;
      *rv.b_loc = P.cap;
      T.best = w;
    }
  }
  __syncthreads();
  const int w = T.best;
  for (int i = tid; i < LOPA_MAX_WINDOW; i += NT) {
    const bool in = i < W && nb > 0;
    rv.tokens[i] = in ? T.tok[w * W + i] : 0;
    rv.conf[i] = in ? T.conf[w * W + i] : 0.f;
    rv.argmax[i] = in ? T.amax[w * W + i] : -1;
    rv.mask[i] = in ? T.msk[w * W + i] : (uint8_t)0;
  }
}

// ------------------------------------------------------------------ the fused kernel
#ifdef LOPA_K1_TL
// experiment: per-item %globaltimer stamps of K1's TMA form (lopa_debug_k1_timeline):
// [cta][0..95]: producer (wait begin, issue) per item < 48; [cta][96 + 48 wg + 3 n + x]:
// consumer warpgroup wg, its n-th stage (full-wait return, release, partial done)
constexpr int kK1TlWords = 96 + 6 * 48;
__device__ unsigned long long g_k1tl[160][kK1TlWords];
__device__ __forceinline__ unsigned long long k1_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K1TL(idx) (g_k1tl[blockIdx.x][(idx)] = k1_gtime())
#else
#define K1TL(idx) ((void)0)
#endif
#ifndef LOPA_NO_PREWAIT
#define LOPA_NO_PREWAIT 0  // A/B: 1 = the first copy waits for the previous kernel (round-1 form)
#endif
#ifndef LOPA_PREWAIT_ITEMS
#define LOPA_PREWAIT_ITEMS 1  // raw items b, G + b, ... copied before the PDL wait (<= kStages)
#endif
// A work claim.  LOPA_TMA_ASM_ATOM: one atom instruction whose value is waited for where it is
// used (atomicAdd is warp-aggregated by the compiler: vote + shuffle of the returned value,
// which waits for the round trip at the call).
#ifndef LOPA_STATIC_PCT
#define LOPA_STATIC_PCT 0
#endif
constexpr int kStaticPct = LOPA_STATIC_PCT;  // % of K1's items assigned statically
#ifndef LOPA_CLAIM_ITEMS
#define LOPA_CLAIM_ITEMS 1  // items per work claim (one atomic returns this many consecutive items)
#endif
constexpr int kClaimItems = LOPA_CLAIM_ITEMS;
#ifdef LOPA_TMA_ASM_ATOM
#define K1_CLAIM(p) atom_add_u32((p), (uint32_t)kClaimItems)
#else
#define K1_CLAIM(p) atomicAdd((p), (uint32_t)kClaimItems)
#endif
__global__ void __launch_bounds__(kThreads, LOPA_CTAS_PER_SM) lopa_reduce_kernel(const Params P_arg) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* slot_free = empty + kStages;
  int4* stage_info = reinterpret_cast<int4*>(slot_free + kItemSlots);
  float4* ipart = reinterpret_cast<float4*>(stage_info + kStages);  // [kItemSlots][kPartPerItem]
  uint32_t* icnt = reinterpret_cast<uint32_t*>(ipart + kItemSlots * kPartPerItem);
  uint32_t* gbits = icnt + kItemSlots;
  uint16_t* vlist = reinterpret_cast<uint16_t*>(gbits + 2 * kMaxGroups);  // [LOPA_MAX_ROWS]
#ifdef LOPA_CHECKED
  uint32_t* stage_seq = reinterpret_cast<uint32_t*>(vlist + LOPA_MAX_ROWS);  // [kStages]
#endif

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) TL(0);

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarpsPerSeg * kSegPerItem);
    }
    for (int q = 0; q < kItemSlots; ++q) mbar_init(&slot_free[q], 1);
    fence_mbar_init();
  }
  for (int q = tid; q < kItemSlots; q += kThreads) icnt[q] = 0;
  const int n_seg = P_arg.n_seg, n_grp = P_arg.n_grp;
  const uint64_t pol = policy_evict_first();
  uint32_t i = 0;  // producer: item (= stage use) sequence number of this CTA
#ifdef LOPA_CHECKED
  int n_cand_chk = P_arg.n_cand;  // the row bound LOPA_CHK tests (the device window's, after the wait)
#endif
  // Issue one work item (group g, row): ONE bulk copy of its <= kSegPerItem segments.  Uses only
  // window-independent fields (logits, ld, segmentation), so it may run before the PDL wait.
  auto issue = [&](int g, int row) {
    const int s0 = g * kSegPerItem, s1 = min(n_seg, s0 + kSegPerItem);
    const int slot = (int)(i % kItemSlots);
    if (i < 48) K1TL(2 * i);
    if (i >= (uint32_t)kItemSlots) mbar_wait(&slot_free[slot], ((i / kItemSlots) - 1) & 1);
    const int s = (int)(i % kStages);
    if (i >= (uint32_t)kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
    if (i < 48) K1TL(2 * i + 1);
    stage_info[s] = make_int4(row, g, slot, s1 - s0);
#ifdef LOPA_CHECKED
    stage_seq[s] = i;
#endif
    const int e0 = s0 * P_arg.seg_len;
    const int e1 = min(P_arg.vocab, s1 * P_arg.seg_len);
    const uint32_t bytes = (uint32_t)(((e1 - e0 + 7) >> 3) << 4);
    LOPA_CHK(row >= 0 && row < n_cand_chk && g >= 0 && g < n_grp && (int64_t)e0 + bytes / 2 <= P_arg.ld, 1);
    mbar_arrive_expect_tx(&full[s], bytes);
    bulk_g2s(stages + (size_t)s * kStageBytes, P_arg.logits + (size_t)row * P_arg.ld + e0, bytes,
             &full[s], pol);
    ++i;
  };
  const int b = blockIdx.x;
  // The first item of CTA b, (0, raw row b), is copied BEFORE the PDL wait when the row count is
  // a launch argument (no device window): the logits are never written by the kernel this one
  // waits for (the previous step's K2 writes tables only; a forward that writes them does not
  // trigger its dependents early), so the copy overlaps the previous kernel's tail — the K2
  // decisions of the previous step, or the previous launch's last CTAs.
#ifndef LOPA_NO_SPEC
  const bool pre_issue = P_arg.window_dev == nullptr && P_arg.prefetch != 0 && !LOPA_NO_PREWAIT;
  if (tid == 0 && pre_issue) {
    if (b < P_arg.n_cand) {
      issue(0, b);
    } else if (b < P_arg.n_cand * n_grp) {
      issue(b / P_arg.n_cand, b % P_arg.n_cand);
    }
#pragma unroll 1
    for (int j = 1; j < LOPA_PREWAIT_ITEMS; ++j) {
      int r = j * (int)gridDim.x + b, g = 0;
      if (r >= P_arg.n_cand * n_grp) break;
      while (r >= P_arg.n_cand) {
        r -= P_arg.n_cand;
        ++g;
      }
      issue(g, r);
    }
  }
  const int n_spec = pre_issue ? LOPA_PREWAIT_ITEMS : 1;  // raw items [0, n_spec G) are covered
#else
  const int n_spec = 0;
#endif
  // PDL: wait for the previous kernel's writes (e.g. the previous step's tables) before touching
  // global inputs, then let the dependent fold/tail kernel launch (it may prefetch the inputs).
  grid_dep_wait();
  grid_dep_launch();
  const Params P = with_device_window(P_arg);  // after the wait: the window was written before
#ifdef LOPA_CHECKED
  n_cand_chk = P.n_cand;
#endif
  const uint32_t stamp = P.ctrs[2] + 1u;          // this launch's partial epoch
  if (tid == 0) CHMIN(stamp, 6);
  // ---- work items: (group g, row).  The first item of CTA b, (0, raw row b), is issued before
  // the row masks arrive (speculatively: a copy of a row that turns out invalid is discarded by
  // the consumers).  Every other item is numbered over the VALID rows only (masked rows of
  // present branches, ascending in vlist[0, n_valid)), group-major, without the group-0 items of
  // rows < G already covered by the speculative copies:
  //   d < n0:  (0, vlist[lo + d])   (lo = valid rows below G, n0 = n_valid - lo)
  //   else:    e = d - n0, (1 + e / n_valid, vlist[e % n_valid])
  // so no claim is ever spent on an unmasked row or an absent branch.  CTA b takes d = b, then
  // claims d = G + counter, two claims in flight (the first two sent before the masks arrive).
  const int W = P.window;
  const int G = (int)gridDim.x;
  const int n_items_cap = P.n_cand * n_grp;
  uint32_t p1 = 0x7FFFFFFFu, p2 = 0x7FFFFFFFu;
  const bool dyn = G < n_items_cap;  // claims can be needed (the exact test follows the masks)
  if (tid == 0) {
    TL(1);
    // raw item b (no division on the common path: the kernel's first instructions are fetched
    // cold at every launch, and an integer-division subroutine there measured +0.35 us)
#ifndef LOPA_NO_SPEC
    if (!pre_issue) {
      if (b < P.n_cand) {
        issue(0, b);
      } else if (b < n_items_cap) {
        issue(b / P.n_cand, b % P.n_cand);
      }
    }
#endif
    // the first two claims travel while the masks load
    if (dyn) {
      p1 = K1_CLAIM(&P.ctrs[0]);
      p2 = K1_CLAIM(&P.ctrs[0]);
    }
  }
  // valid-row bits: mask byte and n_branches loaded independently (one round trip)
  const int n_groups = (P.n_cand + 31) >> 5;
  for (int g = warp; g < n_groups; g += kWarps) {
    const int r = g * 32 + lane;
    const bool in = r < P.n_cand;
    const int nb_eff = P.n_branches ? *P.n_branches - P.branch_base : 0x7FFFFFFF;
    // r / W < nb_eff (no division); the mask byte is read only for rows of present branches,
    // so a rank whose shard runs past the table's last branch never reads beyond it
    bool v = in && (!P.n_branches || (int64_t)r < (int64_t)nb_eff * W);
    if (v && P.row_mask) {
      LOPA_CHK((int64_t)P.branch_base * W + r < (int64_t)P.table_rows * W, 2);
      v = P.row_mask[r] != 0;
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, v);
    if (lane == 0) gbits[g] = bits;
  }
  __syncthreads();
  auto row_valid = [&](int r) -> bool { return (gbits[r >> 5] >> (r & 31)) & 1u; };

  if (warp == 0) {
    // ---- item space.  Items are numbered group-major; the raw items [0, G) (item = group *
    // n_cand + row) are the speculative copies issued above.  Mostly-valid row sets (>= 7/8: e.g.
    // a fresh block) number the other items over the raw rows and skip an invalid row's claim;
    // sparser ones (later iterations of a block, absent branches) number them over the valid
    // rows only, listed ascending in vlist by the producer warp, so that no claim is spent on a
    // row without work.  Every CTA takes the same decision from the same masks.
    int nv = 0;
    for (int w = lane; w < n_groups; w += 32) nv += __popc(gbits[w]);
    const int n_valid = (int)__reduce_add_sync(0xffffffffu, (unsigned)nv);
#ifdef LOPA_NO_COMPACT
    const bool compact = false;
#else
    const bool compact = 8 * n_valid < 7 * P.n_cand;
#endif
    // the speculative copies cover the raw items [0, G): groups < q and rows < rq of group q
    // (computed on the compact path only: no division on the common path, see above)
    int n_rows = P.n_cand, lo = 0, q = 0;
    if (compact) {
#ifdef LOPA_NO_SPEC
      q = 0;  // experiment: no speculative copy, so no raw item is covered
      const int rq = 0;
#else
      q = n_spec * G / P.n_cand;  // n_cand > 0 here (compact implies 7 n_cand > 8 n_valid >= 0)
      const int rq = n_spec * G - q * P.n_cand;
#endif
      n_rows = n_valid;
      int base = 0;
#pragma unroll 1
      for (int w = 0; w < n_groups; ++w) {
        const uint32_t bits = gbits[w];
        if ((bits >> lane) & 1u) vlist[base + __popc(bits & ((1u << lane) - 1u))] = (uint16_t)(32 * w + lane);
        if (32 * w < rq) lo += __popc(32 * w + 32 <= rq ? bits : bits & ((1u << (rq - 32 * w)) - 1u));
        base += __popc(bits);
      }
      __syncwarp();
    }
    if (lane == 0) {
      // ---- TMA producer
      // The first rounds of items are assigned statically (CTA b takes item j G + b of round j:
      // no claim round trip on the producer's path while HBM is saturated); the last
      // ~(100 - LOPA_STATIC_PCT)% are claimed dynamically, two claims in flight, to balance the
      // end of the launch.  The round count depends only on the item count (the same in every CTA).
      if (!compact) {
        // raw rows: items b (issued above), G + b, ..., (S - 1) G + b, then S G + counter ...; an
        // invalid row's item is skipped
        const int n_items = P.n_cand * n_grp;
        const int S = max(max(2, n_spec), (int)((int64_t)n_items * kStaticPct / 100) / G);
        auto maybe_issue = [&](int cur) {
          const int g = cur / P.n_cand, row = cur - g * P.n_cand;
          if (row_valid(row)) issue(g, row);
        };
#ifdef LOPA_NO_SPEC
        if (b < n_items) maybe_issue(b);  // experiment: item b only after the masks
#endif
        for (int jr = max(1, n_spec); jr < S && jr * G + b < n_items; ++jr) maybe_issue(jr * G + b);
        if (dyn) {
          while (true) {
            const int c1 = S * G + (int)p1;
            if (c1 >= n_items) break;
            p1 = K1_CLAIM(&P.ctrs[0]);
            maybe_issue(c1);
#pragma unroll
            for (int u = 1; u < kClaimItems; ++u)
              if (c1 + u < n_items) maybe_issue(c1 + u);
            const int c2 = S * G + (int)p2;
            if (c2 >= n_items) break;
            p2 = K1_CLAIM(&P.ctrs[0]);
            maybe_issue(c2);
#pragma unroll
            for (int u = 1; u < kClaimItems; ++u)
              if (c2 + u < n_items) maybe_issue(c2 + u);
          }
        }
      } else {
        // valid rows only, after the speculatively covered ones:  d < n0: (q, vlist[lo + d]);
        // else e = d - n0: (q + 1 + e / n_valid, vlist[e % n_valid]);  items d = b, G + b, ...,
        // (S - 1) G + b, then d = S G + counter, ...
        const int n0 = q < n_grp ? n_rows - lo : 0;
        const int n_dyn = q < n_grp ? n0 + (n_grp - 1 - q) * n_rows : 0;
        const int S = max(1, (int)((int64_t)n_dyn * kStaticPct / 100) / G);
        auto issue_d = [&](int d) {
          int g = q, x = lo + d;
          if (d >= n0) {
            const int e = d - n0;
            g = q + 1 + e / n_rows;
            x = e - (g - q - 1) * n_rows;
          }
          issue(g, vlist[x]);
        };
        for (int jr = 0; jr < S && jr * G + b < n_dyn; ++jr) issue_d(jr * G + b);
        if (dyn) {
          while (true) {
            const int c1 = S * G + (int)p1;
            if (c1 >= n_dyn) break;
            p1 = K1_CLAIM(&P.ctrs[0]);
            issue_d(c1);
#pragma unroll
            for (int u = 1; u < kClaimItems; ++u)
              if (c1 + u < n_dyn) issue_d(c1 + u);
            const int c2 = S * G + (int)p2;
            if (c2 >= n_dyn) break;
            p2 = K1_CLAIM(&P.ctrs[0]);
            issue_d(c2);
#pragma unroll
            for (int u = 1; u < kClaimItems; ++u)
              if (c2 + u < n_dyn) issue_d(c2 + u);
          }
        }
      }
      // Self-reset of the work counter: every producer, once done claiming (its outstanding
      // claims returned), takes a ticket; the last one zeroes the counter and the tickets, so a
      // launch leaves the workspace zeroed without any follow-up kernel.
      asm volatile("" ::"r"(p1), "r"(p2));
      __threadfence();
      if (atomicAdd(&P.ctrs[1], 1u) == (uint32_t)G - 1) {
        __threadfence();
        P.ctrs[0] = 0;
        P.ctrs[1] = 0;
        // no polling consumer (K1 alone, or the fold kernel, which waits for K1's grid): K1
        // advances the epoch itself
        if (P.k1_alone || P.mode == MODE_CONF) P.ctrs[2] = stamp;
      }
      // end-of-work sentinels: one stage per consumer phase (every warpgroup sees one)
      for (int c = 0; c < kWgStride; ++c, ++i) {
        const int s = (int)(i % kStages);
        if (c == 0) TL(14);
        if (i >= (uint32_t)kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
        stage_info[s] = make_int4(-1, 0, 0, 0);
#ifdef LOPA_CHECKED
        stage_seq[s] = i;
#endif
        mbar_arrive(&full[s]);
      }
    }
  } else {
    // ---- consumers: warpgroup w reduces segment (w % kSegPerItem) of the stages with sequence
    // number = w / kSegPerItem (mod kWgStride)
    const int wg = (warp - 1) >> 2;
    const int wq = (warp - 1) & 3;
    const int jseg = wg % kSegPerItem;
    bool first = true;
#ifdef LOPA_K1_TL
    int tln = 0;
#endif
    for (uint32_t i = wg / kSegPerItem;; i += kWgStride) {
      const int s = (int)(i % kStages);
      mbar_wait(&full[s], (i / kStages) & 1);
#ifdef LOPA_K1_TL
      if (wq == 0 && lane == 0 && tln < 16) K1TL(96 + 48 * wg + 3 * tln);
#endif
      if (first && warp == 1 && lane == 0) TL(2);
      first = false;
      const int4 info = stage_info[s];
      LOPA_CHK(stage_seq[s] == i, 4);  // the stage use this warpgroup waited for, not a refill
      if (info.x < 0) break;
      const int row = info.x, g = info.y, slot = info.z, nsi = info.w;
      if (jseg >= nsi || !row_valid(row)) {  // short item, or a speculative copy of a skipped row
        if (jseg == 0 && wq == 0 && lane == 0 && !row_valid(row)) mbar_arrive(&slot_free[slot]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      }
      const int seg = g * kSegPerItem + jseg;
      const int e0 = seg * P.seg_len;
      const int e1 = min(P.vocab, e0 + P.seg_len);
      const int nchunks = (e1 - e0 + 7) >> 3;
      const Partial pr = reduce_slice(stages + (size_t)s * kStageBytes + (size_t)jseg * P.seg_len * 2,
                                      nchunks, e0, P.vocab, wq, lane, &empty[s]);
#ifdef LOPA_K1_TL
      if (wq == 0 && lane == 0 && tln < 16) { K1TL(96 + 48 * wg + 3 * tln + 2); ++tln; }
#endif
      uint32_t done = 0;
      if (lane == 0) {
        ipart[slot * kPartPerItem + jseg * kWarpsPerSeg + wq] =
            make_float4(pr.m, pr.s, __uint_as_float(pr.a), 0.f);
        __threadfence_block();
        done = (atomicAdd_block(&icnt[slot], 1u) + 1u == (uint32_t)(kWarpsPerSeg * nsi)) ? 1u : 0u;
        if (done) {
          // this warp completed the item: fold its warp partials (fixed order) -> group partial
          __threadfence_block();
          const float4* q = ipart + slot * kPartPerItem;
          const FoldAcc f = fold_seq(kWarpsPerSeg * nsi, [&](int p) { return q[p]; });
          LOPA_CHK(g >= 0 && g < P.n_grp && row >= 0 && row < P.n_cand, 3);
          store_partial(P.gpart + (size_t)g * P.n_cand + row, f, stamp);
          icnt[slot] = 0;
          mbar_arrive(&slot_free[slot]);
        }
      }
    }
    if (lane == 0) TLMAX(3);
  }

  if (tid == 0) TL(4);
  __syncthreads();
  if (tid == 0) CHMAX(stamp, 1);
}

// ------------------------------------------------------------------ K1, warp-staged form
// An experiment kept out of the product build: lopa_k1_ldg.cuh (profiles/r02_k1_ab.md).
#ifdef LOPA_K1_LDG
#include "lopa_k1_ldg.cuh"
#endif


// ------------------------------------------------------------------ K2: fold + decisions
// One CTA, launched programmatically dependent on K1: its launch and prologue overlap K1, and
// griddepcontrol.wait returns once K1's writes are visible.  It folds every masked row's group
// partials in fixed order (conf bits depend only on the row's bytes) and runs the tail.
#ifndef LOPA_TAIL_THREADS
#ifdef LOPA_NO_K2_POLL
#define LOPA_TAIL_THREADS 512
#else
// the polling fold keeps 16 slots' loads in flight per thread: 256 threads leave it 255
// registers (512 threads cap it at 128 and spill; measured 21.96 vs 20.37 us per Dream step)
#define LOPA_TAIL_THREADS 256
#endif
#endif
constexpr int kTailThreads = LOPA_TAIL_THREADS;
#ifndef LOPA_POLL_MAX_ROWS
#define LOPA_POLL_MAX_ROWS (1 << 30)  // masked rows up to which K2 folds by polling (A/B knob)
#endif
// K1's group partials are pulled into K2's shared memory with ONE bulk copy when they fit
// (the Dream step: 10 groups x 256 rows x 16 B = 41 KB): a single L2 round trip instead of
// ten loads per thread.
#ifdef LOPA_NO_K2_POLL
constexpr size_t kGpStageBytes = 64 * 1024;
#else
// polling fold: each thread's 16 decoded partials in a private scratch column ([16][threads])
constexpr size_t kGpStageBytes = (size_t)16 * LOPA_TAIL_THREADS * 16;
#endif
constexpr size_t kTailSmemBytes = kTailBytes + LOPA_MAX_ROWS * 2 + 16 + kGpStageBytes;


// Fold one row's group partials (read straight from the group-major workspace: group g of row r
// at q[g * stride], so the loads of consecutive rows are coalesced; all loads in flight) ->
// conf, argmax.  Fixed order: the 16-slot pairwise tree for n_grp <= 16, sequential beyond.
__device__ __forceinline__ FoldAcc fold_row_global(const float4* q, int n_grp, size_t stride) {
  if (n_grp <= 16) {
    float4 qr[16];
#pragma unroll
    for (int p = 0; p < 16; ++p)
      qr[p] = p < n_grp ? __ldcg(q + p * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
    return fold_tree16(n_grp, qr);
  }
  return fold_seq(n_grp, [&](int p) { return __ldcg(q + p * stride); });
}

// The same fold with the partials staged in shared memory (group g of row r at q[g * stride]).
__device__ __forceinline__ FoldAcc fold_row_smem(const float4* q, int n_grp, int stride) {
  if (n_grp <= 16) {
    float4 qr[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) qr[p] = p < n_grp ? q[p * stride] : make_float4(0.f, 0.f, 0.f, 0.f);
    return fold_tree16(n_grp, qr);
  }
  return fold_seq(n_grp, [&](int p) { return q[p * stride]; });
}

__device__ bool bp_wait_flags(const Params& P, const uint32_t* flags, int world, uint32_t epoch,
                              int lane);
template <int S>
__device__ void bp_finish_warp(const Params& P, const uint8_t* records, int world, int b_loc,
                               int n_scores, uint64_t* keys, int lane);

template <int MODE, int S>
__global__ void __launch_bounds__(kTailThreads, 1) lopa_tail_kernel(const Params P_arg) {
  // launched by K1's launch_dependents, i.e. after K1's own wait: a device window is final
  const Params P = with_device_window(P_arg);
  extern __shared__ __align__(128) uint8_t tsm[];
  TailSmem& T = *reinterpret_cast<TailSmem*>(tsm);
  uint16_t* rows = reinterpret_cast<uint16_t*>(tsm + kTailBytes);  // masked rows, ascending
  uint64_t* gbar = reinterpret_cast<uint64_t*>(tsm + kTailBytes + LOPA_MAX_ROWS * 2);
  float4* gst = reinterpret_cast<float4*>(tsm + kTailBytes + LOPA_MAX_ROWS * 2 + 16);
  float4* pscr = gst;  // polling fold's per-thread scratch (the staged copy is unused then)
  const size_t gbytes = (size_t)P.n_grp * P.n_cand * sizeof(float4);
  // conf / argmax come from the previous kernel (the LM head) instead of K1's partials
  const bool decide_only = MODE == MODE_DECIDE || P.conf_ready != 0;
  const bool staged = !decide_only && gbytes <= kGpStageBytes;
  if (threadIdx.x == 0 && staged) {
    mbar_init(gbar, 1);
    fence_mbar_init();
  }
  // When 16 group slots of every row fit, the slots past n_grp hold neutral partials
  // (m = -inf, s = 0), so the 16-slot fold runs without predicates (identical bits: a neutral
  // slot adds +0 and never matches the maximum).
#ifdef LOPA_NO_K2_POLL
  const bool staged16 = staged && P.n_grp <= 16 && (size_t)P.n_cand * 16 * sizeof(float4) <= kGpStageBytes;
#else
  const bool staged16 = false;  // the polling fold decodes into per-thread scratch instead
#endif
  if (staged16) {
    const float4 neutral = make_float4(-INFINITY, 0.f, __uint_as_float(0xFFFFFFFFu), 0.f);
    for (int e = threadIdx.x; e < (16 - P.n_grp) * P.n_cand; e += kTailThreads)
      gst[(size_t)P.n_grp * P.n_cand + e] = neutral;
  }
  __shared__ uint32_t s_wcnt[kTailThreads / 32 + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = P.window;
  grid_dep_launch();
  // Inputs are not written by K1 (the tables were produced before K1 passed its own wait), so
  // they are staged, and the masked-row list built, while K1 still streams.
  const int nb = max(0, min(*P.n_branches - P.branch_base, P.cap));
  const int nt = nb * W;  // <= LOPA_MAX_ROWS
  const uint8_t* bmask = P.branch_mask + (size_t)P.branch_base * W;
  const int32_t* btok = P.branch_tokens + (size_t)P.branch_base * W;
  constexpr int kRowsPerThread = LOPA_MAX_ROWS / kTailThreads;
  uint32_t mine[kRowsPerThread];  // thread owns a contiguous run of rows (ascending order)
  int cnt = 0;
#pragma unroll
  for (int u = 0; u < kRowsPerThread; ++u) {
    const int idx = kRowsPerThread * tid + u;
    if (idx < nt) LOPA_CHK((int64_t)P.branch_base * W + idx < (int64_t)P.table_rows * W, 5);
    const uint8_t mk = idx < nt ? bmask[idx] : (uint8_t)0;
    if (idx < nt) {
      T.msk[idx] = mk;
      T.tok[idx] = btok[idx];
      T.conf[idx] = 0.f;
      T.amax[idx] = -1;
    }
    mine[u] = mk ? 1u : 0u;
    cnt += mk ? 1 : 0;
  }
  if (P.tau_pos)
    for (int i = tid; i < W; i += kTailThreads) T.taus[i] = P.tau_pos[i];
  // block-wide exclusive scan of the per-thread masked counts -> compacted row list
  int incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) s_wcnt[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = lane < kTailThreads / 32 ? (int)s_wcnt[lane] : 0;
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane < kTailThreads / 32) s_wcnt[lane] = x - v;  // exclusive warp offsets
    if (lane == kTailThreads / 32 - 1) s_wcnt[kTailThreads / 32] = x;
  }
  __syncthreads();
  {
    int pos = (int)s_wcnt[warp] + incl - cnt;
#pragma unroll
    for (int u = 0; u < kRowsPerThread; ++u)
      if (mine[u]) rows[pos++] = (uint16_t)(kRowsPerThread * tid + u);
  }
  const int n_masked = (int)s_wcnt[kTailThreads / 32];
#ifndef LOPA_NO_TLB_WARM
  // Touch the pages K1 writes and this kernel reads or writes after the wait (workspace partials,
  // outputs) so their address translations are cached before the critical path needs them.
  // The values loaded are discarded: nothing read here is used.
  if (warp == kTailThreads / 32 - 1) {
    const size_t gbytes = (size_t)P.n_grp * P.n_cand * sizeof(float4);
    const char* gp = reinterpret_cast<const char*>(P.gpart);
    for (size_t off = (size_t)lane * 65536; off < gbytes; off += 32 * 65536) touch_global(gp + off);
    if (lane == 0) touch_global(P.conf);
    if (lane == 1) touch_global(P.argmax);
    if (lane == 2 && P.scores) touch_global(P.scores);
    if (lane == 3 && P.next_tokens) touch_global(P.next_tokens);
    if (lane == 4 && P.next_mask) touch_global(P.next_mask);
    if (lane == 5 && P.lookahead) touch_global(P.lookahead);
    if (lane == 6 && P.winner) touch_global(P.winner);
    if (lane == 7 && P.n_next) touch_global(P.n_next);
    if (lane == 8) touch_global(P.dev_status);
  }
#endif
  __syncthreads();
  const int n_grp = P.n_grp;
  const uint32_t stamp = P.ctrs[2] + 1u;  // the epoch K1 stamps (ctrs[2] is constant during K1)
  if (tid == 0) CHSET(stamp, 2);
#ifndef LOPA_NO_K2_POLL
  // Polling fold while K1 streams (every step size by default).  The wait-then-fold path below
  // (K1's grid first, then two rows per thread with every load in flight) is the A/B
  // alternative for wide steps (LOPA_POLL_MAX_ROWS=256): measured slower at 481-1945 rows
  // (profiles/r02_k2_phases.md).
  const bool poll = n_masked <= LOPA_POLL_MAX_ROWS;
  if (!decide_only && poll) {
    // Fold every masked row as soon as its n_grp partials of THIS launch have landed (each
    // 64-bit half self-validating, store_partial), while K1 still streams: no grid-wide wait.
    // poll one masked row's n_grp partials and fold them (conf, argmax -> global and T)
    auto poll_fold_row = [&](const int row) {
        const float4* q = P.gpart + row;
        FoldAcc f;
        if (n_grp <= 16) {
          // poll the row's pending slots (all loads in flight at once); a slot whose two halves
          // both carry this launch's epoch is decoded into this thread's scratch column
          uint32_t pend = (1u << n_grp) - 1u;
          for (uint32_t spin = 0;; ++spin) {
#pragma unroll
            for (int h = 0; h < 16; h += 8) {  // two batches of 8 loads in flight
              uint64_t A[8], B[8];
#pragma unroll
              for (int p = 0; p < 8; ++p)
                if ((pend >> (h + p)) & 1u) load_partial_raw(q + (size_t)(h + p) * P.n_cand, &A[p], &B[p]);
#pragma unroll
              for (int p = 0; p < 8; ++p)
                if (((pend >> (h + p)) & 1u) && stamped(A[p], B[p], stamp)) {
                  pscr[(h + p) * kTailThreads + tid] = decode_partial(A[p], B[p]);
                  pend &= ~(1u << (h + p));
                }
            }
            if (!pend) break;
            if (spin >= kPollSpins) {
              atomicOr(P.dev_status, kDevInternal);
              LOPA_CHK(false, 6);
              break;
            }
            __nanosleep(64);
          }
          float4 qr[16];
#pragma unroll
          for (int p = 0; p < 16; ++p)
            qr[p] = (p < n_grp && !((pend >> p) & 1u))
                        ? pscr[p * kTailThreads + tid]
                        : make_float4(-INFINITY, 0.f, __uint_as_float(0xFFFFFFFFu), 0.f);
          f = fold_tree16(n_grp, qr);
        } else {
          // > 16 groups (V > 2^18): poll each partial in turn, then the sequential fold re-reads
          // them (already stamped, so the values are final)
          for (int p = 0; p < n_grp; ++p) {
            uint64_t A, B;
            uint32_t spin = 0;
            for (load_partial_raw(q + (size_t)p * P.n_cand, &A, &B); !stamped(A, B, stamp);
                 load_partial_raw(q + (size_t)p * P.n_cand, &A, &B)) {
              if (++spin >= kPollSpins) {
                atomicOr(P.dev_status, kDevInternal);
                LOPA_CHK(false, 6);
                break;
              }
              __nanosleep(64);
            }
          }
          f = fold_seq(n_grp, [&](int p) {
            uint64_t A, B;
            load_partial_raw(q + (size_t)p * P.n_cand, &A, &B);
            return decode_partial(A, B);
          });
        }
        LOPA_CHK(row < P.n_cand, 7);
        const float c = __fdiv_rn(1.0f, f.S);
        P.conf[row] = c;
        P.argmax[row] = (int32_t)f.a;
        if (!(f.S >= 1.0f)) atomicOr(P.dev_status, kDevNonfinite);
        T.conf[row] = c;
        T.amax[row] = (int32_t)f.a;
    };
#ifndef LOPA_NO_PAIR_POLL
    // Wide steps (more masked rows than threads) with <= 10 groups per row: each thread polls TWO
    // rows at once (rows rc and rc + threads), their decoded partials kept in three planes
    // (m, s, argmax) of the scratch, [20][threads] each -- so a thread's second row no longer
    // waits behind its first.  Same fold (the 16-slot tree), same bits.
    constexpr int kPS = 10;
    if (n_masked > kTailThreads && n_grp <= kPS) {
      float* px = reinterpret_cast<float*>(pscr);
      float* py = px + 2 * kPS * kTailThreads;
      uint32_t* pz = reinterpret_cast<uint32_t*>(py + 2 * kPS * kTailThreads);
      const uint32_t full = (1u << n_grp) - 1u;
      for (int rc = tid; rc < n_masked; rc += 2 * kTailThreads) {
        const int rr[2] = {rows[rc], rc + kTailThreads < n_masked ? rows[rc + kTailThreads] : -1};
        uint32_t pend = full | (rr[1] >= 0 ? full << 16 : 0u);
        for (uint32_t spin = 0;; ++spin) {
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            if (!((pend >> (16 * r)) & full)) continue;
            const float4* q = P.gpart + rr[r];
            uint64_t A[kPS], B[kPS];
#pragma unroll
            for (int p = 0; p < kPS; ++p)
              if ((pend >> (16 * r + p)) & 1u) load_partial_raw(q + (size_t)p * P.n_cand, &A[p], &B[p]);
#pragma unroll
            for (int p = 0; p < kPS; ++p)
              if (((pend >> (16 * r + p)) & 1u) && stamped(A[p], B[p], stamp)) {
                const float4 d = decode_partial(A[p], B[p]);
                const int sl = (r * kPS + p) * kTailThreads + tid;
                px[sl] = d.x;
                py[sl] = d.y;
                pz[sl] = __float_as_uint(d.z);
                pend &= ~(1u << (16 * r + p));
              }
          }
          if (!pend) break;
          if (spin >= kPollSpins) {
            atomicOr(P.dev_status, kDevInternal);
            LOPA_CHK(false, 6);
            break;
          }
          __nanosleep(64);
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          if (rr[r] < 0) continue;
          float4 qr[16];
#pragma unroll
          for (int p = 0; p < 16; ++p) {
            const int sl = (r * kPS + p) * kTailThreads + tid;
            qr[p] = (p < n_grp && !((pend >> (16 * r + p)) & 1u))
                        ? make_float4(px[sl], py[sl], __uint_as_float(pz[sl]), 0.f)
                        : make_float4(-INFINITY, 0.f, __uint_as_float(0xFFFFFFFFu), 0.f);
          }
          const FoldAcc f = fold_tree16(n_grp, qr);
          const int row = rr[r];
          LOPA_CHK(row < P.n_cand, 7);
          const float cf = __fdiv_rn(1.0f, f.S);
          P.conf[row] = cf;
          P.argmax[row] = (int32_t)f.a;
          if (!(f.S >= 1.0f)) atomicOr(P.dev_status, kDevNonfinite);
          T.conf[row] = cf;
          T.amax[row] = (int32_t)f.a;
        }
      }
    } else
#endif
    for (int rc = tid; rc < n_masked; rc += kTailThreads) poll_fold_row(rows[rc]);
  } else if (decide_only) {
    grid_dep_wait();  // decide only: conf / argmax written by the previous kernel
    for (int rc = tid; rc < n_masked; rc += kTailThreads) {
      const int row = rows[rc];
      T.conf[row] = __ldcg(P.conf + row);
      T.amax[row] = __ldcg(P.argmax + row);
    }
  } else {
    grid_dep_wait();  // K1's group partials are final and visible from here on
    // two rows per thread per round, all of their partials' loads in flight together (a wide
    // window has several rows per thread: their L2 round trips overlap instead of adding up)
    auto finish_row = [&](int row, const FoldAcc& f) {
      LOPA_CHK(row < P.n_cand, 7);
      const float c = __fdiv_rn(1.0f, f.S);
      P.conf[row] = c;
      P.argmax[row] = (int32_t)f.a;
      if (!(f.S >= 1.0f)) atomicOr(P.dev_status, kDevNonfinite);
      T.conf[row] = c;
      T.amax[row] = (int32_t)f.a;
    };
    for (int rc = tid; rc < n_masked; rc += 2 * kTailThreads) {
      const int rc2 = rc + kTailThreads;
      const int row0 = rows[rc], row1 = rc2 < n_masked ? rows[rc2] : -1;
      if (n_grp <= 16) {
        float4 q0[16], q1[16];
        uint32_t st_bad = 0;
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          q0[p] = q1[p] = make_float4(-INFINITY, 0.f, __uint_as_float(0xFFFFFFFFu), 0.f);
          if (p < n_grp) {
            uint64_t A, B, A1, B1;
            load_partial_raw(P.gpart + row0 + (size_t)p * P.n_cand, &A, &B);
            if (row1 >= 0) load_partial_raw(P.gpart + row1 + (size_t)p * P.n_cand, &A1, &B1);
            st_bad |= stamped(A, B, stamp) ? 0u : 1u;
            q0[p] = decode_partial(A, B);
            if (row1 >= 0) {
              st_bad |= stamped(A1, B1, stamp) ? 0u : 1u;
              q1[p] = decode_partial(A1, B1);
            }
          }
        }
        LOPA_CHK(!st_bad, 6);
        if (st_bad) atomicOr(P.dev_status, kDevInternal);
        finish_row(row0, fold_tree16(n_grp, q0));
        if (row1 >= 0) finish_row(row1, fold_tree16(n_grp, q1));
      } else {
        for (int rr = 0; rr < 2; ++rr) {
          const int row = rr ? row1 : row0;
          if (row < 0) continue;
          finish_row(row, fold_seq(n_grp, [&](int p) {
            uint64_t A, B;
            load_partial_raw(P.gpart + row + (size_t)p * P.n_cand, &A, &B);
            return decode_partial(A, B);
          }));
        }
      }
    }
  }
  if (tid == 0) { TL(6); TLC(16); }
#else
  grid_dep_wait();  // K1's group partials are visible from here on
  if (tid == 0) { TL(6); TLC(16); }
  if (decide_only) {
    for (int rc = tid; rc < n_masked; rc += kTailThreads) {
      const int row = rows[rc];
      T.conf[row] = __ldcg(P.conf + row);
      T.amax[row] = __ldcg(P.argmax + row);
    }
  } else if (staged) {
    if (tid == 0) {
      mbar_arrive_expect_tx(gbar, (uint32_t)gbytes);
      bulk_g2s(gst, P.gpart, (uint32_t)gbytes, gbar, policy_evict_first());
    }
    mbar_wait(gbar, 0);
    const int stride = P.n_cand;
    for (int rc = tid; rc < n_masked; rc += kTailThreads) {
      const int row = rows[rc];
      float4 qr[16];
      uint32_t st_bad = 0;
      for (int p = 0; p < 16; ++p) {
        uint32_t sp = stamp;
        qr[p] = p < n_grp ? decode_slot(gst[row + p * stride], &sp)
                          : make_float4(-INFINITY, 0.f, __uint_as_float(0xFFFFFFFFu), 0.f);
        st_bad |= sp != stamp;
      }
      LOPA_CHK(!st_bad, 6);
      LOPA_CHK(row < P.n_cand, 7);
      const FoldAcc f = n_grp <= 16 ? fold_tree16(n_grp, qr)
                                    : fold_seq(n_grp, [&](int p) {
                                        uint32_t sp;
                                        return decode_slot(gst[row + p * stride], &sp);
                                      });
      const float c = __fdiv_rn(1.0f, f.S);
      P.conf[row] = c;
      P.argmax[row] = (int32_t)f.a;
      if (!(f.S >= 1.0f)) atomicOr(P.dev_status, kDevNonfinite);
      T.conf[row] = c;
      T.amax[row] = (int32_t)f.a;
    }
  } else
  for (int rc = tid; rc < n_masked; rc += kTailThreads) {
    const int row = rows[rc];
    const FoldAcc f = fold_seq(n_grp, [&](int p) {
      uint64_t A, B;
      load_partial_raw(P.gpart + row + (size_t)p * P.n_cand, &A, &B);
      return decode_partial(A, B);
    });
    const float c = __fdiv_rn(1.0f, f.S);
    P.conf[row] = c;
    P.argmax[row] = (int32_t)f.a;
    if (!(f.S >= 1.0f)) atomicOr(P.dev_status, kDevNonfinite);
    T.conf[row] = c;
    T.amax[row] = (int32_t)f.a;
  }
#endif
  if (tid == 0) TLC(18);
  __syncthreads();
  if (tid == 0) { TL(7); TLC(19); CHSET(stamp, 3); T.stamp = stamp; }
#ifdef LOPA_K2_CYC
  if (tid == 0) g_k2cur = stamp;
#endif
#ifdef LOPA_CHAIN_TL
  __syncthreads();
#endif
  if (MODE == MODE_STEP || MODE == MODE_DECIDE) cta_tail_step<kTailThreads, S>(P, T, tid, nb);
  // MODE_BP_FUSED: this rank's exchange epoch lives in its own buffer (after the flags), so the
  // step is CUDA-graph safe: e = counter + 1, records double-buffered by e's parity
  uint32_t bp_e = 0;
  uint8_t* bp_record = nullptr;
  if (MODE == MODE_BP_FUSED) {
    const uint32_t* ectr = reinterpret_cast<const uint32_t*>(P.peer_base[P.bp_rank] + P.bp_flags_off + 192);
    bp_e = *ectr + 1u;
    bp_record = P.peer_base[P.bp_rank] +
                ((size_t)(bp_e & 1u) * P.bp_world + P.bp_rank) * (size_t)P.bp_rb;
  }
  if (MODE == MODE_BP_LOCAL) cta_tail_bp_local<kTailThreads, S>(P, T, tid, nb);
  if (MODE == MODE_BP_FUSED) cta_tail_bp_local<kTailThreads, S>(P, T, tid, nb, bp_record);
  if (MODE == MODE_BP_FUSED) {
    // the exchange in the same kernel: this rank's record (its slot of this epoch's parity) is
    // stored into the same slot of every peer over NVLink, then this rank's epoch flag is raised
    // in every peer (system-scope release after a system fence; the CTA barrier orders every
    // thread's stores before it), then warp 0 waits for every rank's flag and finishes the step
    __syncthreads();
    const size_t rb = (size_t)P.bp_rb;
    const int parity = (int)(bp_e & 1u);
    const size_t slot = ((size_t)parity * P.bp_world + P.bp_rank) * rb;
    const uint4* src = reinterpret_cast<const uint4*>(bp_record);
    for (int q = 0; q < P.bp_world; ++q) {
      if (q == P.bp_rank) continue;
      uint4* dst = reinterpret_cast<uint4*>(P.peer_base[q] + slot);
      for (size_t e = tid; e < rb / 16; e += kTailThreads) dst[e] = src[e];
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      for (int q = 0; q < P.bp_world; ++q) {
        uint32_t* f = reinterpret_cast<uint32_t*>(P.peer_base[q] + P.bp_flags_off) + P.bp_rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(bp_e) : "memory");
      }
    }
    if (warp == 0) {
      uint8_t* own = P.peer_base[P.bp_rank];
      const uint32_t* flags = reinterpret_cast<const uint32_t*>(own + P.bp_flags_off);
      if (bp_wait_flags(P, flags, P.bp_world, bp_e, lane))
        bp_finish_warp<S>(P, own + (size_t)parity * P.bp_world * rb, P.bp_world, P.bp_b_loc,
                          P.table_rows, T.keys, lane);
      if (lane == 0)  // the next step's epoch (read by the next K2 of this rank only)
        *reinterpret_cast<uint32_t*>(own + P.bp_flags_off + 192) = bp_e;
    }
  }
  if (tid == 0) {
    TL(5);
    TLC(20);
  }
  if (tid == 0) CHSET(stamp, 4);
  if (MODE != MODE_DECIDE) {
    // K2 completes only after K1 (the next kernel on the stream depends on K2 alone, and K1's
    // last CTAs still reset the work counter), then advances the partial epoch
    grid_dep_wait();
    if (tid == 0) CHSET(stamp, 5);
    if (tid == 0) P.ctrs[2] = stamp;
  }
}

// MODE_CONF: one thread per candidate row, no decisions.
// One block per 256 rows.  With <= 16 groups the block's partials are pulled into shared
// memory with one bulk copy per group (a single L2 round trip), as in K2; beyond that each
// thread reads its row's partials directly.
constexpr int kFoldRows = 256;
constexpr size_t kFoldSmemBytes = 16 + (size_t)16 * kFoldRows * sizeof(float4);
__global__ void __launch_bounds__(kFoldRows) lopa_fold_kernel(const Params P) {
  extern __shared__ __align__(16) uint8_t fsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(fsm);
  float4* st = reinterpret_cast<float4*>(fsm + 16);  // [16][kFoldRows]
  grid_dep_launch();
  const int r0 = blockIdx.x * kFoldRows;
  const int nrows = min(kFoldRows, P.n_cand - r0);
  const int r = r0 + threadIdx.x;
  const bool valid = r < P.n_cand && (P.row_mask == nullptr || P.row_mask[r] != 0);
  const bool staged = P.n_grp <= 16;
  if (staged) {
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
    }
    const float4 neutral = make_float4(-INFINITY, 0.f, __uint_as_float(0xFFFFFFFFu), 0.f);
    for (int e = threadIdx.x; e < (16 - P.n_grp) * kFoldRows; e += kFoldRows)
      st[P.n_grp * kFoldRows + e] = neutral;
    __syncthreads();
  }
  grid_dep_wait();
  const uint32_t stamp = P.ctrs[2];  // K1 (complete) stamped its partials and advanced the epoch
  FoldAcc f;
  if (staged) {
    if (threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(nrows * sizeof(float4));
      mbar_arrive_expect_tx(bar, bytes * (uint32_t)P.n_grp);
      const uint64_t pol = policy_evict_first();
      for (int g = 0; g < P.n_grp; ++g)
        bulk_g2s(st + g * kFoldRows, P.gpart + (size_t)g * P.n_cand + r0, bytes, bar, pol);
    }
    mbar_wait(bar, 0);
    float4 qr[16];
    uint32_t bad = 0;
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      uint32_t sp = stamp;
      qr[p] = p < P.n_grp ? decode_slot(st[p * kFoldRows + threadIdx.x], &sp) : st[p * kFoldRows + threadIdx.x];
      bad |= sp != stamp;
    }
    if (valid) LOPA_CHK(!bad, 10);
    (void)bad;
    f = fold_tree16(16, qr);
  } else if (valid) {
    f = fold_seq(P.n_grp, [&](int p) {
      uint64_t A, B;
      load_partial_raw(P.gpart + r + (size_t)p * P.n_cand, &A, &B);
      LOPA_CHK(stamped(A, B, stamp), 10);
      return decode_partial(A, B);
    });
  }
  if (valid) {
    P.conf[r] = __fdiv_rn(1.0f, f.S);
    P.argmax[r] = (int32_t)f.a;
    if (!(f.S >= 1.0f)) atomicOr(P.dev_status, kDevNonfinite);
  }
}

static_assert(kTailThreads >= LOPA_MAX_WINDOW, "one tail thread per window position");
static_assert(LOPA_MAX_ROWS % kTailThreads == 0, "rows per tail thread");

constexpr size_t kSmemBytes = (size_t)kStages * kStageBytes + (2 * kStages + kItemSlots) * 8 +
                              kStages * 16 + kItemSlots * kPartPerItem * 16 + kItemSlots * 4 +
                              2 * kMaxGroups * 4 + kVlistBytes + 16
#ifdef LOPA_CHECKED
                              + kStages * 4
#endif
    ;

// ------------------------------------------------------------------ small decision kernels
template <int S>
__global__ void anchor_kernel(const float* conf, const int32_t* argmax, const int32_t* tokens,
                              const uint8_t* mask, int W, float tau, const float* tau_pos,
                              int32_t* tok_out, uint8_t* msk_out, int32_t* dev_status) {
  const int lane = threadIdx.x;
  WinRegs<S> r;
  load_window<S>(r, conf, argmax, tokens, mask, W, lane);
  const int st = warp_anchor<S>(r, tau, tau_pos, W, lane);
  if (st && lane == 0) atomicOr(dev_status, st);
  store_window<S>(r, tok_out, msk_out, W, lane);
}

template <int S>
__global__ void spawn_kernel(const float* conf, const int32_t* argmax, const int32_t* tok_b0,
                             const uint8_t* msk_b0, int W, int k, int32_t* br_tok,
                             uint8_t* br_msk, int32_t* look, int32_t* n_branches) {
  __shared__ uint64_t keys[32 * S];
  const int lane = threadIdx.x;
  WinRegs<S> r;
  load_window<S>(r, conf, argmax, tok_b0, msk_b0, W, lane);
  warp_spawn<S>(r, W, k, keys, br_tok, br_msk, look, n_branches, lane);
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

// Eq. 2 variants for the standalone call: one warp scores every branch in turn.
template <int S>
__global__ void verify_ex_kernel(const float* conf, const uint8_t* mask, const int32_t* n_branches,
                                 int max_br, int W, int metric, float param, float* scores,
                                 int32_t* winner) {
  __shared__ double dscr[32 * S];
  __shared__ float fscr[32 * S];
  const int lane = threadIdx.x;
  const int nb = max(0, min(*n_branches, max_br));
  float mine = -INFINITY;
  for (int j = 0; j < max_br; ++j) {
    float sc = -INFINITY;
    if (j < nb)
      sc = warp_metric_score<S>(conf + (size_t)j * W, mask + (size_t)j * W, W, metric, param, dscr,
                                fscr, lane);
    if (lane == 0) scores[j] = sc;
    if (lane == j) mine = sc;
  }
  const int w = warp_select(mine, lane, nb);
  if (lane == 0) *winner = w;
}

// Peer-memory exchange: wait (one warp; lane r polls rank r's flag, acquire at system scope,
// bounded) until every rank's record of this epoch has landed.  A rank that never arrives is
// reported as LOPA_DEV_PEER_TIMEOUT and the step decides nothing (n_next = 0, tables untouched:
// the caller must check dev_status after every peer-memory step).  Returns false then.
__device__ bool bp_wait_flags(const Params& P, const uint32_t* flags, int world, uint32_t epoch,
                              int lane) {
  if (lane < world) {
    uint32_t v = 0;
    // bounded (>= 1 s: 2^24 polls 64 ns apart): a healthy exchange lands within microseconds;
    // the slack absorbs ranks that reach their first step at different times (module loading)
    for (uint32_t spin = 0; spin < (1u << 24); ++spin) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + lane) : "memory");
      if (v >= epoch) break;
      __nanosleep(64);
    }
    if (v < epoch) atomicOr(P.dev_status, kDevPeerTimeout);
  }
  bool late = false;
  if (lane < world) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + lane) : "memory");
    late = v < epoch;
  }
  if (__any_sync(0xffffffffu, late)) {
    if (lane == 0) *P.n_next = 0;
    return false;
  }
  __syncwarp();
  return true;
}

// Global half of a BP step on one warp over the `world` records (lane r reads record r's
// header): the global select, the scores of every branch, the anchor on the owner's row and the
// spawn.  keys: 32 S entries of shared scratch.
template <int S>
__device__ void bp_finish_warp(const Params& P, const uint8_t* records, int world, int b_loc,
                               int n_scores, uint64_t* keys, int lane) {
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
      LOPA_CHK(*rv.n_present <= b_loc && *rv.b_loc == b_loc, 9);
      if (jl < *rv.n_present) v = rv.scores[jl];
    }
    LOPA_CHK(j < P.table_rows, 9);
    P.scores[j] = v;
  }
  const int W = P.window;
  const bool none = (wid == 0xFFFFFFFFu) || (wid == 0x7FFFFFFFu);
  if (lane == 0) *P.winner = none ? 0 : (int)wid;
  WinRegs<S> r;
  if (none) {  // no branch present anywhere: pass branch 0 through as complete
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane + 32 * s;
      r.msk[s] = 0;
      r.tok[s] = i < W ? P.branch_tokens[i] : 0;
      r.conf[s] = 0.f;
      r.amax[s] = -1;
    }
  } else {
    RecordView rv = record_view(const_cast<uint8_t*>(records) + rb * owner, b_loc);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int i = lane + 32 * s;
      const bool in = i < W;
      r.msk[s] = in ? (uint32_t)(rv.mask[i] != 0) : 0u;
      r.tok[s] = in ? rv.tokens[i] : 0;
      r.conf[s] = (in && r.msk[s]) ? rv.conf[i] : 0.f;
      r.amax[s] = (in && r.msk[s]) ? rv.argmax[i] : -1;
    }
  }
  bool anym = false;
#pragma unroll
  for (int s = 0; s < S; ++s) anym |= r.msk[s] != 0;
  const bool any = __any_sync(0xffffffffu, anym);
  if (!any) {
    store_window<S>(r, P.next_tokens, P.next_mask, W, lane);
    if (P.lookahead)
      for (int q = lane; q < P.k; q += 32) P.lookahead[q] = -1;
    if (lane == 0) *P.n_next = 0;
    return;
  }
  warp_anchor<S>(r, P.tau, P.tau_pos, W, lane);
  warp_spawn<S>(r, W, P.k, keys, P.next_tokens, P.next_mask, P.lookahead, P.n_next, lane);
}

// Global half of a BP step as its own kernel (NCCL all-gather path; flags: the round-1
// three-kernel peer-memory path, LOPA_BP_P2P_3K).
template <int S>
__global__ void bp_finish_kernel(const Params P, const uint8_t* records, int world, int b_loc,
                                 int n_scores, const uint32_t* flags, uint32_t epoch) {
  __shared__ uint64_t keys[32 * S];
  const int lane = threadIdx.x;
  grid_dep_wait();  // PDL (peer-memory path): the publisher before us has been issued
  if (flags != nullptr && !bp_wait_flags(P, flags, world, epoch, lane)) return;
  bp_finish_warp<S>(P, records, world, b_loc, n_scores, keys, lane);
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

// The K2 instantiation for a mode and window: S = window slots per lane (1, 2 or 8).
using TailKernel = void (*)(const Params);
static TailKernel tail_kernel_for(int mode, int window) {
  const int S = window <= 32 ? 1 : (window <= 64 ? 2 : 8);
  if (mode == MODE_STEP)
    return S == 1 ? lopa_tail_kernel<MODE_STEP, 1> : S == 2 ? lopa_tail_kernel<MODE_STEP, 2> : lopa_tail_kernel<MODE_STEP, 8>;
  if (mode == MODE_DECIDE)
    return S == 1 ? lopa_tail_kernel<MODE_DECIDE, 1> : S == 2 ? lopa_tail_kernel<MODE_DECIDE, 2> : lopa_tail_kernel<MODE_DECIDE, 8>;
  if (mode == MODE_BP_FUSED)
    return S == 1 ? lopa_tail_kernel<MODE_BP_FUSED, 1> : S == 2 ? lopa_tail_kernel<MODE_BP_FUSED, 2> : lopa_tail_kernel<MODE_BP_FUSED, 8>;
  return S == 1 ? lopa_tail_kernel<MODE_BP_LOCAL, 1> : S == 2 ? lopa_tail_kernel<MODE_BP_LOCAL, 2> : lopa_tail_kernel<MODE_BP_LOCAL, 8>;
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
  cudaError_t e = cudaFuncSetAttribute(lopa_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kSmemBytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lopa_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kFoldSmemBytes);
#ifdef LOPA_K1_LDG
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lopa_reduce_ldg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kLSmemBytes);
#endif
  for (int mode : {(int)MODE_STEP, (int)MODE_BP_LOCAL, (int)MODE_DECIDE, (int)MODE_BP_FUSED})
    for (int w : {32, 64, 256})
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tail_kernel_for(mode, w), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTailSmemBytes);
  if (e != cudaSuccess) return cuda_status(e);
  std::lock_guard<std::mutex> lk(g_mu);
  if (device >= 0 && device < 64) g_attr[device] = true;
  return LOPA_OK;
}

bool bind_device(void* stream, const void* ptr, int* device) {
  int dev = -1;
  if (stream != nullptr) {
    // During CUDA-graph capture, device queries on the stream invalidate the capture: the
    // capturing thread's current device is the stream's device.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &cs) == cudaSuccess &&
        cs != cudaStreamCaptureStatusNone)
      return cudaGetDevice(device) == cudaSuccess;
  }
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
  return 256 + (size_t)max_rows * num_groups(ns) * sizeof(float4);
}

bool carve_workspace(void* ws, size_t bytes, int32_t max_rows, int32_t vocab, Workspace* out) {
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 255) != 0) return false;
  if (bytes < workspace_bytes(max_rows, vocab)) return false;
  uint8_t* p = static_cast<uint8_t*>(ws);
  out->ctrs = reinterpret_cast<uint32_t*>(p);
  out->gpart = reinterpret_cast<float4*>(p + 256);
  return true;
}

template <typename Kern>
static cudaError_t launch_pdl(Kern kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              const Params& P) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
#ifdef LOPA_NO_PDL
  attr[0].val.programmaticStreamSerializationAllowed = 0;
#else
  attr[0].val.programmaticStreamSerializationAllowed = 1;
#endif
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, P);
}

// Optional K1 timing (lopa_profile_enable / lopa_profile_read).
struct Profiler {
  std::mutex mu;
  int cap = 0, n = 0;
  cudaEvent_t* ev = nullptr;  // [cap][2]
};
static Profiler g_prof;

static void prof_record(int which, cudaStream_t s, int* slot) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  if (!g_prof.ev) return;
  if (which == 0) {
    if (g_prof.n >= g_prof.cap) { *slot = -1; return; }
    *slot = g_prof.n++;
  }
  if (*slot >= 0) cudaEventRecord(g_prof.ev[2 * *slot + which], s);
}

// K1 (streaming reduction) then K2 (fold + decisions, or the fold only for MODE_CONF), both
// with programmatic dependent launch so launch latency overlaps the previous kernel.
// K1's form: register-fed (lopa_reduce_ldg_kernel) or TMA-ring (lopa_reduce_kernel).
#ifdef LOPA_K1_LDG
#define LOPA_K1_KERNEL lopa_reduce_ldg_kernel
constexpr int kK1Threads = kLThreads;
constexpr size_t kK1Smem = kLSmemBytes;
constexpr int kK1CtasPerSm = 1;
#else
#define LOPA_K1_KERNEL lopa_reduce_kernel
constexpr int kK1Threads = kThreads;
constexpr size_t kK1Smem = kSmemBytes;
constexpr int kK1CtasPerSm = LOPA_CTAS_PER_SM;
#endif

// lopa_set_logits_prefetch: process-wide, read at every launch of K1
static std::atomic<int> g_logits_prefetch{1};

static int launch_reduce(const Params& P0, int device, cudaStream_t s, bool k1_only = false) {
  int st = ensure_kernel_attrs(device);
  if (st != LOPA_OK) return st;
  Params P = P0;
  P.prefetch = g_logits_prefetch.load(std::memory_order_relaxed);
  if (P.conf_ready) {  // no K1: the fold/decision kernel on the previous kernel's conf / argmax
    auto kern = tail_kernel_for(P.mode, P.window);
    return cuda_status(launch_pdl(kern, dim3(1), dim3(kTailThreads), kTailSmemBytes, s, P));
  }
  P.k1_alone = k1_only ? 1 : 0;
  if (k1_only) {  // measurement: K1 alone, in the step's launch configuration
    const int g = kK1CtasPerSm * (num_sms(device) - 1);
    return cuda_status(launch_pdl(LOPA_K1_KERNEL, dim3(g), dim3(kK1Threads), kK1Smem, s, P));
  }
  // One SM is left to the fold/tail kernel: it becomes resident there while K1 streams (PDL)
  // and, landing on the same SM step after step, runs with a warm instruction cache.
  const int grid = kK1CtasPerSm * (num_sms(device) - (P.mode == MODE_CONF ? 0 : 1));
  if (grid <= 0) return LOPA_ERR_CUDA;
  int pslot = -1;
  prof_record(0, s, &pslot);
  cudaError_t e = launch_pdl(LOPA_K1_KERNEL, dim3(grid), dim3(kK1Threads), kK1Smem, s, P);
  if (e != cudaSuccess) return cuda_status(e);
  prof_record(1, s, &pslot);
  if (P.mode == MODE_CONF) {
    const int nb = (P.n_cand + 255) / 256;
    e = launch_pdl(lopa_fold_kernel, dim3(nb), dim3(kFoldRows), kFoldSmemBytes, s, P);
  } else {
    // window slots per lane: 2 (W <= 64) or 8 (the D2F multi-block window, W <= 256)
    // window slots per lane: 1 (W <= 32), 2 (W <= 64), 8 (the D2F multi-block window)
    auto kern = tail_kernel_for(P.mode, P.window);
    e = launch_pdl(kern, dim3(1), dim3(kTailThreads), kTailSmemBytes, s, P);
  }
  return cuda_status(e);
}

static bool metric_ok(int32_t metric, float param) {
  if (metric == LOPA_METRIC_MEAN) return true;
  if (metric == LOPA_METRIC_SLIDING_MIN) return param >= 1.f && param <= 1e6f && param == (float)(int)param;
  if (metric == LOPA_METRIC_BOTTOM_FRACTION) return param > 0.f && param <= 1.f;
  return false;
}

static bool logits_ok(const void* logits, int64_t ld, int32_t vocab) {
  return logits && vocab >= 1 && ld >= vocab && (ld % 8) == 0 &&
         (reinterpret_cast<uintptr_t>(logits) & 15) == 0;
}

int validate_step_args(const lopa_step_args_t* a, bool need_next, bool need_logits) {
  if (!a) return LOPA_ERR_INVALID_ARG;
  if (need_logits && !logits_ok(a->logits, a->ld, a->vocab)) return LOPA_ERR_INVALID_ARG;
  if (!need_logits && (a->vocab < 1)) return LOPA_ERR_INVALID_ARG;
  if (a->window < 1 || a->max_branches < 1 || a->k < 0) return LOPA_ERR_INVALID_ARG;
  if (!(a->tau > 0.f && a->tau <= 1.f)) return LOPA_ERR_INVALID_ARG;
  if (!metric_ok(a->metric, a->metric_param)) return LOPA_ERR_INVALID_ARG;
  if (!a->n_branches || !a->branch_tokens || !a->branch_mask || !a->conf || !a->argmax ||
      !a->dev_status || !a->workspace)
    return LOPA_ERR_INVALID_ARG;
  if (need_next && (!a->scores || !a->winner || !a->next_tokens || !a->next_mask ||
                    !a->n_branches_next || (a->k > 0 && !a->lookahead_pos)))
    return LOPA_ERR_INVALID_ARG;
  if (a->window > LOPA_MAX_WINDOW || a->vocab > LOPA_MAX_VOCAB) return LOPA_ERR_UNSUPPORTED;
  if (a->window > 64 && a->vocab > (1 << 22)) return LOPA_ERR_UNSUPPORTED;  // R24 exact sums
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
  P.n_grp = num_groups(P.n_seg);
  P.window = a->window;
  P.table_rows = a->max_branches;
  P.n_branches = a->n_branches;
  P.conf = a->conf;
  P.argmax = a->argmax;
  P.dev_status = a->dev_status;
  P.ctrs = ws.ctrs;
  P.gpart = ws.gpart;
  P.branch_tokens = a->branch_tokens;
  P.branch_mask = a->branch_mask;
  P.k = a->k;
  P.tau = a->tau;
  P.tau_pos = a->tau_pos;
  P.metric = a->metric;
  P.metric_param = a->metric_param;
  P.scores = a->scores;
  P.winner = a->winner;
  P.next_tokens = a->next_tokens;
  P.next_mask = a->next_mask;
  P.lookahead = a->lookahead_pos;
  P.n_next = a->n_branches_next;
  return P;
}

int launch_bp_local(const lopa_step_args_t* a, int32_t branch_base, int32_t b_loc, void* record,
                    cudaStream_t s, bool conf_ready) {
  int st = validate_step_args(a, false, !conf_ready);
  if (st != LOPA_OK) return st;
  if (!record || b_loc < 1 || branch_base < 0) return LOPA_ERR_INVALID_ARG;
  if (b_loc > LOPA_MAX_BRANCHES || (int64_t)b_loc * a->window > LOPA_MAX_ROWS)
    return LOPA_ERR_UNSUPPORTED;
  Workspace ws;
  if (!carve_workspace(a->workspace, a->workspace_bytes, b_loc * a->window, a->vocab, &ws))
    return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!bind_device(s, conf_ready ? static_cast<const void*>(a->conf) : a->logits, &dev)) return LOPA_ERR_CUDA;
  Params P = base_params(a, ws);
  P.mode = MODE_BP_LOCAL;
  P.conf_ready = conf_ready ? 1 : 0;
  P.branch_base = branch_base;
  P.cap = b_loc;
  P.n_cand = b_loc * a->window;
  P.row_mask = a->branch_mask + (size_t)branch_base * a->window;
  P.record = static_cast<uint8_t*>(record);
  return launch_reduce(P, dev, s);
}

// lopa_bp_step_p2p in two kernels: K1 + K2 in MODE_BP_FUSED (local half, the peer-memory
// exchange and the global half).  record = this rank's slot of this epoch's parity.
int launch_bp_fused(const lopa_step_args_t* a, int32_t b_loc, void* record, uint8_t* const* peer_base,
                    int32_t world, int32_t rank, size_t rb, size_t flags_off, int32_t parity,
                    uint32_t epoch, cudaStream_t s, bool conf_ready) {
  int st = validate_step_args(a, true, !conf_ready);
  if (st != LOPA_OK) return st;
  if (!record || !peer_base || b_loc < 1 || world < 1 || world > 32 || rank < 0 || rank >= world)
    return LOPA_ERR_INVALID_ARG;
  if (b_loc > LOPA_MAX_BRANCHES || (int64_t)b_loc * a->window > LOPA_MAX_ROWS)
    return LOPA_ERR_UNSUPPORTED;
  Workspace ws;
  if (!carve_workspace(a->workspace, a->workspace_bytes, b_loc * a->window, a->vocab, &ws))
    return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!bind_device(s, conf_ready ? static_cast<const void*>(a->conf) : a->logits, &dev)) return LOPA_ERR_CUDA;
  Params P = base_params(a, ws);
  P.mode = MODE_BP_FUSED;
  P.conf_ready = conf_ready ? 1 : 0;
  P.branch_base = rank * b_loc;
  P.cap = b_loc;
  P.n_cand = b_loc * a->window;
  P.row_mask = a->branch_mask + (size_t)P.branch_base * a->window;
  P.record = static_cast<uint8_t*>(record);
  P.peer_base = peer_base;
  P.bp_world = world;
  P.bp_rank = rank;
  P.bp_b_loc = b_loc;
  P.bp_parity = parity;
  P.bp_epoch = epoch;
  P.bp_rb = (int64_t)rb;
  P.bp_flags_off = (int64_t)flags_off;
  return launch_reduce(P, dev, s);
}

// a2 -> a3 -> a4 on conf / argmax already in a->conf / a->argmax (written by the previous kernel
// on the stream: K2 is launched programmatically dependent on it).
int launch_step_decide(const lopa_step_args_t* a, cudaStream_t s) {
  int st = validate_step_args(a, true, false);
  if (st != LOPA_OK) return st;
  const int32_t rows = a->max_branches * a->window;
  if (rows > LOPA_MAX_ROWS) return LOPA_ERR_UNSUPPORTED;
  Workspace ws;
  if (!carve_workspace(a->workspace, a->workspace_bytes, rows, a->vocab, &ws))
    return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!bind_device(s, a->conf, &dev)) return LOPA_ERR_CUDA;
  st = ensure_kernel_attrs(dev);
  if (st != LOPA_OK) return st;
  Params P = base_params(a, ws);
  P.mode = MODE_DECIDE;
  P.cap = a->max_branches;
  P.n_cand = rows;
  P.row_mask = a->branch_mask;
  auto kern = tail_kernel_for(MODE_DECIDE, P.window);
  return cuda_status(launch_pdl(kern, dim3(1), dim3(kTailThreads), kTailSmemBytes, s, P));
}

int launch_bp_finish(const lopa_step_args_t* a, int32_t b_loc, int32_t world, const void* records,
                     cudaStream_t s, const uint32_t* flags, uint32_t epoch) {
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
  auto kern = a->window > 64 ? bp_finish_kernel<8> : bp_finish_kernel<2>;
  const uint8_t* rec = static_cast<const uint8_t*>(records);
  if (flags == nullptr) {
    kern<<<1, 32, 0, s>>>(P, rec, world, b_loc, n_scores, flags, epoch);
    return cuda_status(cudaGetLastError());
  }
  // peer-memory path: launched programmatically dependent on the publisher (it waits for the
  // flags anyway), so its launch overlaps the publish
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_status(cudaLaunchKernelEx(&cfg, kern, P, rec, world, b_loc, n_scores, flags, epoch));
}

}  // namespace lopa

// =================================================================== C ABI
using namespace lopa;

extern "C" int lopa_version(void) { return LOPA_VERSION; }

static thread_local char g_last_cuda_error[256];
void lopa::note_cuda_error(cudaError_t e) {
  snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s: %s", cudaGetErrorName(e),
           cudaGetErrorString(e));
}
extern "C" const char* lopa_last_cuda_error(void) { return g_last_cuda_error; }

extern "C" int lopa_set_logits_prefetch(int32_t enabled) {
  return lopa::g_logits_prefetch.exchange(enabled ? 1 : 0);
}

extern "C" int lopa_profile_enable(int32_t max_records) {
  if (max_records < 1) return LOPA_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(lopa::g_prof.mu);
  if (lopa::g_prof.ev) {
    for (int i = 0; i < 2 * lopa::g_prof.cap; ++i) cudaEventDestroy(lopa::g_prof.ev[i]);
    delete[] lopa::g_prof.ev;
    lopa::g_prof.ev = nullptr;
  }
  lopa::g_prof.ev = new cudaEvent_t[2 * max_records];
  for (int i = 0; i < 2 * max_records; ++i)
    if (cudaEventCreate(&lopa::g_prof.ev[i]) != cudaSuccess) return LOPA_ERR_CUDA;
  lopa::g_prof.cap = max_records;
  lopa::g_prof.n = 0;
  return LOPA_OK;
}

extern "C" int lopa_profile_read(float* k1_ms, int32_t max, int32_t* n_out) {
  if (!k1_ms || !n_out || max < 0) return LOPA_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lk(lopa::g_prof.mu);
  *n_out = 0;
  if (!lopa::g_prof.ev) return LOPA_OK;
  int st = LOPA_OK;
  const int n = std::min(max, lopa::g_prof.n);
  for (int i = 0; i < n; ++i) {
    if (cudaEventSynchronize(lopa::g_prof.ev[2 * i + 1]) != cudaSuccess ||
        cudaEventElapsedTime(&k1_ms[i], lopa::g_prof.ev[2 * i], lopa::g_prof.ev[2 * i + 1]) != cudaSuccess) {
      st = LOPA_ERR_CUDA;
      break;
    }
    *n_out = i + 1;
  }
  for (int i = 0; i < 2 * lopa::g_prof.cap; ++i) cudaEventDestroy(lopa::g_prof.ev[i]);
  delete[] lopa::g_prof.ev;
  lopa::g_prof.ev = nullptr;
  lopa::g_prof.cap = lopa::g_prof.n = 0;
  return st;
}

// Debug: copy the per-CTA phase timeline of the last launch (timeline builds only; returns the
// number of slots per CTA, 0 if the build has no timeline).
extern "C" int lopa_debug_timeline(unsigned long long* out, int n_ctas) {
#ifdef LOPA_TIMELINE
  if (!out || n_ctas < 1 || n_ctas > 256) return 0;
  cudaDeviceSynchronize();

  if (cudaMemcpyFromSymbol(out, lopa::g_timeline, sizeof(unsigned long long) * n_ctas * lopa::kTlSlots) != cudaSuccess) return 0;
  return lopa::kTlSlots;
#else
  (void)out; (void)n_ctas;
  return 0;
#endif
}

// Debug (LOPA_CHAIN_TL builds): per-step marks of chained steps ([64][8] ns), then cleared.
extern "C" int lopa_debug_chain_timeline(unsigned long long* out, int n_words) {
#if defined(LOPA_CHAIN_TL) || defined(LOPA_K2_CYC)
  constexpr int kW = (int)(sizeof(lopa::g_chain[0]) / sizeof(unsigned long long));
  const int need = 64 * kW;
  if (!out || n_words < need) return -need;
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, lopa::g_chain, sizeof(lopa::g_chain)) != cudaSuccess) return 0;
  unsigned long long init[64][kW];
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < kW; ++j) init[i][j] = (j == 0 || j == 6) ? ~0ull : 0ull;
  cudaMemcpyToSymbol(lopa::g_chain, init, sizeof(init));
  return need;
#else
  (void)out; (void)n_words;
  return 0;
#endif
}

// Debug (LOPA_K1_TL builds): per-item timeline of K1's TMA form, last launch.
extern "C" int lopa_debug_k1_timeline(unsigned long long* out, int n_words) {
#ifdef LOPA_K1_TL
  const int need = (int)(sizeof(lopa::g_k1tl) / 8);
  if (!out || n_words < need) return -need;
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, lopa::g_k1tl, sizeof(lopa::g_k1tl)) != cudaSuccess) return 0;
  return need;
#else
  (void)out; (void)n_words;
  return 0;
#endif
}

// Debug (LOPA_LDG_TL builds): per-warp timeline of the warp-staged K1's last launch.
extern "C" int lopa_debug_ldg_timeline(unsigned long long* out, int n_words) {
#ifdef LOPA_LDG_TL
  const int need = (int)(sizeof(lopa::g_ldg_tl) / 8);
  if (!out || n_words < need) return -need;
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, lopa::g_ldg_tl, sizeof(lopa::g_ldg_tl)) != cudaSuccess) return 0;
  return need;
#else
  (void)out; (void)n_words;
  return 0;
#endif
}

// Checked builds: {violations, first violating site, bitmask of sites} since the last read, then
// reset.  LOPA_ERR_UNSUPPORTED in product builds.
extern "C" int lopa_debug_check_read(uint32_t* out3) {
  if (!out3) return LOPA_ERR_INVALID_ARG;
#ifdef LOPA_CHECKED
  cudaDeviceSynchronize();
  unsigned v[3] = {0, 0, 0};
  if (cudaMemcpyFromSymbol(&v[0], lopa::g_chk_count, 4) != cudaSuccess ||
      cudaMemcpyFromSymbol(&v[1], lopa::g_chk_first, 4) != cudaSuccess ||
      cudaMemcpyFromSymbol(&v[2], lopa::g_chk_sites, 4) != cudaSuccess)
    return LOPA_ERR_CUDA;
  const unsigned z = 0;
  cudaMemcpyToSymbol(lopa::g_chk_count, &z, 4);
  cudaMemcpyToSymbol(lopa::g_chk_first, &z, 4);
  cudaMemcpyToSymbol(lopa::g_chk_sites, &z, 4);
  out3[0] = v[0];
  out3[1] = v[1];
  out3[2] = v[2];
  return LOPA_OK;
#else
  out3[0] = out3[1] = out3[2] = 0;
  return LOPA_ERR_UNSUPPORTED;
#endif
}

// Debug: resource attributes of the K1 kernel this build launches: {registers per thread,
// max threads per block, static shared bytes, local bytes per thread, launch block size}.
extern "C" int lopa_debug_k1_attrs(int32_t* out5) {
  if (!out5) return LOPA_ERR_INVALID_ARG;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, LOPA_K1_KERNEL);
  if (e != cudaSuccess) return cuda_status(e);
  out5[0] = fa.numRegs;
  out5[1] = fa.maxThreadsPerBlock;
  out5[2] = (int32_t)fa.sharedSizeBytes;
  out5[3] = (int32_t)fa.localSizeBytes;
  out5[4] = kK1Threads;
  return LOPA_OK;
}

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

static int confidence_impl(const void* logits, int64_t ld, int32_t n_rows, int32_t vocab,
                           const uint8_t* row_mask, float* conf, int32_t* argmax,
                           int32_t* dev_status, void* workspace, size_t workspace_bytes,
                           void* stream, bool k1_only);

extern "C" int lopa_confidence(const void* logits, int64_t ld, int32_t n_rows, int32_t vocab,
                               const uint8_t* row_mask, float* conf, int32_t* argmax,
                               int32_t* dev_status, void* workspace, size_t workspace_bytes,
                               void* stream) {
  return confidence_impl(logits, ld, n_rows, vocab, row_mask, conf, argmax, dev_status, workspace,
                         workspace_bytes, stream, false);
}

extern "C" int lopa_debug_reduce_only(const void* logits, int64_t ld, int32_t n_rows,
                                      int32_t vocab, const uint8_t* row_mask, int32_t* dev_status,
                                      void* workspace, size_t workspace_bytes, void* stream) {
  static float dummy_conf;
  static int32_t dummy_argmax;
  return confidence_impl(logits, ld, n_rows, vocab, row_mask, &dummy_conf, &dummy_argmax,
                         dev_status, workspace, workspace_bytes, stream, true);
}

static int confidence_impl(const void* logits, int64_t ld, int32_t n_rows, int32_t vocab,
                           const uint8_t* row_mask, float* conf, int32_t* argmax,
                           int32_t* dev_status, void* workspace, size_t workspace_bytes,
                           void* stream, bool k1_only) {
  if (n_rows < 0) return LOPA_ERR_INVALID_ARG;
  if (!logits_ok(logits, ld, vocab) || !conf || !argmax || !dev_status || !workspace)
    return LOPA_ERR_INVALID_ARG;
  if (n_rows > LOPA_MAX_ROWS || vocab > LOPA_MAX_VOCAB) return LOPA_ERR_UNSUPPORTED;
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
  P.n_grp = num_groups(P.n_seg);
  P.n_cand = n_rows;
  P.row_mask = row_mask;
  P.window = 1;
  P.table_rows = n_rows;
  P.conf = conf;
  P.argmax = argmax;
  P.dev_status = dev_status;
  P.ctrs = ws.ctrs;
  P.gpart = ws.gpart;
  P.mode = MODE_CONF;
  return launch_reduce(P, dev, s, k1_only);
}

extern "C" int lopa_anchor_fill_ex(const float* conf, const int32_t* argmax, const int32_t* tokens,
                                   const uint8_t* mask, int32_t window, float tau,
                                   const float* tau_pos, int32_t* tokens_out, uint8_t* mask_out,
                                   int32_t* dev_status, void* stream) {
  if (!conf || !argmax || !tokens || !mask || !tokens_out || !mask_out || !dev_status)
    return LOPA_ERR_INVALID_ARG;
  if (window < 1 || !(tau > 0.f && tau <= 1.f)) return LOPA_ERR_INVALID_ARG;
  if (window > LOPA_MAX_WINDOW) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!bind_device(stream, conf, &dev)) return LOPA_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (window > 64)
    anchor_kernel<8><<<1, 32, 0, s>>>(conf, argmax, tokens, mask, window, tau, tau_pos, tokens_out,
                                      mask_out, dev_status);
  else
    anchor_kernel<2><<<1, 32, 0, s>>>(conf, argmax, tokens, mask, window, tau, tau_pos, tokens_out,
                                      mask_out, dev_status);
  return cuda_status(cudaGetLastError());
}

extern "C" int lopa_anchor_fill(const float* conf, const int32_t* argmax, const int32_t* tokens,
                                const uint8_t* mask, int32_t window, float tau,
                                int32_t* tokens_out, uint8_t* mask_out, int32_t* dev_status,
                                void* stream) {
  return lopa_anchor_fill_ex(conf, argmax, tokens, mask, window, tau, nullptr, tokens_out,
                             mask_out, dev_status, stream);
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
  if (window > 64)
    spawn_kernel<8><<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        conf, argmax, tokens_b0, mask_b0, window, k, branch_tokens, branch_mask, lookahead_pos,
        n_branches);
  else
    spawn_kernel<2><<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
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

extern "C" int lopa_verify_select_ex(const float* conf, const uint8_t* branch_mask,
                                     const int32_t* n_branches, int32_t max_branches,
                                     int32_t window, int32_t metric, float metric_param,
                                     float* scores, int32_t* winner, void* stream) {
  if (!conf || !branch_mask || !n_branches || !scores || !winner) return LOPA_ERR_INVALID_ARG;
  if (window < 1 || max_branches < 1 || !metric_ok(metric, metric_param))
    return LOPA_ERR_INVALID_ARG;
  if (window > LOPA_MAX_WINDOW || max_branches > LOPA_MAX_BRANCHES) return LOPA_ERR_UNSUPPORTED;
  int dev;
  if (!bind_device(stream, conf, &dev)) return LOPA_ERR_CUDA;
  if (window > 64)
    verify_ex_kernel<8><<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        conf, branch_mask, n_branches, max_branches, window, metric, metric_param, scores, winner);
  else
    verify_ex_kernel<2><<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
        conf, branch_mask, n_branches, max_branches, window, metric, metric_param, scores, winner);
  return cuda_status(cudaGetLastError());
}

extern "C" int lopa_step(const lopa_step_args_t* a, void* stream) {
  int st = validate_step_args(a, true, true);
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
  P.window_dev = a->window_dev;  // device-resident window (lopa_d2f_*): read by K1 / K2
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
