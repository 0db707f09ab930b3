// EXPERIMENT, included by lopa_core.cu only with -DLOPA_K1_LDG (never in the product library):
// the warp-staged K1 of profiles/r02_k1_ab.md (bit-identical to the TMA form, 1.9x slower).
// It uses lopa_core.cu's Params, Partial, FoldAcc, reduce helpers and store_partial.
#pragma once
// ------------------------------------------------------------------ K1, warp-staged form
// EXPERIMENT (built only with -DLOPA_K1_LDG; not in the product library).  Bit-identical to the
// TMA form and parity-green on the B200, but 1.9x slower on the Dream step (DESIGN.md §5,
// profiles/r02_k1_ab.md): the per-warp cp.async streams reach ~25 GB/s per SM where the TMA
// ring reaches ~45.
// The same work items, canonical slices and folds as lopa_reduce_kernel (so the group partials
// are bit-identical), but with no shared TMA stage: every consumer warp streams its own slice
// of an item through a private ring of shared-memory buffers with 16-byte cp.async copies, and
// waits for them with cp.async.wait_group (per-thread commit groups complete in order, so a
// warp keeps kLDepth slices in flight while it reduces the oldest one):
//   * kTeams teams of 8 warps and no producer warp.  Warp (jseg, wq) of a team reduces chunks
//     c = 128 i + 32 wq + lane (i < 8) of segment jseg of each of the team's items -- exactly
//     reduce_slice's quarter; each lane copies and later reads only its own chunks.
//   * Lane 0 of the team's first warp (the team leader) publishes the team's item descriptors
//     into the team's ring of kLSlots slots (mbarrier `ready` per slot; a slot is reused once its
//     item is folded, mbarrier `sfree`), kLDepth + 1 items ahead of its own reduction.  It keeps
//     two claims on the global work counter in flight: a claim's value is consumed one publish
//     after it is issued, so the atomic's round trip hides behind the team's work.
//   * The first item of the first kLSpec teams of CTA b is the raw item t G + b, published and
//     copied before the row masks arrive (a copy of a row that turns out invalid is discarded).
//     Further items follow K1's numbering: raw items n_spec + claim over mostly-valid row sets
//     (a claim on an invalid row is skipped), otherwise items numbered over the valid rows only
//     (vlist), group-major.
//   * All 8 warps of an item count into icnt; the last one folds the item's warp partials
//     (fold_seq, fixed order) into the group partial, as K1's TMA form does.
// (A first form that loaded the slices straight into two register buffers per warp lost all
// overlap: ptxas gives every LDG the same scoreboard, so reducing one buffer waited for the
// other buffer's loads too.  Commit groups make the wait explicit.)
#ifndef LOPA_LDG_TEAMS
#define LOPA_LDG_TEAMS 2
#endif
#ifndef LOPA_LDG_DEPTH
#define LOPA_LDG_DEPTH 2
#endif
#ifndef LOPA_LDG_SLOTS
#define LOPA_LDG_SLOTS (LOPA_LDG_DEPTH + 2)
#endif
#ifndef LOPA_LDG_SPEC
#define LOPA_LDG_SPEC 1
#endif
constexpr int kTeams = LOPA_LDG_TEAMS;
constexpr int kTeamWarps = kSegPerItem * kWarpsPerSeg;  // one warp per (segment, quarter)
constexpr int kLThreads = 32 * kTeamWarps * kTeams;
constexpr int kLDepth = LOPA_LDG_DEPTH;  // slices in flight per warp beyond the one reduced
constexpr int kLBufs = kLDepth + 1;
constexpr int kLSlots = LOPA_LDG_SLOTS;  // item slots per team
constexpr int kLSpec = LOPA_LDG_SPEC;    // teams whose first item is speculative
constexpr int kSliceChunks = kChunksPerLane * 32;  // 16-byte chunks of one warp slice (4 KB)
constexpr size_t kLSmemBytes = (size_t)kTeams * kTeamWarps * kLBufs * kSliceChunks * 16;
// The leader publishes item k + kLDepth + 1 before reducing item k: that item's slot must have
// been freed by item k - 1, which every warp of the team has reduced before reaching item k.
static_assert(kLSlots >= kLDepth + 2, "item ring too short for the staging depth");
static_assert(kLSpec >= 0 && kLSpec <= kTeams, "speculative teams");
static_assert(kLDepth >= 1, "at least one slice in flight");
static_assert(kTeamWarps * 32 == 256, "team = 8 warps");

// reduce_slice's arithmetic on a slice already in registers (identical operations and order,
// so identical bits); the first-argmax chunk is selected from the registers.
__device__ __forceinline__ Partial reduce_regs(uint4 (&v)[kChunksPerLane], int nchunks, int e0,
                                               int vocab, int wq, int lane) {
  const bool ragged = (vocab & 7) != 0;
  if (ragged) {
#pragma unroll
    for (int t = 0; t < kChunksPerLane; ++t) {
      const int c = 128 * t + 32 * wq + lane;
      const int nvalid = vocab - (e0 + 8 * c);
      if (c < nchunks && nvalid < 8) mask_tail(v[t], nvalid);
    }
  }
  uint32_t cm[kChunksPerLane];
#pragma unroll
  for (int t = 0; t < kChunksPerLane; ++t) cm[t] = bmax2(bmax2(v[t].x, v[t].y), bmax2(v[t].z, v[t].w));
  uint32_t mm = cm[0];
#pragma unroll
  for (int t = 1; t < kChunksPerLane; ++t) mm = bmax2(mm, cm[t]);
  const float ml = fmax_nan(bf16lo(mm), bf16hi(mm));
  const float m = unordered(__reduce_max_sync(0xffffffffu, ordered_bits(ml)));
  Partial p;
  p.m = m;
  if (m == -INFINITY) {  // warp-uniform: every element is -inf (or NaN)
    bool bad = false;
#pragma unroll
    for (int t = 0; t < kChunksPerLane; ++t) bad |= chunk_has_nan(v[t]);
    p.s = __any_sync(0xffffffffu, bad) ? __int_as_float(0x7FC00000) : 0.f;
    p.a = 0xFFFFFFFFu;
    return p;
  }
  uint32_t cand = 0xFFFFFFFFu;
  if (ml == m) {
    const __nv_bfloat162 m2 = __floats2bfloat162_rn(m, m);
    int tf = kChunksPerLane - 1;
#pragma unroll
    for (int t = kChunksPerLane - 1; t >= 0; --t)
      if (!__hbne2(*reinterpret_cast<const __nv_bfloat162*>(&cm[t]), m2)) tf = t;
    uint4 w = v[0];
#pragma unroll
    for (int t = 1; t < kChunksPerLane; ++t)
      if (tf == t) w = v[t];
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    int ef = 7;
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      const unsigned eq = __heq2_mask(*reinterpret_cast<const __nv_bfloat162*>(&ws[j]), m2);
      if (eq) ef = 2 * j + ((eq & 0xFFFFu) ? 0 : 1);
    }
    cand = (uint32_t)(e0 + 8 * (128 * tf + 32 * wq + lane) + ef);
  }
  const float negm = -m;
  float2 acc = chunk_exp_sum2(v[0], negm);
#pragma unroll
  for (int t = 1; t < kChunksPerLane; ++t) acc = __fadd2_rn(acc, chunk_exp_sum2(v[t], negm));
  float ls = acc.x + acc.y;
  p.a = __reduce_min_sync(0xffffffffu, cand);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
  p.s = ls;
  return p;
}

#ifdef LOPA_LDG_TL
// experiment: per-warp %globaltimer stamps of the warp-staged K1 (lopa_debug_ldg_timeline)
constexpr int kLtlItems = 40;
__device__ unsigned long long g_ldg_tl[160][kLThreads / 32][2 + 3 * kLtlItems];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
__global__ void __launch_bounds__(kLThreads, 1) lopa_reduce_ldg_kernel(const Params P) {
  extern __shared__ __align__(128) uint8_t lsm[];  // [warp][kLBufs][kSliceChunks] 16-byte chunks
  // per team: slot ring of item descriptors (row, group, segments in the item, -); row -1 = end
  // of the team's work, -2 = no item
  __shared__ int4 sinfo[kTeams][kLSlots];
  __shared__ __align__(8) uint64_t ready[kTeams][kLSlots];
  __shared__ __align__(8) uint64_t sfree[kTeams][kLSlots];
  __shared__ float4 ipart[kTeams][kLSlots][kTeamWarps];
  __shared__ uint32_t icnt[kTeams][kLSlots];
  __shared__ uint32_t gbits[2 * kMaxGroups];
  __shared__ uint16_t vlist[kTeams][LOPA_MAX_ROWS];  // a team leader's valid-row list

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = warp / kTeamWarps, j = warp % kTeamWarps;
  const int jseg = j / kWarpsPerSeg, wq = j % kWarpsPerSeg;
  const bool leader = j == 0 && lane == 0;
  const int W = P.window;
  const int n_seg = P.n_seg, n_grp = P.n_grp;
  const int G = (int)gridDim.x;
  const int b = blockIdx.x;
  const int n_items_cap = P.n_cand * n_grp;
  const int n_spec = kLSpec * G;  // raw items [0, n_spec) are speculative first items
  const bool dyn = n_spec < n_items_cap;
  const uint64_t pol = policy_evict_first();
  uint4* bufs = reinterpret_cast<uint4*>(lsm) + (size_t)warp * kLBufs * kSliceChunks + lane;
#ifdef LOPA_LDG_TL
  unsigned long long* tl = g_ldg_tl[blockIdx.x][warp];
  if (lane == 0) tl[0] = gtime();
#endif
  if (tid < kTeams * kLSlots) {
    mbar_init(&ready[0][0] + tid, 1);
    mbar_init(&sfree[0][0] + tid, 1);
    (&icnt[0][0])[tid] = 0;
  }
  fence_mbar_init();
  grid_dep_wait();
  grid_dep_launch();
  __syncthreads();  // mbarrier inits

  uint32_t u = 0;  // leader: items published so far by its team
  auto publish = [&](int row, int g) {
    const int slot = (int)(u % kLSlots);
    if (u >= (uint32_t)kLSlots) mbar_wait(&sfree[team][slot], ((u / kLSlots) - 1) & 1);
    const int s0 = g * kSegPerItem;
    sinfo[team][slot] = make_int4(row, g, row >= 0 ? min(n_seg, s0 + kSegPerItem) - s0 : 0, 0);
    mbar_arrive(&ready[team][slot]);
    ++u;
  };
  uint32_t p1 = 0x7FFFFFFFu, p2 = 0x7FFFFFFFu;
  if (leader) {
    if (team < kLSpec) {
      const int r = team * G + b;  // no division for the common first item
      if (r < P.n_cand) publish(r, 0);
      else if (r < n_items_cap) publish(r % P.n_cand, r / P.n_cand);
      else publish(-2, 0);
    }
    if (dyn) {  // the first two claims travel while the masks load
      p1 = atom_add_u32(&P.ctrs[0], 1u);
      p2 = atom_add_u32(&P.ctrs[0], 1u);
    }
  }
  struct Task {
    int row, g, slot, nsi;
  };
  auto fetch = [&](uint32_t k) -> Task {
    const int slot = (int)(k % kLSlots);
    mbar_wait(&ready[team][slot], (k / kLSlots) & 1);
    const int4 in = sinfo[team][slot];
    return Task{in.x, in.y, slot, in.z};
  };
  auto seg_geom = [&](const Task& t, int* e0, int* nch) {
    const int seg = t.g * kSegPerItem + jseg;
    *e0 = seg * P.seg_len;
    const int e1 = min(P.vocab, *e0 + P.seg_len);
    *nch = (e1 - *e0 + 7) >> 3;
  };
  // copy this warp's slice of item t into buffer `buf` (this lane's chunks only)
  auto stage = [&](const Task& t, int buf) {
    int e0, nch;
    seg_geom(t, &e0, &nch);
    const uint4* src = reinterpret_cast<const uint4*>(P.logits + (size_t)t.row * P.ld + e0);
    uint4* dst = bufs + buf * kSliceChunks;
#pragma unroll
    for (int i = 0; i < kChunksPerLane; ++i) {
      const int c = 128 * i + 32 * wq + lane;
      if (c < nch) cp_async16(dst + 32 * i, src + c, pol);
    }
  };
  if (team < kLSpec) {
    // the speculative first item: its copies leave before the masks arrive
    const Task t = fetch(0);
    if (t.row >= 0 && jseg < t.nsi) stage(t, 0);
    cp_async_commit();
  }
  // valid-row bits: mask byte and n_branches loaded independently (one round trip)
  const int n_groups = (P.n_cand + 31) >> 5;
  for (int gq = warp; gq < n_groups; gq += kLThreads / 32) {
    const int r = gq * 32 + lane;
    const bool in = r < P.n_cand;
    const int nb_eff = P.n_branches ? *P.n_branches - P.branch_base : 0x7FFFFFFF;
    // the mask byte is read only for rows of present branches (r / W < nb_eff)
    bool v = in && (!P.n_branches || (int64_t)r < (int64_t)nb_eff * W);
    if (v && P.row_mask) {
      LOPA_CHK((int64_t)P.branch_base * W + r < (int64_t)P.table_rows * W, 2);
      v = P.row_mask[r] != 0;
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, v);
    if (lane == 0) gbits[gq] = bits;
  }
  __syncthreads();
  auto row_valid = [&](int r) -> bool { return (gbits[r >> 5] >> (r & 31)) & 1u; };

  // ---- the leader warp's item space (the same decision in every team of every CTA)
  bool compact = false;
  int n_rows = P.n_cand, lo = 0, q = 0, n0 = 0, n_dyn = 0;
  if (j == 0) {
    int nv = 0;
    for (int w = lane; w < n_groups; w += 32) nv += __popc(gbits[w]);
    const int n_valid = (int)__reduce_add_sync(0xffffffffu, (unsigned)nv);
#ifndef LOPA_NO_COMPACT
    compact = 8 * n_valid < 7 * P.n_cand;
#endif
    if (compact) {
      q = n_spec / P.n_cand;  // n_cand > 0 here
      const int rq = n_spec - q * P.n_cand;
      n_rows = n_valid;
      int base = 0;
#pragma unroll 1
      for (int w = 0; w < n_groups; ++w) {
        const uint32_t bits = gbits[w];
        if ((bits >> lane) & 1u) vlist[team][base + __popc(bits & ((1u << lane) - 1u))] = (uint16_t)(32 * w + lane);
        if (32 * w < rq) lo += __popc(32 * w + 32 <= rq ? bits : bits & ((1u << (rq - 32 * w)) - 1u));
        base += __popc(bits);
      }
      __syncwarp();
      n0 = q < n_grp ? n_rows - lo : 0;
      n_dyn = q < n_grp ? n0 + (n_grp - 1 - q) * n_rows : 0;
    } else {
      n_dyn = dyn ? n_items_cap - n_spec : 0;
    }
  }
  // Leader: publish the team's next item from the oldest claim (the end sentinel once the claims
  // run out), and keep two claims in flight.  Returns false once the sentinel is published.
  bool claiming = dyn;
  auto publish_next = [&]() -> bool {
    while (claiming) {
      const int d = (int)p1;
      if (d >= n_dyn) {
        claiming = false;
        break;
      }
      p1 = p2;
      p2 = atom_add_u32(&P.ctrs[0], 1u);
      if (compact) {
        int g = q, x = lo + d;
        if (d >= n0) {
          const int e = d - n0;
          g = q + 1 + e / n_rows;
          x = e - (g - q - 1) * n_rows;
        }
        publish(vlist[team][x], g);
        return true;
      }
      const int c = n_spec + d;
      const int g = c / P.n_cand, row = c - g * P.n_cand;
      if (row_valid(row)) {
        publish(row, g);
        return true;
      }
    }
    // done claiming: every outstanding claim has returned (p1, p2 consumed); the last of all
    // the leaders to get here zeroes the counter (K1 leaves the workspace zeroed)
    asm volatile("" ::"r"(p1), "r"(p2));
    if (dyn) {
      __threadfence();
      if (atomicAdd(&P.ctrs[1], 1u) == (uint32_t)(G * kTeams) - 1) {
        __threadfence();
        P.ctrs[0] = 0;
        P.ctrs[1] = 0;
      }
    }
    publish(-1, 0);
    return false;
  };
  bool more = true;  // leader: items remain to be published
  auto ensure_published = [&](uint32_t last) {  // items 0 .. last (or up to the sentinel)
    while (more && u <= last) more = publish_next();
  };

  // ---- reduce item t from buffer `buf`; the last of the 8 warps folds the item
  auto consume = [&](const Task& t, int buf) {
    const bool valid = t.row >= 0 && row_valid(t.row);
    if (valid && jseg < t.nsi) {
      int e0, nch;
      seg_geom(t, &e0, &nch);
      const uint4* src = bufs + buf * kSliceChunks;
      uint4 v[kChunksPerLane];
#pragma unroll
      for (int i = 0; i < kChunksPerLane; ++i) {
        const int c = 128 * i + 32 * wq + lane;
        v[i] = (c < nch) ? lds128(src + 32 * i)
                         : make_uint4(kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2, kNegInfBf16x2);
      }
#ifdef LOPA_LDG_NOCOMPUTE
      // streaming experiment: consume the slice and return a dummy partial
      uint32_t acc = 0;
#pragma unroll
      for (int i = 0; i < kChunksPerLane; ++i) acc ^= v[i].x ^ v[i].y ^ v[i].z ^ v[i].w;
      Partial pr;
      pr.m = 0.f;
      pr.s = 1.0f + (acc == 0x12345678u ? 1.f : 0.f);
      pr.a = 0;
      (void)e0;
#else
      const Partial pr = reduce_regs(v, nch, e0, P.vocab, wq, lane);
#endif
      if (lane == 0) ipart[team][t.slot][jseg * kWarpsPerSeg + wq] = make_float4(pr.m, pr.s, __uint_as_float(pr.a), 0.f);
    }
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd_block(&icnt[team][t.slot], 1u) + 1u == (uint32_t)kTeamWarps) {
        __threadfence_block();
        if (valid) {
          const float4* qp = ipart[team][t.slot];
          const FoldAcc f = fold_seq(kWarpsPerSeg * t.nsi, [&](int p) { return qp[p]; });
          store_partial(P.gpart + (size_t)t.g * P.n_cand + t.row, f, P.ctrs[2] + 1u);
        }
        icnt[team][t.slot] = 0;
        mbar_arrive(&sfree[team][t.slot]);
      }
    }
    __syncwarp();
  };

  // ---- stage kLDepth items ahead; one commit group per item (empty once the end is staged)
  uint32_t k_staged = team < kLSpec ? 1u : 0u;  // next item to stage
  uint32_t k_end = 0xFFFFFFFFu;                 // the item holding the end sentinel
  auto stage_next = [&]() {
    if (k_end == 0xFFFFFFFFu) {
      const Task t = fetch(k_staged);
      if (t.row == -1) k_end = k_staged;
      else if (t.row >= 0 && jseg < t.nsi && row_valid(t.row)) stage(t, (int)(k_staged % kLBufs));
      ++k_staged;
    }
    cp_async_commit();
  };
  if (leader) ensure_published(kLDepth);
  for (uint32_t c = k_staged; c < (uint32_t)kLDepth; ++c) stage_next();
#ifdef LOPA_LDG_TL
  if (lane == 0) tl[1] = gtime();
#endif
  for (uint32_t k = 0;; ++k) {
#ifdef LOPA_LDG_TL
    if (lane == 0 && k < kLtlItems) tl[2 + 3 * k] = gtime();
#endif
    if (leader) ensure_published(k + kLDepth + 1);
    stage_next();               // item k + kLDepth
    cp_async_wait<kLDepth>();   // item k has landed
#ifdef LOPA_LDG_TL
    if (lane == 0 && k < kLtlItems) tl[3 + 3 * k] = gtime();
#endif
    if (k == k_end) break;
    const int slot = (int)(k % kLSlots);
    const int4 in = sinfo[team][slot];
    consume(Task{in.x, in.y, slot, in.z}, (int)(k % kLBufs));
#ifdef LOPA_LDG_TL
    if (lane == 0 && k < kLtlItems) tl[4 + 3 * k] = gtime();
#endif
  }
}
