// NEXT-1 on the device: the D2F block pipeline (readings R25 / R26)
// as device state plus one scheduler kernel, so a whole multi-block decode -- forward,
// lopa_step on the active window (window read on the device), scheduler -- runs with no host
// read and can be captured in one CUDA graph (lopa.D2FDeviceLoop).  The rules are those of the
// host pipeline paper_2512_16229_b200/d2f.py, which the GPU tests compare against the oracle:
//   after each verify step, on the selected branch B* (x_{t+1} = B* on the window):
//   (a) commit the oldest active blocks that B* fills completely, stopping at the first that is
//       not full;
//   (b) if no block is active, activate the next; else activate it when the newest active
//       block's fill ratio >= tau_add (exact, in double) and the window stays <= max_window;
//   the spawned branches carry over (committed columns dropped, new blocks appended from the
//   region, i.e. fully masked); a step that completed its window (n_next = 0, R21) is followed
//   by the new window's initial predict (one branch = the region).
#include <cstdint>

#include "liblopa.h"
#include "lopa_internal.h"

namespace lopa {
namespace d2f {

constexpr int kInactive = 0, kActive = 1, kCommitted = 2;
constexpr int kThreads = 256;  // one thread per window position (W <= 256)

__device__ __forceinline__ float window_tau(const lopa_d2f_t& d, int q0, int c, int last_active) {
  return ((q0 + c) / d.block_size == last_active) ? d.tau_act : d.tau_conf;
}

__global__ void __launch_bounds__(kThreads) init_kernel(const lopa_d2f_t d) {
  const int B = d.block_size, nblk = d.gen_len / B;
  for (int p = threadIdx.x; p < d.gen_len; p += kThreads) d.region_mask[p] = 1;
  for (int b = threadIdx.x; b < nblk; b += kThreads) {
    d.block_status[b] = b == 0 ? kActive : kInactive;
    d.commit_order[b] = -1;
  }
  for (int c = threadIdx.x; c < B; c += kThreads) {
    d.branch_tokens[c] = d.region_tokens[c];
    d.branch_mask[c] = 1;
    d.tau_pos[c] = d.tau_act;
  }
  if (threadIdx.x == 0) {
    d.sched[0] = 0;   // window start p0
    d.sched[1] = B;   // window W
    d.sched[2] = 1;   // branches of the next step (the initial predict)
    d.sched[3] = 0;   // done
    d.sched[4] = 0;   // forwards
    d.sched[5] = 0;   // committed blocks
  }
}

__global__ void __launch_bounds__(kThreads) update_kernel(const lopa_d2f_t d, const int32_t* winner,
                                                          const int32_t* n_next,
                                                          const int32_t* next_tokens,
                                                          const uint8_t* next_mask) {
  __shared__ int s_cnt[LOPA_MAX_WINDOW];  // masked positions of B* per active block
  __shared__ int s_q0, s_wn, s_last, s_done;
  const int tid = threadIdx.x;
  const int B = d.block_size, nblk = d.gen_len / B;
  if (d.sched[3]) return;  // the decode is complete: later iterations are no-ops
  const int p0 = d.sched[0], W = d.sched[1], n = d.sched[2];
  const int w = *winner, nn = *n_next;
  const int b0 = p0 / B, nact = W / B;
  if (tid == 0 && d.trace && d.sched[4] < d.trace_cap) {
    int32_t* t = d.trace + 4 * d.sched[4];
    t[0] = p0;
    t[1] = W;
    t[2] = n;
    t[3] = w;
  }
  for (int a = tid; a < nact; a += kThreads) s_cnt[a] = 0;
  __syncthreads();
  // x_{t+1} = B* on the window; masked count per active block
  for (int c = tid; c < W; c += kThreads) {
    const uint8_t m = d.branch_mask[(size_t)w * W + c];
    d.region_tokens[p0 + c] = d.branch_tokens[(size_t)w * W + c];
    d.region_mask[p0 + c] = m;
    if (m) atomicAdd(&s_cnt[c / B], 1);
  }
  __syncthreads();
  if (tid == 0) {
    // (a) commit the oldest active blocks that are full
    int ncomm = d.sched[5];
    int first = b0;
    for (int a = 0; a < nact; ++a) {
      if (s_cnt[a] != 0) break;
      d.block_status[b0 + a] = kCommitted;
      d.commit_order[ncomm++] = b0 + a;
      first = b0 + a + 1;
    }
    int last = b0 + nact - 1;  // newest active block (if any remains)
    int na = last - first + 1;
    // (b) activate the next block
    const int nxt = b0 + nact;
    if (nxt < nblk) {
      bool act = false;
      if (na <= 0) {
        act = true;
      } else {
        const int filled = B - s_cnt[last - b0];
        act = (double)filled / (double)B >= d.tau_add && (na + 1) * B <= d.max_window;
      }
      if (act) {
        d.block_status[nxt] = kActive;
        if (na <= 0) first = nxt;
        last = nxt;
        na = last - first + 1;
      }
    }
    d.sched[5] = ncomm;
    s_done = ncomm == nblk;
    s_q0 = first * B;
    s_wn = na * B;
    s_last = last;
  }
  __syncthreads();
  if (s_done) {
    if (tid == 0) {
      d.sched[2] = 0;
      d.sched[3] = 1;
      d.sched[4] += 1;
    }
    return;
  }
  const int q0 = s_q0, WN = s_wn;
  for (int c = tid; c < WN; c += kThreads) d.tau_pos[c] = window_tau(d, q0, c, s_last);
  // the next step's tables, laid out [n_new][WN]
  const int n_new = nn == 0 ? 1 : nn;
  for (int e = tid; e < n_new * WN; e += kThreads) {
    const int j = e / WN, c = e - j * WN;
    const int p = q0 + c;
    int32_t t;
    uint8_t m;
    if (nn > 0 && p >= p0 && p < p0 + W) {
      t = next_tokens[(size_t)j * W + (p - p0)];
      m = next_mask[(size_t)j * W + (p - p0)];
    } else {
      t = d.region_tokens[p];
      m = d.region_mask[p];
    }
    d.branch_tokens[(size_t)j * WN + c] = t;
    d.branch_mask[(size_t)j * WN + c] = m;
  }
  if (tid == 0) {
    d.sched[0] = q0;
    d.sched[1] = WN;
    d.sched[2] = n_new;
    d.sched[4] += 1;
  }
}

static bool config_ok(const lopa_d2f_t* d) {
  return d && d->block_size >= 1 && d->gen_len >= d->block_size && d->gen_len % d->block_size == 0 &&
         d->max_window >= d->block_size && d->max_window <= LOPA_MAX_WINDOW && d->k >= 0 &&
         d->k + 1 <= LOPA_MAX_BRANCHES && d->trace_cap >= 0 && d->tau_act > 0.f &&
         d->tau_act <= 1.f && d->tau_conf > 0.f && d->tau_conf <= 1.f && d->region_tokens &&
         d->region_mask && d->block_status && d->sched && d->tau_pos && d->branch_tokens &&
         d->branch_mask && d->commit_order && (d->trace || d->trace_cap == 0);
}

}  // namespace d2f
}  // namespace lopa

extern "C" int lopa_d2f_init(const lopa_d2f_t* d, void* stream) {
  if (!lopa::d2f::config_ok(d)) return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!lopa::bind_device(stream, d->sched, &dev)) return LOPA_ERR_CUDA;
  lopa::d2f::init_kernel<<<1, lopa::d2f::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(*d);
  return lopa::cuda_status(cudaGetLastError());
}

extern "C" int lopa_d2f_update(const lopa_d2f_t* d, const int32_t* winner, const int32_t* n_next,
                               const int32_t* next_tokens, const uint8_t* next_mask, void* stream) {
  if (!lopa::d2f::config_ok(d) || !winner || !n_next || !next_tokens || !next_mask)
    return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!lopa::bind_device(stream, d->sched, &dev)) return LOPA_ERR_CUDA;
  lopa::d2f::update_kernel<<<1, lopa::d2f::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      *d, winner, n_next, next_tokens, next_mask);
  return lopa::cuda_status(cudaGetLastError());
}
