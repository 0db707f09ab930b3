// Microbenchmark: streaming read bandwidth of a persistent TMA (cp.async.bulk) ring, vs stage
// size / depth / CTAs per SM / consumer work; and an LDG.128 streaming kernel.  Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_16229_b200/csrc/lopa_ptx.cuh"
using namespace lopa;

__global__ void tma_stream(const uint8_t* src, size_t total, int stage_bytes, int stages,
                           int n_cons_warps, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], n_cons_warps); }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t n_chunks = total / stage_bytes;
  const size_t G = gridDim.x;
  // contiguous interleave: CTA b takes chunks b, b + G, ...
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t i = 0;
      for (size_t c = blockIdx.x; c < n_chunks; c += G, ++i) {
        const int s = i % stages;
        if (i >= (uint32_t)stages) mbar_wait(&empty[s], ((i / stages) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        bulk_g2s(sm + (size_t)s * stage_bytes, src + c * stage_bytes, stage_bytes, &full[s], pol);
      }
    }
    return;
  }
  unsigned acc = 0;
  uint32_t i = 0;
  for (size_t c = blockIdx.x; c < n_chunks; c += G, ++i) {
    const int s = i % stages;
    mbar_wait(&full[s], (i / stages) & 1);
    const uint4* b = reinterpret_cast<const uint4*>(sm + (size_t)s * stage_bytes);
    const int nw = stage_bytes / 16;
    for (int q = (warp - 1) * 32 + lane; q < nw; q += n_cons_warps * 32) {
      uint4 v = lds128(b + q);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

__global__ void ldg_stream(const uint4* src, size_t n16, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { uint4 v = src[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

int main() {
  const size_t total = (size_t)8 * 77792256;  // 8 Dream-size buffers (622 MB)
  uint8_t* src; unsigned* sink;
  cudaMalloc(&src, total); cudaMalloc(&sink, 4);
  cudaMemset(src, 1, total);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { int sb, st, cps, cw; };
  Cfg cfgs[] = {{16384, 8, 1, 12}, {16384, 12, 1, 12}, {32768, 6, 1, 12}, {65536, 3, 1, 12},
                {16384, 6, 2, 8}, {32768, 3, 2, 8}, {8192, 12, 2, 4}, {16384, 4, 3, 4},
                {8192, 8, 3, 4}, {4096, 16, 4, 2}, {32768, 6, 1, 4}, {16384, 12, 1, 4}};
  for (auto c : cfgs) {
    const size_t smem = (size_t)c.sb * c.st + 2 * c.st * 8;
    const int grid = sms * c.cps, threads = 32 * (1 + c.cw);
    for (int w = 0; w < 3; ++w) tma_stream<<<grid, threads, smem>>>(src, total, c.sb, c.st, c.cw, sink);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) tma_stream<<<grid, threads, smem>>>(src, total, c.sb, c.st, c.cw, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("TMA stage=%6d stages=%2d ctas/sm=%d cons_warps=%2d : %7.1f GB/s  (%s)\n", c.sb, c.st, c.cps,
           c.cw, reps * total / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  for (int tpb : {256, 512, 1024}) for (int cps : {1, 2, 4}) {
    if (tpb * cps > 2048) continue;
    for (int w = 0; w < 3; ++w) ldg_stream<<<sms * cps, tpb>>>((const uint4*)src, total / 16, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) ldg_stream<<<sms * cps, tpb>>>((const uint4*)src, total / 16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("LDG tpb=%4d ctas/sm=%d : %7.1f GB/s\n", tpb, cps, 5.0 * total / (ms / 1e3) / 1e9);
  }
  // Dream-size single buffers (77.8 MB each), rotating over 8 (L2-cold): per-launch time
  const size_t one = 77792256;
  for (auto c : cfgs) {
    const size_t smem = (size_t)c.sb * c.st + 2 * c.st * 8;
    const int grid = sms * c.cps, threads = 32 * (1 + c.cw);
    for (int w = 0; w < 8; ++w) tma_stream<<<grid, threads, smem>>>(src + (w % 8) * one, one, c.sb, c.st, c.cw, sink);
    cudaEventRecord(a);
    const int reps = 64;
    for (int r = 0; r < reps; ++r) tma_stream<<<grid, threads, smem>>>(src + (r % 8) * one, one, c.sb, c.st, c.cw, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("77.8MB TMA stage=%6d stages=%2d ctas/sm=%d cw=%2d : %6.2f us/launch %7.1f GB/s\n", c.sb, c.st, c.cps,
           c.cw, ms * 1e3 / reps, reps * one / (ms / 1e3) / 1e9);
  }
  for (int tpb : {512, 1024}) for (int cps : {1, 2}) {
    if (tpb * cps > 2048) continue;
    cudaEventRecord(a);
    for (int r = 0; r < 64; ++r) ldg_stream<<<sms * cps, tpb>>>((const uint4*)(src + (r % 8) * one), one / 16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("77.8MB LDG tpb=%4d ctas/sm=%d : %6.2f us/launch %7.1f GB/s\n", tpb, cps, ms * 1e3 / 64, 64.0 * one / (ms / 1e3) / 1e9);
  }
  return 0;
}
