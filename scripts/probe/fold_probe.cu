// Microbenchmark of the K2 row fold (one thread per row, 16-slot tree) — not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_16229_b200/csrc/lopa_ptx.cuh"
using namespace lopa;
struct FoldAcc { float M, S; uint32_t a; };
__device__ __forceinline__ FoldAcc fold_tree16(int n, const float4 (&q)[16]) {
  float M = -INFINITY;
#pragma unroll
  for (int p = 0; p < 16; ++p) M = fmaxf(M, p < n ? q[p].x : -INFINITY);
  float t[16]; uint32_t a = 0xFFFFFFFFu;
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    t[p] = p < n ? q[p].y * (M == -INFINITY ? 1.f : ex2((q[p].x - M) * kLog2e)) : 0.f;
    a = (p < n && q[p].x == M) ? min(a, __float_as_uint(q[p].z)) : a;
  }
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
    for (int p = 0; p < w; ++p) t[p] = t[2 * p] + t[2 * p + 1];
  return FoldAcc{M, t[0], a};
}
__global__ void writer(float4* g, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    g[i] = make_float4((i % 7) * 0.5f, 100.f + i, (float)i, 0.f);
}
__global__ void k(const float4* g, int nrows, int n_grp, float* conf, int* am, long long* clk, int variant) {
  long long t0 = clock64();
  for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
    float4 qr[16];
    if (variant >= 2) {  // group-major (coalesced)
#pragma unroll
      for (int p = 0; p < 16; ++p) qr[p] = p < n_grp ? __ldcg(g + (size_t)p * 256 + r) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const float4* q = g + (size_t)r * n_grp;
#pragma unroll
      for (int p = 0; p < 16; ++p) qr[p] = p < n_grp ? __ldcg(q + p) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    long long t1 = clock64();
    FoldAcc f = fold_tree16(n_grp, qr);
    long long t2 = clock64();
    float c = variant ? 1.0f / f.S : __fdiv_rn(1.0f, f.S);
    conf[r] = c; am[r] = f.a;
    long long t3 = clock64();
    if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; }
  }
}
int main() {
  const int nrows = 241, n_grp = 10;
  float4* g; float* conf; int* am; long long* clk;
  cudaMalloc(&g, nrows * n_grp * 16); cudaMalloc(&conf, 4096); cudaMalloc(&am, 4096); cudaMallocManaged(&clk, 64);
  float4 h[nrows * n_grp];
  for (int i = 0; i < nrows * n_grp; ++i) { float m = (i % 7) * 0.5f; h[i] = make_float4(m, 100.f + i, (float)i, 0.f); }
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaFree(g); cudaMalloc(&g, 256 * 16 * 16);
  for (int rep = 0; rep < 8; ++rep) {
    if (rep >= 4) writer<<<148, 256>>>(g, 256 * 16);
    k<<<1, 512>>>(g, nrows, n_grp, conf, am, clk, 2 + (rep & 1));
    cudaDeviceSynchronize();
    printf("rep %d (%s): load %lld  fold %lld  div+store %lld cycles\n", rep, rep >= 4 ? "after writer kernel" : "warm", clk[0], clk[1], clk[2]);
  }
  return 0;
}
