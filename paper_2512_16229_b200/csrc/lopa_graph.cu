// Device-terminated loops: a CUDA graph whose body repeats on the device, under a conditional
// WHILE node, until a condition word says stop -- the Alg. 1 loop ("until the selected
// branch has no masked position", R21) and the D2F decode ("until every block is committed")
// with no host involvement and no iteration budget (CUDA graphs instead of a tracing compiler).
// The body is whatever the caller issues on the stream between lopa_while_begin and
// lopa_while_end (captured into the conditional node's body graph); lopa_while_end appends the
// condition kernel.
#include <cstdint>
#include <new>

#include "liblopa.h"
#include "lopa_internal.h"

namespace lopa {
namespace wg {

// Continue while the word is non-zero (until_zero) / zero (!until_zero), and fewer than
// max_iters iterations have run (the iteration counter is reset by lopa_while_launch).
__global__ void continue_kernel(cudaGraphConditionalHandle h, const int32_t* word, int32_t until_zero,
                                int32_t* iters, int32_t max_iters) {
  const int32_t it = ++(*iters);
  const bool go = (until_zero ? (*word != 0) : (*word == 0)) && it < max_iters;
  cudaGraphSetConditional(h, go ? 1u : 0u);
}

__global__ void reset_kernel(int32_t* iters) { *iters = 0; }

}  // namespace wg
}  // namespace lopa

struct lopa_while {
  cudaGraph_t graph = nullptr;
  cudaGraph_t body = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
  cudaStream_t stream = nullptr;
  const int32_t* word = nullptr;
  int32_t until_zero = 1;
  int32_t max_iters = 1;
  int32_t* iters = nullptr;  // device counter
  bool capturing = false;
};

extern "C" int lopa_while_begin(void* stream, const int32_t* cond_word, int32_t until_zero,
                                int32_t max_iters, lopa_while_t** out) {
  if (!stream || !cond_word || !out || max_iters < 1) return LOPA_ERR_INVALID_ARG;
  int dev;
  if (!lopa::bind_device(stream, cond_word, &dev)) return LOPA_ERR_CUDA;
  lopa_while_t* w = new (std::nothrow) lopa_while_t;
  if (!w) return LOPA_ERR_CUDA;
  w->stream = static_cast<cudaStream_t>(stream);
  w->word = cond_word;
  w->until_zero = until_zero ? 1 : 0;
  w->max_iters = max_iters;
  cudaError_t e = cudaMalloc(&w->iters, sizeof(int32_t));
  if (e == cudaSuccess) e = cudaGraphCreate(&w->graph, 0);
  // the loop runs at least once per launch (default value 1), then as the body's last kernel says
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&w->handle, w->graph, 1, cudaGraphCondAssignDefault);
  cudaGraphNode_t node;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = w->handle;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  if (e == cudaSuccess) e = cudaGraphAddNode(&node, w->graph, nullptr, 0, &p);
  if (e == cudaSuccess) {
    w->body = p.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(w->stream, w->body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
  }
  if (e != cudaSuccess) {
    if (w->graph) cudaGraphDestroy(w->graph);
    if (w->iters) cudaFree(w->iters);
    delete w;
    return lopa::cuda_status(e);
  }
  w->capturing = true;
  *out = w;
  return LOPA_OK;
}

extern "C" int lopa_while_end(lopa_while_t* w) {
  if (!w || !w->capturing) return LOPA_ERR_INVALID_ARG;
  lopa::wg::continue_kernel<<<1, 1, 0, w->stream>>>(w->handle, w->word, w->until_zero, w->iters,
                                                      w->max_iters);
  cudaError_t e = cudaGetLastError();
  cudaGraph_t captured = nullptr;
  const cudaError_t e2 = cudaStreamEndCapture(w->stream, &captured);
  w->capturing = false;
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&w->exec, w->graph, 0);
  return lopa::cuda_status(e);
}

extern "C" int lopa_while_launch(lopa_while_t* w, void* stream) {
  if (!w || !w->exec || w->capturing) return LOPA_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
  lopa::wg::reset_kernel<<<1, 1, 0, s>>>(w->iters);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaGraphLaunch(w->exec, s);
  return lopa::cuda_status(e);
}

extern "C" int lopa_while_iterations(const lopa_while_t* w, int32_t* out_host) {
  if (!w || !out_host) return LOPA_ERR_INVALID_ARG;
  return lopa::cuda_status(cudaMemcpy(out_host, w->iters, sizeof(int32_t), cudaMemcpyDeviceToHost));
}

extern "C" void lopa_while_destroy(lopa_while_t* w) {
  if (!w) return;
  if (w->capturing) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(w->stream, &g);
  }
  if (w->exec) cudaGraphExecDestroy(w->exec);
  if (w->graph) cudaGraphDestroy(w->graph);
  if (w->iters) cudaFree(w->iters);
  delete w;
}
