// glb_peak.cu -- measured ceilings of the relaxation's memory pattern on the
// graph itself (glb_measure_gather): the rate at which the device can stream
// a graph's col array and gather one 8-byte cell per edge, dist[col[e]], at
// full occupancy -- the random-sector gather every relaxation does before its
// atomicMin.  bench.py reports the relax kernels against it next to the HBM
// roofline: this path is bound by random 32 B sector gathers through L1TEX
// (about one per cycle per SM), not by HBM bytes.  tools/gather_peak.cu is
// the standalone version over synthetic indices.
#include <cuda_runtime.h>

#include <algorithm>

#include "glb_internal.cuh"

namespace glb {
namespace {

template <int U>
__global__ void k_peak_gather(const uint32_t* __restrict__ col, const unsigned long long* cells,
                              long long m, unsigned long long* sink) {
  unsigned long long acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; e0 < m; e0 += stride * U) {
    uint32_t v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = e0 + k * stride < m ? __ldcs(col + e0 + k * stride) : 0u;
    unsigned long long d[U];
#pragma unroll
    for (int k = 0; k < U; ++k) d[k] = cells[v[k]];
#pragma unroll
    for (int k = 0; k < U; ++k) acc += d[k];
  }
  if (acc == 0x5bd1e995ull) atomicAdd(sink, 1ull);  // keeps the loads alive
}

template <int U>
__global__ void k_peak_atomic(const uint32_t* __restrict__ col, unsigned long long* cells,
                              long long m, unsigned long long* sink) {
  unsigned long long acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; e0 < m; e0 += stride * U) {
    uint32_t v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = e0 + k * stride < m ? __ldcs(col + e0 + k * stride) : 0u;
    unsigned long long o[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      o[k] = e0 + k * stride < m ? atomicMin(cells + v[k], (unsigned long long)(e0 + k)) : 0ull;
#pragma unroll
    for (int k = 0; k < U; ++k) acc += o[k];
  }
  if (acc == 0x5bd1e995ull) atomicAdd(sink, 1ull);
}

__global__ void k_peak_stream(const uint32_t* __restrict__ col, long long m,
                              unsigned long long* sink) {
  uint32_t acc = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x)
    acc += __ldcs(col + e);
  if (acc == 0x5bd1e995u) atomicAdd(sink, 1ull);
}

template <typename F>
float best_ms(cudaStream_t s, cudaEvent_t a, cudaEvent_t b, int reps, F f) {
  f();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    GLB_CUDA_TRY(cudaEventRecord(a, s));
    f();
    GLB_CUDA_TRY(cudaEventRecord(b, s));
    GLB_CUDA_TRY(cudaEventSynchronize(b));
    float ms = 0;
    GLB_CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  return best;
}

}  // namespace

void measure_gather(glb_graph* g, double out[4]) {
  const long long m = g->m, n = g->n;
  out[0] = out[1] = out[2] = out[3] = 0;
  if (m == 0 || n == 0) return;
  cudaStream_t s = g->stream;
  unsigned long long* cells = (unsigned long long*)dmalloc((size_t)n * 8 + 64);
  unsigned long long* sink = cells + n;
  cudaEvent_t a = nullptr, b = nullptr;
  try {
    GLB_CUDA_TRY(cudaEventCreate(&a));
    GLB_CUDA_TRY(cudaEventCreate(&b));
    GLB_CUDA_TRY(cudaMemsetAsync(cells, 0xFF, (size_t)n * 8 + 64, s));
    const unsigned grid = (unsigned)g->num_sms * 8;
    const float ts = best_ms(s, a, b, 3, [&] {
      k_peak_stream<<<grid, kBlock, 0, s>>>(g->col, m, sink);
      GLB_CHECK_LAUNCH();
    });
    const float tg = best_ms(s, a, b, 3, [&] {
      k_peak_gather<8><<<grid, kBlock, 0, s>>>(g->col, cells, m, sink);
      GLB_CHECK_LAUNCH();
    });
    const float ta = best_ms(s, a, b, 3, [&] {
      k_peak_atomic<4><<<grid, kBlock, 0, s>>>(g->col, cells, m, sink);
      GLB_CHECK_LAUNCH();
    });
    out[0] = (double)m * 4 / (ts * 1e-3) / 1e9;  // col stream, GB/s
    out[1] = (double)m / (tg * 1e-3) / 1e9;      // col + dist[col] gathers, G/s
    out[2] = (double)m / (ta * 1e-3) / 1e9;      // col + atomicMin(dist[col]), G/s
    out[3] = (double)n * 8 / 1e6;                // gathered array, MB
  } catch (...) {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    cudaStreamSynchronize(s);
    dfree(cells);
    throw;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  GLB_CUDA_TRY(cudaStreamSynchronize(s));
  dfree(cells);
}

}  // namespace glb
