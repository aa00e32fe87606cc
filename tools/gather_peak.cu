// gather_peak.cu -- measured ceilings for the relaxation's memory pattern on
// this GPU (the denominator the relax kernels are judged against besides HBM
// bandwidth):
//   * stream:  coalesced u32 read of the index stream alone
//   * gather:  idx = col[e] (coalesced u32 stream), then one random 8 B load
//              cells[idx] -- the dist[dst] pre-check of every relaxation
//   * atomic:  idx stream + random 64-bit atomicMin on cells[idx]
// over a cells array of N 8-byte cells (N = 2^22: the C2 distance array,
// 33.5 MB) and E = 2^26 indices drawn uniformly (worst case) or from the
// C2-like skewed R-MAT-ish distribution (a power law via squaring).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_peak tools/gather_peak.cu
//   ./gather_peak [log2N=22] [log2E=26]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void k_stream(const uint32_t* __restrict__ col, long long E, unsigned long long* sink) {
  uint32_t acc = 0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
       e += (long long)gridDim.x * blockDim.x)
    acc += __ldcs(col + e);
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int U>
__global__ void k_gather(const uint32_t* __restrict__ col, const unsigned long long* cells,
                         long long E, unsigned long long* sink) {
  unsigned long long acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; e0 < E; e0 += stride * U) {
    uint32_t v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = e0 + k * stride < E ? __ldcs(col + e0 + k * stride) : 0u;
    unsigned long long d[U];
#pragma unroll
    for (int k = 0; k < U; ++k) d[k] = cells[v[k]];
#pragma unroll
    for (int k = 0; k < U; ++k) acc += d[k];
  }
  if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

template <int U>
__global__ void k_atomic(const uint32_t* __restrict__ col, unsigned long long* cells, long long E,
                         unsigned long long* sink) {
  unsigned long long acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; e0 < E; e0 += stride * U) {
    uint32_t v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = e0 + k * stride < E ? __ldcs(col + e0 + k * stride) : 0u;
    unsigned long long o[U];
#pragma unroll
    for (int k = 0; k < U; ++k) o[k] = atomicMin(cells + v[k], (unsigned long long)(e0 & 0xFFFF));
#pragma unroll
    for (int k = 0; k < U; ++k) acc += o[k];
  }
  if (acc == 0x12345678ull) atomicAdd(sink, 1ull);
}

template <typename F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const int ln = argc > 1 ? atoi(argv[1]) : 22;
  const int le = argc > 2 ? atoi(argv[2]) : 26;
  const long long N = 1ll << ln, E = 1ll << le;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<uint32_t> h(E);
  uint64_t x = 88172645463325252ull;
  for (int dist = 0; dist < 2; ++dist) {
    for (long long i = 0; i < E; ++i) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      double u = (double)(x >> 11) * (1.0 / 9007199254740992.0);
      if (dist == 1) u = u * u * u;  // skewed: low ids are hot (as in R-MAT)
      h[i] = (uint32_t)(u * (double)N) & (uint32_t)(N - 1);
    }
    uint32_t* col;
    unsigned long long *cells, *sink;
    CK(cudaMalloc(&col, E * 4));
    CK(cudaMalloc(&cells, N * 8));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemcpy(col, h.data(), E * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(cells, 0xFF, N * 8));
    const int block = 256;
    float ts = time_ms([&] { k_stream<<<sms * 8, block>>>(col, E, sink); }, 5);
    printf("{\"indices\": \"%s\", \"N\": %lld, \"E\": %lld, \"stream_GBs\": %.1f",
           dist ? "skewed(u^3)" : "uniform", N, E, E * 4 / ts / 1e6);
    for (int cps : {2, 4, 8}) {  // CTAs of 256 threads per SM: outstanding gathers per SM
      const int grid = sms * cps;
      float tg4 = time_ms([&] { k_gather<4><<<grid, block>>>(col, cells, E, sink); }, 5);
      float tg8 = time_ms([&] { k_gather<8><<<grid, block>>>(col, cells, E, sink); }, 5);
      float tg16 = time_ms([&] { k_gather<16><<<grid, block>>>(col, cells, E, sink); }, 5);
      float ta4 = time_ms([&] { k_atomic<4><<<grid, block>>>(col, cells, E, sink); }, 5);
      printf(", \"cta%d\": {\"gather_u4_Gps\": %.1f, \"gather_u8_Gps\": %.1f, \"gather_u16_Gps\": %.1f, "
             "\"atomic_u4_Gps\": %.1f}", cps, E / tg4 / 1e6, E / tg8 / 1e6, E / tg16 / 1e6, E / ta4 / 1e6);
    }
    printf("}\n");
    cudaFree(col);
    cudaFree(cells);
    cudaFree(sink);
  }
  return 0;
}
