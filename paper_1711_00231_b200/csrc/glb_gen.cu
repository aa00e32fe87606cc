// glb_gen.cu -- R-MAT generation straight into HBM, draw-for-draw identical to
// the reference generator (generators.py:23-58 + CsrGraph.from_edges,
// csr.py:97-118) under numpy's PCG64 (XSL-RR 128/64) stream:
//   * level l, edge i uses raw draw l*m + i as a double (raw >> 11) * 2^-53;
//   * weights follow: u32 draw d (raw (scale*m + d/2), low half first) maps
//     to 1 + ((u32 * W) >> 32) with Lemire rejection of leftover < 2^32 mod W
//     (numpy's buffered_bounded_lemire_uint32);
//   * CSR grouping by source is a stable radix sort of (src, edge index).
// Every thread jumps the LCG to its own offset (O(log k) affine powers), so
// the whole generation is one pass over the edges per phase.  This makes the
// scale-27 configuration (2^31 edges) buildable and the benchmark inputs
// bit-identical to graphlb.generate_rmat at every scale.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>

#include "glb_internal.cuh"

namespace glb {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

// state after `delta` further steps (PCG's pcg_advance_lcg_128)
__host__ __device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ unsigned long long pcg_output(u128 s) {
  const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const unsigned long long x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct RmatParams {
  unsigned long long s_hi, s_lo, i_hi, i_lo;  // PCG64 state / increment
  unsigned long long m;                      // edges
  int scale;
  double t_a, t_ab, t_abc;                   // a, a+b, a+b+c as the reference computes them
  unsigned long long jump_m_mult_hi, jump_m_mult_lo, jump_m_plus_hi, jump_m_plus_lo;
};

constexpr int kGenB = 16;  // consecutive edges per thread

// src/dst of every edge: scale rounds of quadrant descent (generators.py:50-55)
__global__ void k_rmat_edges(RmatParams p, uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                             uint32_t* __restrict__ idx) {
  const u128 s0 = ((u128)p.s_hi << 64) | p.s_lo, inc = ((u128)p.i_hi << 64) | p.i_lo;
  const u128 jm = ((u128)p.jump_m_mult_hi << 64) | p.jump_m_mult_lo;
  const u128 jp = ((u128)p.jump_m_plus_hi << 64) | p.jump_m_plus_lo;
  const u128 mult = pcg_mult();
  const unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) * kGenB;
  if (base >= p.m) return;
  const int cnt = (int)(p.m - base < (unsigned long long)kGenB ? p.m - base : kGenB);
  uint32_t s[kGenB], d[kGenB];
#pragma unroll
  for (int j = 0; j < kGenB; ++j) s[j] = d[j] = 0;
  u128 lvl = pcg_advance(s0, inc, base);  // state before edge `base` of level 0
  for (int l = 0; l < p.scale; ++l) {
    u128 st = lvl;
#pragma unroll
    for (int j = 0; j < kGenB; ++j) {
      st = st * mult + inc;
      const double u = (double)(pcg_output(st) >> 11) * (1.0 / 9007199254740992.0);
      const uint32_t row_bit = u >= p.t_ab;
      const uint32_t col_bit = (u >= p.t_a && u < p.t_ab) || u >= p.t_abc;
      s[j] = (s[j] << 1) | row_bit;
      d[j] = (d[j] << 1) | col_bit;
    }
    lvl = jm * lvl + jp;  // jump m draws: next level, same edges
  }
  for (int j = 0; j < cnt; ++j) {
    src[base + j] = s[j];
    dst[base + j] = d[j];
    idx[base + j] = (uint32_t)(base + j);
  }
}

// u32 draws d in [0, ndraw) of rng.integers(1, W+1): value + rejection flag
__global__ void k_rmat_weight_draws(RmatParams p, unsigned long long ndraw, unsigned W,
                                    unsigned threshold, uint32_t* __restrict__ value,
                                    unsigned char* __restrict__ accept,
                                    unsigned long long* __restrict__ rejects_below_m) {
  const u128 s0 = ((u128)p.s_hi << 64) | p.s_lo, inc = ((u128)p.i_hi << 64) | p.i_lo;
  const u128 mult = pcg_mult();
  const unsigned long long d0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) * kGenB;
  if (d0 >= ndraw) return;
  // raw index of draw d is scale*m + d/2 (d0 is even)
  u128 st = pcg_advance(s0, inc, (unsigned long long)p.scale * p.m + d0 / 2);
  unsigned long long rej = 0;
#pragma unroll
  for (int j = 0; j < kGenB; j += 2) {
    st = st * mult + inc;
    const unsigned long long raw = pcg_output(st);
    const uint32_t half[2] = {(uint32_t)raw, (uint32_t)(raw >> 32)};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned long long d = d0 + j + h;
      if (d >= ndraw) break;
      const unsigned long long mm = (unsigned long long)half[h] * W;
      const bool ok = (uint32_t)mm >= threshold;
      value[d] = 1u + (uint32_t)(mm >> 32);
      accept[d] = ok;
      if (!ok && d < p.m) ++rej;
    }
  }
  if (rej) atomicAdd(rejects_below_m, rej);
}

__global__ void k_count_src(const uint32_t* __restrict__ src, unsigned long long m,
                            unsigned long long* __restrict__ cnt) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < m;
       i += (unsigned long long)gridDim.x * blockDim.x)
    atomicAdd(cnt + src[i], 1ull);
}

__global__ void k_gather_edges(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ dst,
                               const uint32_t* __restrict__ wdraw, unsigned long long m,
                               uint32_t* __restrict__ col, uint32_t* __restrict__ wt) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < m;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t e = perm[i];
    col[i] = dst[e];
    if (wt) wt[i] = wdraw[e];
  }
}

__global__ void k_i64_from_u64(const unsigned long long* __restrict__ s, long long* __restrict__ d,
                               long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = (long long)s[i];
}

// Fills g->row / g->col / g->wt (device) with the R-MAT graph.
void rmat_device(glb_graph* g, int scale, long long edge_factor, double t_a, double t_ab,
                 double t_abc, const unsigned long long state[2], const unsigned long long inc[2],
                 bool weighted, long long max_weight) {
  const long long n = 1ll << scale;
  const unsigned long long m = (unsigned long long)edge_factor * (unsigned long long)n;
  cudaStream_t s = g->stream;
  RmatParams p;
  p.s_hi = state[0];
  p.s_lo = state[1];
  p.i_hi = inc[0];
  p.i_lo = inc[1];
  p.m = m;
  p.scale = scale;
  p.t_a = t_a;
  p.t_ab = t_ab;
  p.t_abc = t_abc;
  {  // affine map of m LCG steps
    const u128 incv = ((u128)inc[0] << 64) | inc[1];
    // A = MULT^m, C = advance(0, inc, m): state' = A*state + C
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = incv;
    unsigned long long delta = m;
    while (delta) {
      if (delta & 1ull) {
        acc_mult *= cur_mult;
        acc_plus = acc_plus * cur_mult + cur_plus;
      }
      cur_plus = (cur_mult + 1) * cur_plus;
      cur_mult *= cur_mult;
      delta >>= 1;
    }
    p.jump_m_mult_hi = (unsigned long long)(acc_mult >> 64);
    p.jump_m_mult_lo = (unsigned long long)acc_mult;
    p.jump_m_plus_hi = (unsigned long long)(acc_plus >> 64);
    p.jump_m_plus_lo = (unsigned long long)acc_plus;
  }
  DevBuf b_src, b_dst, b_idx, b_keys2, b_idx2, b_val, b_acc, b_cnt, b_tmp, b_vsel;
  auto cleanup = [&] {
    DevBuf* all[] = {&b_src, &b_dst, &b_idx, &b_keys2, &b_idx2, &b_val, &b_acc, &b_cnt, &b_tmp, &b_vsel};
    for (auto* b : all) free_buf(*b);
  };
  try {
    const size_t mb = (size_t)std::max<unsigned long long>(m, 1);
    uint32_t* src = (uint32_t*)ensure(b_src, mb * 4);
    uint32_t* dst = (uint32_t*)ensure(b_dst, mb * 4);
    uint32_t* idx = (uint32_t*)ensure(b_idx, mb * 4);
    const unsigned long long threads = (m + kGenB - 1) / kGenB;
    if (m) {
      k_rmat_edges<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(p, src, dst, idx);
      GLB_CHECK_LAUNCH();
    }
    // ---- weights (drawn after the descent, generators.py:56)
    uint32_t* wdraw = nullptr;
    if (weighted && m) {
      const unsigned W = (unsigned)max_weight;
      const unsigned threshold = (unsigned)((1ull << 32) % W);
      unsigned long long slack = 256;
      unsigned long long* rej = (unsigned long long*)ensure(b_cnt, 64);
      while (true) {
        const unsigned long long ndraw = m + slack;
        uint32_t* val = (uint32_t*)ensure(b_val, (size_t)ndraw * 4);
        unsigned char* acc = (unsigned char*)ensure(b_acc, (size_t)ndraw);
        GLB_CUDA_TRY(cudaMemsetAsync(rej, 0, 8, s));
        const unsigned long long t2 = (ndraw + kGenB - 1) / kGenB;
        k_rmat_weight_draws<<<(unsigned)((t2 + 127) / 128), 128, 0, s>>>(p, ndraw, W, threshold, val,
                                                                         acc, rej);
        GLB_CHECK_LAUNCH();
        unsigned long long nrej = 0;
        GLB_CUDA_TRY(cudaMemcpyAsync(&nrej, rej, 8, cudaMemcpyDeviceToHost, s));
        GLB_CUDA_TRY(cudaStreamSynchronize(s));
        if (nrej == 0) {
          wdraw = val;  // draw i is weight i
          break;
        }
        if (nrej + 64 > slack) {  // not enough spare draws: widen and redo
          slack = (nrej + 64) * 2;
          continue;
        }
        // keep accepted draws in order (rare path): stable compaction
        uint32_t* sel = (uint32_t*)ensure(b_vsel, (size_t)ndraw * 4);
        long long* nsel = (long long*)ensure(b_tmp, 64);
        size_t tb = 0;
        GLB_CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, tb, val, acc, sel, nsel, (long long)ndraw, s));
        DevBuf scratch;
        void* tmp = ensure(scratch, tb);
        cudaError_t e = cub::DeviceSelect::Flagged(tmp, tb, val, acc, sel, nsel, (long long)ndraw, s);
        GLB_CUDA_TRY(cudaStreamSynchronize(s));
        free_buf(scratch);
        GLB_CUDA_TRY(e);
        wdraw = sel;
        break;
      }
    }
    // ---- stable grouping by source (CsrGraph.from_edges, csr.py:111-116)
    uint32_t* keys2 = (uint32_t*)ensure(b_keys2, mb * 4);
    uint32_t* idx2 = (uint32_t*)ensure(b_idx2, mb * 4);
    if (m) {
      size_t tb = 0;
      GLB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, src, keys2, idx, idx2, (long long)m, 0,
                                                   scale, s));
      DevBuf scratch;
      void* tmp = ensure(scratch, tb);
      cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tb, src, keys2, idx, idx2, (long long)m, 0,
                                                      scale, s);
      GLB_CUDA_TRY(cudaStreamSynchronize(s));
      free_buf(scratch);
      GLB_CUDA_TRY(e);
    }
    g->row = (long long*)dmalloc((size_t)(n + 1) * 8);
    g->col = (uint32_t*)dmalloc(mb * 4 + kEdgePad);
    if (weighted) g->wt = (uint32_t*)dmalloc(mb * 4 + kEdgePad);
    // row offsets: counts per source, exclusive scan
    unsigned long long* cnt = (unsigned long long*)ensure(b_tmp, (size_t)(n + 1) * 8);
    GLB_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)(n + 1) * 8, s));
    if (m) {
      k_count_src<<<grid_for((long long)m, kBlock, g->num_sms * 8), kBlock, 0, s>>>(keys2, m, cnt);
      GLB_CHECK_LAUNCH();
    }
    {
      unsigned long long* scanned = (unsigned long long*)ensure(b_src, (size_t)(n + 1) * 8);
      size_t tb = 0;
      GLB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, scanned, n + 1, s));
      DevBuf scratch;
      void* tmp = ensure(scratch, tb);
      cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, scanned, n + 1, s);
      GLB_CUDA_TRY(cudaStreamSynchronize(s));
      free_buf(scratch);
      GLB_CUDA_TRY(e);
      k_i64_from_u64<<<grid_for(n + 1, kBlock, g->num_sms * 8), kBlock, 0, s>>>(scanned, g->row, n + 1);
      GLB_CHECK_LAUNCH();
    }
    if (m) {
      k_gather_edges<<<grid_for((long long)m, kBlock, g->num_sms * 8), kBlock, 0, s>>>(
          idx2, dst, wdraw, m, g->col, weighted ? g->wt : nullptr);
      GLB_CHECK_LAUNCH();
    }
    GLB_CUDA_TRY(cudaStreamSynchronize(s));
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace glb
