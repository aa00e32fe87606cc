// glb_scan.cuh -- single-pass decoupled look-back prefix scan over int64
// vectors.  Replaces the block-structured host scan of scan.py:19-65 (4096-item
// blocks + carry pass) with one kernel pass: each CTA scans a tile with
// cub::BlockScan, publishes its aggregate, and looks back over predecessor
// tiles for its carry.  Tile flags carry an epoch so no reset pass is needed
// between invocations.
#pragma once

#include <cub/block/block_scan.cuh>

#include "glb_internal.cuh"

namespace glb {

// Vector of NW int64 lanes, added lane-wise (edges, items, ...).
template <int NW>
struct Vec {
  long long w[NW];
  __host__ __device__ __forceinline__ Vec() {
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = 0;
  }
  __host__ __device__ __forceinline__ Vec operator+(const Vec& o) const {
    Vec r;
#pragma unroll
    for (int i = 0; i < NW; ++i) r.w[i] = w[i] + o.w[i];
    return r;
  }
};

struct VecSum {
  template <typename T>
  __device__ __forceinline__ T operator()(const T& a, const T& b) const {
    return a + b;
  }
};

enum : unsigned { kTileAgg = 1u, kTileIncl = 2u };

template <int NW>
__device__ __forceinline__ void st_vec_cg(Vec<NW>* p, const Vec<NW>& v) {
#pragma unroll
  for (int i = 0; i < NW; ++i) __stcg(&p->w[i], v.w[i]);
}
template <int NW>
__device__ __forceinline__ Vec<NW> ld_vec_cg(const Vec<NW>* p) {
  Vec<NW> v;
#pragma unroll
  for (int i = 0; i < NW; ++i) v.w[i] = __ldcg(&p->w[i]);
  return v;
}

// Look-back storage: flags[t] = epoch << 2 | state; aggs / incls per tile.
template <int NW>
struct LookbackState {
  unsigned int* flags;
  Vec<NW>* aggs;
  Vec<NW>* incls;
};

// Scan of one tile held as per-thread partials.  `thread_sum` is the sum of the
// calling thread's items; returns the exclusive prefix of that thread's first
// item across the whole sequence, and (via tile_incl) the inclusive total
// through this tile.  All threads of the CTA must call it.
//
// Forward progress: tiles are visited as blockIdx.x + k*gridDim.x and the grid
// never exceeds the number of co-resident CTAs, so every predecessor tile is
// owned by a running CTA.
template <int NW, int BLOCK>
struct TileScan {
  using BlockScan = cub::BlockScan<Vec<NW>, BLOCK, cub::BLOCK_SCAN_WARP_SCANS>;
  struct Storage {
    typename BlockScan::TempStorage scan;
    Vec<NW> prefix;
    Vec<NW> incl;
  };

  __device__ __forceinline__ static Vec<NW> warp_sum(Vec<NW> v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int i = 0; i < NW; ++i) v.w[i] += __shfl_xor_sync(0xffffffffu, v.w[i], off);
    return v;
  }

  __device__ __forceinline__ static Vec<NW> run(Storage& st, const LookbackState<NW>& lb,
                                                 unsigned epoch, long long tile,
                                                 const Vec<NW>& thread_sum,
                                                 Vec<NW>& tile_incl) {
    Vec<NW> thread_ex, block_total;
    BlockScan(st.scan).ExclusiveScan(thread_sum, thread_ex, Vec<NW>(), VecSum(), block_total);
    if (threadIdx.x < 32) {
      const unsigned lane = threadIdx.x;
      Vec<NW> prefix;
      if (tile == 0) {
        if (lane == 0) {
          st_vec_cg(lb.incls, block_total);
          __threadfence();
          atomicExch(lb.flags, (epoch << 2) | kTileIncl);
        }
      } else {
        if (lane == 0) {
          st_vec_cg(lb.aggs + tile, block_total);
          __threadfence();
          atomicExch(lb.flags + tile, (epoch << 2) | kTileAgg);
        }
        // warp-parallel look-back: lane l inspects predecessor p - l
        long long p = tile - 1;
        while (true) {
          const long long q = p - (long long)lane;
          unsigned f = (epoch << 2) | kTileIncl;  // q < 0: virtual inclusive zero
          if (q >= 0) {
            do {
              f = *((volatile unsigned int*)(lb.flags + q));
            } while ((f >> 2) != epoch);
          }
          __threadfence();
          const unsigned incl_mask = __ballot_sync(0xffffffffu, (f & 3u) == kTileIncl);
          const int stop = incl_mask ? __ffs(incl_mask) - 1 : 32;
          Vec<NW> val;
          if ((int)lane < stop)
            val = ld_vec_cg(lb.aggs + q);
          else if ((int)lane == stop && q >= 0)
            val = ld_vec_cg(lb.incls + q);
          prefix = prefix + warp_sum(val);
          if (incl_mask) break;
          p -= 32;
        }
        if (lane == 0) {
          st_vec_cg(lb.incls + tile, prefix + block_total);
          __threadfence();
          atomicExch(lb.flags + tile, (epoch << 2) | kTileIncl);
        }
      }
      if (lane == 0) {
        st.prefix = prefix;
        st.incl = prefix + block_total;
      }
    }
    __syncthreads();
    Vec<NW> r = st.prefix + thread_ex;
    tile_incl = st.incl;
    __syncthreads();  // Storage is reused by the next tile
    return r;
  }
};

}  // namespace glb
