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

  __device__ __forceinline__ static Vec<NW> run(Storage& st, const LookbackState<NW>& lb,
                                                 unsigned epoch, long long tile,
                                                 const Vec<NW>& thread_sum,
                                                 Vec<NW>& tile_incl) {
    Vec<NW> thread_ex, block_total;
    BlockScan(st.scan).ExclusiveScan(thread_sum, thread_ex, Vec<NW>(), VecSum(), block_total);
    if (threadIdx.x == 0) {
      Vec<NW> prefix;
      if (tile == 0) {
        st_vec_cg(lb.incls, block_total);
        __threadfence();
        atomicExch(lb.flags, (epoch << 2) | kTileIncl);
      } else {
        st_vec_cg(lb.aggs + tile, block_total);
        __threadfence();
        atomicExch(lb.flags + tile, (epoch << 2) | kTileAgg);
        long long p = tile - 1;
        while (true) {
          unsigned f;
          do {
            f = *((volatile unsigned int*)(lb.flags + p));
          } while ((f >> 2) != epoch);
          __threadfence();
          if ((f & 3u) == kTileIncl) {
            prefix = ld_vec_cg(lb.incls + p) + prefix;
            break;
          }
          prefix = ld_vec_cg(lb.aggs + p) + prefix;
          --p;
        }
        st_vec_cg(lb.incls + tile, prefix + block_total);
        __threadfence();
        atomicExch(lb.flags + tile, (epoch << 2) | kTileIncl);
      }
      st.prefix = prefix;
      st.incl = prefix + block_total;
    }
    __syncthreads();
    Vec<NW> r = st.prefix + thread_ex;
    tile_incl = st.incl;
    __syncthreads();  // Storage is reused by the next tile
    return r;
  }
};

}  // namespace glb
