// glb_tiles.cuh -- edge tiles over CSR: CTA b owns edges [b*kEdgeTile,
// (b+1)*kEdgeTile) and finds each edge's source node with a segmented "head"
// fill + max-scan in shared memory.  Used by the COO expansion (csr.py:168)
// and the node-split scatter (splitting.py:72-99); the same idea drives the
// WD relax tiles over the frontier.
#pragma once

#include <cub/block/block_scan.cuh>

#include "glb_internal.cuh"

namespace glb {

constexpr int kEdgeEPT = 8;
constexpr int kEdgeTile = kBlock * kEdgeEPT;  // 2048 edges per tile

// tile_node[b] = node holding edge b*kEdgeTile (every boundary written once).
__global__ void k_tile_nodes(const long long* __restrict__ row, long long n,
                             unsigned int* __restrict__ tile_node) {
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const long long lo = row[v], hi = row[v + 1];
    for (long long b = (lo + kEdgeTile - 1) / kEdgeTile; b * kEdgeTile < hi; ++b)
      tile_node[b] = (unsigned)v;
  }
}

struct HeadMax {
  __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};

// For the tile [e0, e1) whose edges belong to nodes v0..v1: calls
// store(v, h) for every non-empty node with its head position h (first edge
// of the node inside the tile), then leaves s_head[i] = head position of the
// node owning edge e0 + i.  All threads of the CTA must call it.
template <typename Store>
__device__ __forceinline__ void tile_heads(const long long* __restrict__ row, long long v0,
                                           long long v1, long long e0, long long e1, int* s_head,
                                           typename cub::BlockScan<int, kBlock>::TempStorage& ts,
                                           Store&& store) {
  int4* h4 = reinterpret_cast<int4*>(s_head);
  for (int k = threadIdx.x; k < kEdgeTile / 4; k += kBlock) h4[k] = make_int4(0, 0, 0, 0);
  __syncthreads();
  for (long long v = v0 + threadIdx.x; v <= v1; v += kBlock) {
    const long long lo = row[v], hi = row[v + 1];
    if (hi > lo && lo < e1) {
      const int h = (int)((lo > e0 ? lo : e0) - e0);
      s_head[h] = h;
      store(v, h);
    }
  }
  __syncthreads();
  int loc[kEdgeEPT];
  const int4* p = reinterpret_cast<const int4*>(s_head + threadIdx.x * kEdgeEPT);
  const int4 a = p[0], b = p[1];
  loc[0] = a.x; loc[1] = a.y; loc[2] = a.z; loc[3] = a.w;
  loc[4] = b.x; loc[5] = b.y; loc[6] = b.z; loc[7] = b.w;
  int run = 0;
#pragma unroll
  for (int k = 0; k < kEdgeEPT; ++k) {
    run = loc[k] > run ? loc[k] : run;
    loc[k] = run;
  }
  int carry;
  cub::BlockScan<int, kBlock>(ts).ExclusiveScan(run, carry, 0, HeadMax());
  __syncthreads();
  int4* q = reinterpret_cast<int4*>(s_head + threadIdx.x * kEdgeEPT);
#pragma unroll
  for (int k = 0; k < kEdgeEPT; ++k) loc[k] = loc[k] > carry ? loc[k] : carry;
  q[0] = make_int4(loc[0], loc[1], loc[2], loc[3]);
  q[1] = make_int4(loc[4], loc[5], loc[6], loc[7]);
  __syncthreads();
}

}  // namespace glb
