// glb_relax.cuh -- the five task-distribution kernels for BFS/SSSP relaxation.
//
//   k_bs_relax   node-based (BS, node_based.py:43-67): one thread per worklist
//                node relaxes all its out-edges -- the imbalance is kept on
//                purpose; it is the baseline the other strategies beat.
//   k_ns_relax   node splitting (NS, splitting.py:141-162): BS over the split
//                graph + mirroring each improved parent onto its children.
//   k_ep_relax   edge-based (EP, edge_based.py:70-87): one thread per worklist
//                edge over the COO source array; a successful relax appends
//                the destination's whole out-edge range with ONE reservation
//                (work chunking), written cooperatively by the warp.
//   k_wd_scan +  workload decomposition (WD, workload.py:75-159): single-pass
//   k_wd_relax   look-back scan of the frontier's remaining degrees (compacting
//                away empty items and emitting the first item of every edge
//                tile), then equal edge tiles per CTA with an in-smem
//                segmented owner fill, lanes on consecutive edges.
//   k_hp_window  hierarchical processing (HP, hierarchical.py:95-120): window
//                [s*mdt, (s+1)*mdt) of every sublist node, dispatched at CTA /
//                warp / thread granularity by window length.
//
// Every kernel reads its worklist size from device memory (*nin) and strides
// over it, so the same kernels run under the host loop and the device-driven
// CUDA-graph loop.
#pragma once

#include <cub/block/block_scan.cuh>

#include "glb_internal.cuh"
#include "glb_scan.cuh"

namespace glb {

// --------------------------------------------------------- relax helper ---
template <typename D, bool W>
struct Relaxer {
  const uint32_t* __restrict__ col;
  const uint32_t* __restrict__ wt;
  D* dist;
  uint32_t* stamp;
  uint32_t gen;
  uint32_t* qout;
  unsigned int* nout;
  unsigned int* ovf;

  // Relax edge e out of a node at distance dn (dn != INF). Returns the
  // destination when its distance strictly decreased.
  __device__ __forceinline__ bool edge(long long e, D dn, ThreadCounters& c, uint32_t& v,
                                       D& cand) const {
    v = __ldcs(col + e);
    ++c.work;
    ++c.relax;
    if (!make_cand<D>(dn, W ? __ldcs(wt + e) : 1u, cand, ovf)) return false;
    return relax_min(dist, v, cand);
  }
  __device__ __forceinline__ void push(uint32_t v, ThreadCounters& c) const {
    if (claim(stamp, v, gen)) {
      q_append(qout, nout, v);
      ++c.push;
    }
  }
  __device__ __forceinline__ void edge_push(long long e, D dn, ThreadCounters& c) const {
    uint32_t v;
    D cand;
    if (edge(e, dn, c, v, cand)) push(v, c);
  }
};

// ============================================================ BS (K1) ===
template <typename D, bool W>
__global__ void __launch_bounds__(kBlock) k_bs_relax(const long long* __restrict__ row,
                                                     Relaxer<D, W> rx,
                                                     const uint32_t* __restrict__ qin,
                                                     const unsigned int* nin, LaunchStats* ls) {
  ThreadCounters c;
  const unsigned n = *nin;
  for (unsigned i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
    uint32_t u = qin[i];
    D du = rx.dist[u];
    if (du == DistTraits<D>::kInf) continue;
    long long lo = row[u], hi = row[u + 1];
    for (long long e = lo; e < hi; ++e) rx.edge_push(e, du, c);
  }
  flush_counters(ls, c);
}

// ============================================================ NS (K9) ===
// children of original node v: n_orig + cs[v] .. n_orig + cs[v+1]
template <typename D, bool W>
__global__ void __launch_bounds__(kBlock) k_ns_relax(const long long* __restrict__ row,
                                                     const long long* __restrict__ cs,
                                                     long long n_orig, Relaxer<D, W> rx,
                                                     const uint32_t* __restrict__ qin,
                                                     const unsigned int* nin, LaunchStats* ls) {
  ThreadCounters c;
  const unsigned n = *nin;
  for (unsigned i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
    uint32_t u = qin[i];
    D du = rx.dist[u];
    if (du == DistTraits<D>::kInf) continue;
    long long lo = row[u], hi = row[u + 1];
    for (long long e = lo; e < hi; ++e) {
      uint32_t v;
      D cand;
      if (!rx.edge(e, du, c, v, cand)) continue;
      rx.push(v, c);
      if (v < n_orig) {
        // reflect the parent's value onto its children (splitting.py:154-160)
        const long long k1 = cs[v + 1];
        for (long long k = cs[v]; k < k1; ++k) {
          uint32_t child = (uint32_t)(n_orig + k);
          ++c.relax;
          relax_min(rx.dist, child, cand);
          rx.push(child, c);
        }
      }
    }
  }
  flush_counters(ls, c);
}

// ============================================================ EP (K2) ===
template <typename D, bool W, bool CHUNKED>
__global__ void __launch_bounds__(kBlock) k_ep_relax(const long long* __restrict__ row,
                                                     const uint32_t* __restrict__ src,
                                                     Relaxer<D, W> rx,
                                                     const uint32_t* __restrict__ qin,
                                                     const unsigned int* nin, LaunchStats* ls) {
  ThreadCounters c;
  const unsigned n = *nin;
  const unsigned lane = lane_id();
  for (unsigned base = blockIdx.x * kBlock + (threadIdx.x & ~31u); base < n;
       base += gridDim.x * kBlock) {
    unsigned i = base + lane;
    long long plo = 0;
    unsigned pdeg = 0;
    if (i < n) {
      uint32_t e = qin[i];
      ++c.work;
      D du = rx.dist[__ldcs(src + e)];
      if (du != DistTraits<D>::kInf) {
        uint32_t v = __ldcs(rx.col + e);
        ++c.relax;
        D cand;
        if (make_cand<D>(du, W ? __ldcs(rx.wt + e) : 1u, cand, rx.ovf) &&
            relax_min(rx.dist, v, cand) && claim(rx.stamp, v, rx.gen)) {
          plo = row[v];
          pdeg = (unsigned)(row[v + 1] - plo);
        }
      }
    }
    unsigned slot = 0;
    if (CHUNKED && pdeg > 0) {  // one reservation for the whole range (worklist.py:84-104)
      slot = atomicAdd(rx.nout, pdeg);
      ++c.push;
    }
    unsigned ball = __ballot_sync(0xffffffffu, pdeg > 0);
    while (ball) {
      int leader = __ffs(ball) - 1;
      ball &= ball - 1;
      long long lo = __shfl_sync(0xffffffffu, plo, leader);
      unsigned dg = __shfl_sync(0xffffffffu, pdeg, leader);
      unsigned sl = __shfl_sync(0xffffffffu, slot, leader);
      for (unsigned k = lane; k < dg; k += 32) {
        unsigned s = sl + k;
        if (!CHUNKED) {
          s = atomicAdd(rx.nout, 1u);
          ++c.push;
        }
        rx.qout[s] = (uint32_t)(lo + k);
      }
    }
  }
  flush_counters(ls, c);
}

// ====================================================== WD (K4 + K5/K6) ===
constexpr int kWdIPT = 4;                    // frontier items per thread in the scan
constexpr int kWdScanTile = kBlock * kWdIPT;  // 1024 items per scan tile
constexpr int kWdEPT = 8;                    // edges per thread per relax tile
constexpr int kWdTile = kBlock * kWdEPT;     // 2048 edges per relax tile

// Remaining degree of every frontier item (minus the HP base offset
// min(window, deg), hierarchical.py:69-72), scanned as {edges, non-empty}.
// Non-empty items are compacted to j = exclusive count: c_pre[j] = first
// active edge, c_base[j] = CSR index of that edge minus c_pre[j], c_node[j].
// tile_first[b] = item holding active edge b*kWdTile.
__global__ void __launch_bounds__(kBlock) k_wd_scan(
    const long long* __restrict__ row, const uint32_t* __restrict__ q, const unsigned int* nin,
    long long window, LookbackState<2> lb, unsigned epoch, long long* __restrict__ c_pre,
    long long* __restrict__ c_base, uint32_t* __restrict__ c_node,
    unsigned int* __restrict__ tile_first, DevCtrl* ctrl) {
  using TS = TileScan<2, kBlock>;
  __shared__ typename TS::Storage st;
  const long long n = *nin;
  const long long ntiles = (n + kWdScanTile - 1) / kWdScanTile;
  if (ntiles == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    ctrl->wd_total = 0;
    ctrl->wd_items = 0;
  }
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    long long first = t * kWdScanTile + (long long)threadIdx.x * kWdIPT;
    uint32_t v[kWdIPT];
    long long beg[kWdIPT], rem[kWdIPT];
    Vec<2> sum;
#pragma unroll
    for (int k = 0; k < kWdIPT; ++k) {
      rem[k] = 0;
      if (first + k < n) {
        v[k] = q[first + k];
        long long lo = row[v[k]], hi = row[v[k] + 1];
        long long b = hi - lo < window ? hi - lo : window;
        beg[k] = lo + b;
        rem[k] = hi - lo - b;
      }
      sum.w[0] += rem[k];
      sum.w[1] += rem[k] > 0;
    }
    Vec<2> incl;
    Vec<2> ex = TS::run(st, lb, epoch, t, sum, incl);
#pragma unroll
    for (int k = 0; k < kWdIPT; ++k) {
      if (rem[k] > 0) {
        long long j = ex.w[1], pre = ex.w[0];
        c_pre[j] = pre;
        c_base[j] = beg[k] - pre;
        c_node[j] = v[k];
        for (long long b = (pre + kWdTile - 1) / kWdTile; b * kWdTile < pre + rem[k]; ++b)
          tile_first[b] = (unsigned)j;
        ex.w[0] += rem[k];
        ex.w[1] += 1;
      }
    }
    if (t == ntiles - 1 && threadIdx.x == 0) {
      ctrl->wd_total = incl.w[0];
      ctrl->wd_items = incl.w[1];
    }
  }
}

struct MaxOp {
  __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};

template <typename D, bool W>
__global__ void __launch_bounds__(kBlock) k_wd_relax(Relaxer<D, W> rx,
                                                     const long long* __restrict__ c_pre,
                                                     const long long* __restrict__ c_base,
                                                     const uint32_t* __restrict__ c_node,
                                                     const unsigned int* __restrict__ tile_first,
                                                     const DevCtrl* ctrl, LaunchStats* ls) {
  using BScan = cub::BlockScan<int, kBlock, cub::BLOCK_SCAN_WARP_SCANS>;
  __shared__ __align__(16) int s_own[kWdTile];
  __shared__ long long s_base[kWdTile + 1];
  __shared__ D s_dn[kWdTile + 1];
  __shared__ typename BScan::TempStorage s_scan;
  ThreadCounters c;
  const long long total = ctrl->wd_total;
  const long long nitems = ctrl->wd_items;
  const long long ntiles = (total + kWdTile - 1) / kWdTile;
  for (long long b = blockIdx.x; b < ntiles; b += gridDim.x) {
    const long long e0 = b * kWdTile;
    const long long e1 = e0 + kWdTile < total ? e0 + kWdTile : total;
    const long long j0 = tile_first[b];
    const long long j1 = b + 1 < ntiles ? (long long)tile_first[b + 1] : nitems - 1;
    const int cnt = (int)(j1 - j0 + 1);
    int4* own4 = reinterpret_cast<int4*>(s_own);
    for (int k = threadIdx.x; k < kWdTile / 4; k += kBlock) own4[k] = make_int4(0, 0, 0, 0);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += kBlock) {
      long long j = j0 + k;
      long long pre = c_pre[j];
      s_base[k] = c_base[j];
      s_dn[k] = rx.dist[c_node[j]];  // dn read when the node is entered (workload.py:131,140)
      long long h = pre - e0;
      if (h < 0) h = 0;
      if (h < kWdTile) s_own[h] = k;
    }
    __syncthreads();
    // carry each item head forward: inclusive max-scan over the tile
    int loc[kWdEPT];
    {
      const int4* p = reinterpret_cast<const int4*>(s_own + threadIdx.x * kWdEPT);
      int4 a = p[0], bb = p[1];
      loc[0] = a.x; loc[1] = a.y; loc[2] = a.z; loc[3] = a.w;
      loc[4] = bb.x; loc[5] = bb.y; loc[6] = bb.z; loc[7] = bb.w;
    }
    int tmax = 0;
#pragma unroll
    for (int k = 0; k < kWdEPT; ++k) {
      tmax = loc[k] > tmax ? loc[k] : tmax;
      loc[k] = tmax;
    }
    int carry;
    BScan(s_scan).ExclusiveScan(tmax, carry, 0, MaxOp());
    __syncthreads();
    {
      int4* p = reinterpret_cast<int4*>(s_own + threadIdx.x * kWdEPT);
#pragma unroll
      for (int k = 0; k < kWdEPT; ++k) loc[k] = loc[k] > carry ? loc[k] : carry;
      p[0] = make_int4(loc[0], loc[1], loc[2], loc[3]);
      p[1] = make_int4(loc[4], loc[5], loc[6], loc[7]);
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kWdEPT; ++k) {
      int local = k * kBlock + threadIdx.x;
      long long e = e0 + local;
      if (e < e1) {
        int o = s_own[local];
        D dn = s_dn[o];
        if (dn != DistTraits<D>::kInf) {
          rx.edge_push(s_base[o] + e, dn, c);
        } else {
          ++c.work;
        }
      }
    }
    __syncthreads();
  }
  flush_counters(ls, c);
}

// ============================================================ HP (K10) ===
constexpr long long kHpCtaThreshold = 1024;  // window length handled by a whole CTA
constexpr long long kHpWarpThreshold = 32;   // ... by a warp; shorter: one thread

template <typename D, bool W>
__global__ void __launch_bounds__(kBlock) k_hp_window(const long long* __restrict__ row,
                                                      Relaxer<D, W> rx,
                                                      const uint32_t* __restrict__ qin,
                                                      const unsigned int* nin, long long window,
                                                      long long mdt, uint32_t* qnext,
                                                      unsigned int* nnext, LaunchStats* ls) {
  __shared__ long long s_lo, s_hi;
  __shared__ D s_dn;
  __shared__ int s_owner;
  ThreadCounters c;
  const long long n = *nin;
  for (long long base = blockIdx.x * (long long)kBlock; base < n;
       base += (long long)gridDim.x * kBlock) {
    long long i = base + threadIdx.x;
    long long lo = 0, hi = 0;
    D dn = DistTraits<D>::kInf;
    if (i < n) {
      uint32_t u = qin[i];
      long long r0 = row[u], r1 = row[u + 1];
      long long start = r0 + window;
      if (start < r1) {
        long long end = start + mdt < r1 ? start + mdt : r1;
        dn = rx.dist[u];
        if (dn != DistTraits<D>::kInf) {
          lo = start;
          hi = end;
        }
        if (end < r1) {  // unfinished: carry into the next sublist
          q_append(qnext, nnext, u);
          ++c.push;
        }
      }
    }
    // CTA granularity
    while (true) {
      if (threadIdx.x == 0) s_owner = -1;
      __syncthreads();
      if (hi - lo >= kHpCtaThreshold) s_owner = threadIdx.x;
      __syncthreads();
      const int o = s_owner;
      if (o < 0) break;
      if (threadIdx.x == o) {
        s_lo = lo;
        s_hi = hi;
        s_dn = dn;
        lo = hi;
      }
      __syncthreads();
      const long long clo = s_lo, chi = s_hi;
      const D cdn = s_dn;
      for (long long e = clo + threadIdx.x; e < chi; e += kBlock) rx.edge_push(e, cdn, c);
      __syncthreads();
    }
    // warp granularity
    unsigned ball;
    while ((ball = __ballot_sync(0xffffffffu, hi - lo >= kHpWarpThreshold)) != 0) {
      const int leader = __ffs(ball) - 1;
      const long long wlo = __shfl_sync(0xffffffffu, lo, leader);
      const long long whi = __shfl_sync(0xffffffffu, hi, leader);
      const D wdn = __shfl_sync(0xffffffffu, dn, leader);
      if ((int)lane_id() == leader) lo = hi;
      for (long long e = wlo + lane_id(); e < whi; e += 32) rx.edge_push(e, wdn, c);
    }
    // thread granularity
    for (long long e = lo; e < hi; ++e) rx.edge_push(e, dn, c);
  }
  flush_counters(ls, c);
}

// ============================================================ setup ===
template <typename D>
__global__ void k_init_dist(D* dist, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dist[i] = DistTraits<D>::kInf;
}

// Seed the first worklist: the source (+ its NS children at distance 0,
// splitting.py:123-126) for node worklists, or the source's out-edge range for
// the EP edge worklist (edge_based.py:55).
template <typename D>
__global__ void k_seed(D* dist, uint32_t* q, unsigned int* nq, long long src, long long kid_lo,
                       long long kid_hi, long long edge_lo, long long edge_hi, bool edges) {
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  if (tid == 0) dist[src] = 0;
  if (edges) {
    for (long long e = edge_lo + tid; e < edge_hi; e += stride) q[e - edge_lo] = (uint32_t)e;
    if (tid == 0) *nq = (unsigned)(edge_hi - edge_lo);
  } else {
    if (tid == 0) q[0] = (uint32_t)src;
    for (long long k = kid_lo + tid; k < kid_hi; k += stride) {
      dist[k] = 0;
      q[1 + k - kid_lo] = (uint32_t)k;
    }
    if (tid == 0) *nq = (unsigned)(1 + kid_hi - kid_lo);
  }
}

template <typename D>
__global__ void k_dist_out(const D* __restrict__ dist, long long n, long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    D d = dist[i];
    out[i] = d == DistTraits<D>::kInf ? 0x7FFFFFFFFFFFFFFFll : (long long)d;
  }
}

}  // namespace glb
