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
//                (work chunking), the ranges written cooperatively by warps.
//   k_wd_scan +  workload decomposition (WD, workload.py:75-159): single-pass
//   k_wd_relax   look-back scan of the frontier's remaining degrees (compacting
//                away empty items and emitting the first item of every edge
//                tile), then equal edge tiles per CTA with an in-smem
//                segmented owner fill, lanes on consecutive edges.
//   k_hp_window  hierarchical processing (HP, hierarchical.py:95-120): window
//                [s*mdt, (s+1)*mdt) of every sublist node, dispatched at CTA /
//                warp / thread granularity by window length.
//
// Every relaxation goes through relax_batch<K>: K independent edges per
// thread are gathered first (col/weight loads), then their dist[dst] loads,
// then the atomicMin / stamp claims, so a thread keeps K loads in flight
// instead of one dependent chain.  Improved destinations go to a per-CTA
// shared-memory queue flushed with ONE global reservation per CTA round --
// the worklist cursor of worklist.py:107-130 without a global hot spot.
//
// Every kernel reads its worklist size from device memory (*nin) and strides
// over it, so the same kernels run under the host loop and the device-driven
// CUDA-graph loop.
#pragma once

#include <cub/block/block_scan.cuh>

#include "glb_control.cuh"
#include "glb_internal.cuh"
#include "glb_scan.cuh"

#ifndef GLB_PRECHECK
#define GLB_PRECHECK 1  // plain-load filter before the relaxation atomic
#endif
#ifndef GLB_RELAX_MINB
#define GLB_RELAX_MINB 3  // CTAs per SM the HP window kernel is register-capped for
#endif
#ifndef GLB_CELL_POLICY
#define GLB_CELL_POLICY 1  // evict-last L2 hint on the cell gathers (C2: -3 % WD, -4 % HP)
#endif
#ifndef GLB_RELAX_BRANCHLESS
#define GLB_RELAX_BRANCHLESS 1  // relax_vals without divergent regions (C2 SSSP HP 4.49 -> 3.93 ms, NS 6.23 -> 5.87)
#endif
#ifndef GLB_WD_BRANCHLESS
#define GLB_WD_BRANCHLESS 1  // WD relax stages without divergent regions (C2 SSSP WD -5 %, BFS -8 %)
#endif
#ifndef GLB_WD_MINB
#define GLB_WD_MINB 2  // the pipelined WD relax: 2 CTAs/SM without spills beat 3 with (C2 A/B)
#endif

namespace glb {

// ------------------------------------------------------- CTA push queue ---
constexpr int kQCap = 2048;
struct BlockQ {          // control words; the items live in a separate smem array
  uint32_t* items;       // kQCap entries
  uint32_t* bm;          // BS: the out list's member bitmap (null: none)
  unsigned int count;
  unsigned int base;
};

__device__ __forceinline__ void bm_set(uint32_t* bm, uint32_t v) {
  atomicOr(bm + (v >> 5), 1u << (v & 31u));
}

__device__ __forceinline__ void bq_init(BlockQ& q, uint32_t* items, uint32_t* bm = nullptr) {
  if (threadIdx.x == 0) {
    q.items = items;
    q.bm = bm;
    q.count = 0;
  }
  __syncthreads();
}

// Warp-aggregated slot reservation in the CTA queue; overflow goes straight
// to the global worklist.
__device__ __forceinline__ void bq_push(BlockQ& q, uint32_t* qout, unsigned int* nout,
                                        uint32_t v) {
  const unsigned mask = __activemask();
  const unsigned leader = __ffs(mask) - 1;
  const unsigned rank = __popc(mask & ((1u << lane_id()) - 1u));
  unsigned base = 0;
  if (lane_id() == leader) base = atomicAdd(&q.count, (unsigned)__popc(mask));
  base = __shfl_sync(mask, base, leader) + rank;
  if (base < (unsigned)kQCap) {
    q.items[base] = v;
  } else {
    qout[atomicAdd(nout, 1u)] = v;
    if (q.bm) bm_set(q.bm, v);
  }
}

// All threads of the CTA: one global reservation, coalesced copy-out.
__device__ __forceinline__ void bq_flush(BlockQ& q, uint32_t* qout, unsigned int* nout) {
  __syncthreads();
  const unsigned n = q.count < (unsigned)kQCap ? q.count : (unsigned)kQCap;
  if (threadIdx.x == 0) q.base = n ? atomicAdd(nout, n) : 0u;
  __syncthreads();
  const unsigned b = q.base;
  const uint32_t* items = q.items;
  uint32_t* bm = q.bm;
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t v = items[i];
    qout[b + i] = v;
    if (bm) bm_set(bm, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) q.count = 0;
  __syncthreads();
}

// warp shuffle of a distance value (32- or 64-bit)
__device__ __forceinline__ uint32_t shfl_dist(uint32_t d, int src) {
  return __shfl_sync(0xffffffffu, d, src);
}
__device__ __forceinline__ unsigned long long shfl_dist(unsigned long long d, int src) {
  return __shfl_sync(0xffffffffu, d, src);
}
__device__ __forceinline__ dist24_t shfl_dist(dist24_t d, int src) {
  return (dist24_t)__shfl_sync(0xffffffffu, (uint32_t)d, src);
}

// cell gather with an L2 cache-hint policy (32- or 64-bit cells)
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* p, unsigned long long pol) {
  uint32_t r;
  asm("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ unsigned long long ld_keep(const unsigned long long* p,
                                                      unsigned long long pol) {
  unsigned long long r;
  asm("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
  return r;
}

// --------------------------------------------------------- relax helper ---
template <typename D, bool W>
struct Relaxer {
  const uint32_t* __restrict__ col;
  const uint32_t* __restrict__ wt;
  CellS<D>* cells;            // Cell<D> distance cells
  uint32_t* stamp;            // push dedup for unpacked (64-bit) cells
  uint32_t gen;
  uint32_t* qout;
  unsigned int* nout;
  unsigned int* ovf;
  unsigned long long keep;    // L2 evict-last policy for the cells (GLB_CELL_POLICY)

  __device__ __forceinline__ D dist(uint32_t u) const {
#if GLB_CELL_POLICY
    return Cell<D>::dist(ld_keep(cells + u, keep));
#else
    return Cell<D>::dist(cells[u]);
#endif
  }
  // push claim after a strict decrease (first = packed-cell verdict)
  __device__ __forceinline__ bool claim_push(uint32_t v, bool first) const {
    if (Cell<D>::kPacked) return first;
    return claim(stamp, v, gen);
  }
};

// Bind the per-step fields (out list, its cursor, stamp generation) from the
// control block written by k_control.
template <typename D, bool W>
__device__ __forceinline__ Relaxer<D, W> bind(Relaxer<D, W> rx, DevCtrl* ctrl) {
  rx.gen = ctrl->gen;
  rx.qout = ctrl->qptr[ctrl->out];
  rx.nout = &ctrl->qcount[ctrl->out];
#if GLB_CELL_POLICY
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(rx.keep));
#endif
  return rx;
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void timer_begin(StepTimer& t) {
  if (threadIdx.x == 0) atomicMin(&t.start, gtime());
}
__device__ __forceinline__ void timer_end(StepTimer& t) {
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&t.end, gtime());
}

// Push sinks of improved destinations.  CtaSink: the CTA queue (any thread,
// divergent callers allowed; flushed by bq_flush at CTA barriers).
struct CtaSink {
  BlockQ& bq;
  uint32_t* qout;
  unsigned int* nout;
  template <int K>
  __device__ __forceinline__ void push(unsigned first, const uint32_t (&v)[K], ThreadCounters& c) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (first >> k & 1u) {
        bq_push(bq, qout, nout, v[k]);
        ++c.push;
      }
  }
};

// Relax up to K loaded edges (bit k of `valid`: edge to v[k] of weight w[k]
// out of a node at distance dn[k] != INF).  Returns the mask of edges whose
// atomicMin strictly lowered dist[v[k]] to cand[k] (atomic_relax_min,
// engine.py:120-139); the ones that also won the push claim go to the sink.
// All dist gathers are issued before any atomic, so a thread keeps K loads in
// flight.
template <int K, typename D, bool W, class S>
__device__ __forceinline__ unsigned relax_vals(const Relaxer<D, W>& rx, S& sink,
                                               const uint32_t (&v)[K], const uint32_t (&w)[K],
                                               const D (&dn)[K], unsigned valid, ThreadCounters& c,
                                               D (&cand)[K]) {
  unsigned want = 0;
#if GLB_PRECHECK && GLB_RELAX_BRANCHLESS
  // callers leave v[k] = 0 (a node id) in invalid slots: gathers and the
  // candidate test run without divergent regions
  D cur[K];
#pragma unroll
  for (int k = 0; k < K; ++k) cur[k] = rx.dist(v[k]);
  c.work += __popc(valid);
  c.relax += __popc(valid);
  bool ovf = false;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const unsigned long long c64 = (unsigned long long)dn[k] + (unsigned long long)w[k];
    const bool big = c64 >= (unsigned long long)DistTraits<D>::kInf;
    cand[k] = (D)c64;
    const bool vk = (valid >> k & 1u) != 0;
    ovf |= vk && big;
    want |= (unsigned)(vk && !big && cand[k] < cur[k]) << k;
  }
  if (ovf) atomicOr(rx.ovf, 1u);
#elif GLB_PRECHECK
  D cur[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (valid >> k & 1u) cur[k] = rx.dist(v[k]);
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (valid >> k & 1u) {
      ++c.work;
      ++c.relax;
      if (make_cand<D>(dn[k], w[k], cand[k], rx.ovf) && cand[k] < cur[k]) want |= 1u << k;
    }
#else
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (valid >> k & 1u) {
      ++c.work;
      ++c.relax;
      if (make_cand<D>(dn[k], w[k], cand[k], rx.ovf)) want |= 1u << k;
    }
#endif
  CellS<D> old[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (want >> k & 1u) old[k] = atomicMin(rx.cells + v[k], Cell<D>::make(cand[k], rx.gen));
  unsigned won = 0, first = 0;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if ((want >> k & 1u) && cand[k] < Cell<D>::dist(old[k])) {
      won |= 1u << k;
      if (Cell<D>::gen(old[k]) != Cell<D>::tag(rx.gen)) first |= 1u << k;
    }
  if (!Cell<D>::kPacked) {
    unsigned prev[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (won >> k & 1u) prev[k] = atomicExch(rx.stamp + v[k], rx.gen);
    first = 0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((won >> k & 1u) && prev[k] != rx.gen) first |= 1u << k;
  }
  sink.template push<K>(first, v, c);
  return won;
}

template <int K, typename D, bool W>
__device__ __forceinline__ unsigned relax_vals(const Relaxer<D, W>& rx, BlockQ& bq,
                                               const uint32_t (&v)[K], const uint32_t (&w)[K],
                                               const D (&dn)[K], unsigned valid, ThreadCounters& c,
                                               D (&cand)[K]) {
  CtaSink sink{bq, rx.qout, rx.nout};
  return relax_vals<K>(rx, sink, v, w, dn, valid, c, cand);
}

// Relax up to K edges e[k] (col / weight loads, then relax_vals).
// STREAM: the K edges of a batch are lanes-consecutive across the warp, so
// every col / weight line is consumed by one load instruction and can be
// fetched evict-first; thread-serial walks (BS, NS) reuse a line over several
// batches and keep the default policy.
template <int K, bool STREAM = true, typename D, bool W>
__device__ __forceinline__ unsigned relax_batch(const Relaxer<D, W>& rx, BlockQ& bq,
                                                const long long (&e)[K], const D (&dn)[K],
                                                unsigned valid, ThreadCounters& c,
                                                uint32_t (&v)[K], D (&cand)[K]) {
  uint32_t w[K];
  const unsigned long long pol = STREAM ? l2_evict_first() : 0ull;
#if GLB_RELAX_BRANCHLESS
  if (STREAM) {  // lane-consecutive batches: invalid slots load edge 0 (always mapped)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const long long ek = (valid >> k & 1u) ? e[k] : 0ll;
      v[k] = ld_stream_pol(rx.col + ek, pol);
      w[k] = W ? ld_stream_pol(rx.wt + ek, pol) : 1u;
    }
  } else {  // thread-serial walks (BS): skip the tail slots (measured: C2 SSSP BS +8 % otherwise)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      v[k] = 0;
      w[k] = 1u;
      if (valid >> k & 1u) {
        v[k] = __ldg(rx.col + e[k]);
        if (W) w[k] = __ldg(rx.wt + e[k]);
      }
    }
  }
#else
#pragma unroll
  for (int k = 0; k < K; ++k) {
    v[k] = 0;
    w[k] = 1u;
    if (valid >> k & 1u) {
      v[k] = STREAM ? ld_stream_pol(rx.col + e[k], pol) : __ldg(rx.col + e[k]);
      if (W) w[k] = STREAM ? ld_stream_pol(rx.wt + e[k], pol) : __ldg(rx.wt + e[k]);
    }
  }
#endif
  return relax_vals<K>(rx, bq, v, w, dn, valid, c, cand);
}

// Serial walk over [lo, hi) by one thread in batches of K.
template <int K, typename D, bool W>
__device__ __forceinline__ void relax_range_thread(const Relaxer<D, W>& rx, BlockQ& bq,
                                                   long long lo, long long hi, D dn,
                                                   ThreadCounters& c) {
  for (long long b = lo; b < hi; b += K) {
    long long e[K];
    D d[K];
    unsigned valid = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      e[k] = b + k;
      d[k] = dn;
      if (b + k < hi) valid |= 1u << k;
    }
    uint32_t v[K];
    D cand[K];
    relax_batch<K, false>(rx, bq, e, d, valid, c, v, cand);
  }
}

// Cooperative walk over [lo, hi) by `width` threads (rank r), K per thread.
template <int K, typename D, bool W>
__device__ __forceinline__ void relax_range_coop(const Relaxer<D, W>& rx, BlockQ& bq,
                                                 long long lo, long long hi, D dn, int r,
                                                 int width, ThreadCounters& c) {
  for (long long b = lo; b < hi; b += (long long)K * width) {
    long long e[K];
    D d[K];
    unsigned valid = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      e[k] = b + (long long)k * width + r;
      d[k] = dn;
      if (e[k] < hi) valid |= 1u << k;
    }
    uint32_t v[K];
    D cand[K];
    relax_batch<K>(rx, bq, e, d, valid, c, v, cand);
  }
}

// ============================================================ BS (K1) ===
template <typename D, bool W>
__global__ void __launch_bounds__(kBlock) k_bs_relax(const long long* __restrict__ row,
                                                     Relaxer<D, W> rx0, DevCtrl* ctrl,
                                                     CtlTail tail) {
  __shared__ uint32_t s_q[kQCap];
  __shared__ BlockQ bq;
  const unsigned n = ctrl->qcount[ctrl->in];
  // id-ordered frontiers: a list k_bm_compact did not rebuild clears its
  // members' bitmap words here (this step sets bits in the other bitmap)
  const unsigned bm_thr = ctrl->bm_thr;
  const bool bm_in = bm_thr && ctrl->bm_valid[ctrl->in];
  uint32_t* bm_clear = bm_in && n < bm_thr ? ctrl->bm[ctrl->in] : nullptr;
  if (bm_thr && blockIdx.x == 0 && threadIdx.x == 0) {
    if (bm_in && n >= bm_thr && ctrl->bm_ctr != n) ctrl->bm_err = 1;
    ctrl->bm_ctr = 0;  // k_bm_compact of the next step starts from 0
    ctrl->bm_valid[ctrl->out] = 1;  // this step sets the out list's bits
  }
  if (blockIdx.x * kBlock >= n) {  // idle CTA: no barriers, no atomics
    ctl_tail(tail, ctrl);
    return;
  }
  timer_begin(ctrl->t_relax);
  bq_init(bq, s_q, bm_thr ? ctrl->bm[ctrl->out] : nullptr);
  const Relaxer<D, W> rx = bind(rx0, ctrl);
  const uint32_t* __restrict__ qin = ctrl->qptr[ctrl->in];
  ThreadCounters c;
  for (unsigned base = blockIdx.x * kBlock; base < n; base += gridDim.x * kBlock) {
    const unsigned i = base + threadIdx.x;
    if (i < n) {
      const uint32_t u = qin[i];
      if (bm_clear) bm_clear[u >> 5] = 0u;
      const D du = rx.dist(u);
      if (du != DistTraits<D>::kInf) relax_range_thread<4>(rx, bq, row[u], row[u + 1], du, c);
    }
    bq_flush(bq, rx.qout, rx.nout);
  }
  flush_counters(ctrl, c);
  timer_end(ctrl->t_relax);
  ctl_tail(tail, ctrl);
}

// BS id-ordered frontier: rebuild the in-list from its member bitmap when it
// holds >= bm_thr nodes (the same set and length; node_based.py:43-67 takes
// the worklist in any order).  Each CTA turns 256 consecutive bitmap words
// into ids with one CTA scan, stages them in shared memory and copies them
// out coalesced behind one global reservation, so the list is in id order
// inside every 8K-node chunk; the words are zeroed as
// they are read.  Pushes arrive in warp/CTA-queue order, which on a
// low-degree graph (C3) scatters a lane's row / column / weight / cell
// accesses over separate sectors; in id order they share them.
constexpr int kBmBlock = 256;
__global__ void __launch_bounds__(kBmBlock) k_bm_compact(DevCtrl* ctrl, long long nwords) {
  const unsigned n = ctrl->qcount[ctrl->in];
  // below the threshold the relax kernel clears the words instead; a list
  // the cluster loop produced has no bits (it is taken in push order)
  if (n < ctrl->bm_thr || !ctrl->bm_valid[ctrl->in]) return;
  using Scan = cub::BlockScan<unsigned, kBmBlock>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ uint32_t s_ids[kBmBlock * 32];  // the chunk's ids, copied out coalesced
  __shared__ unsigned s_base;
  uint32_t* __restrict__ bm = ctrl->bm[ctrl->in];
  uint32_t* __restrict__ q = ctrl->qptr[ctrl->in];
  for (long long b = (long long)blockIdx.x * kBmBlock; b < nwords; b += (long long)gridDim.x * kBmBlock) {
    const long long i = b + threadIdx.x;
    const uint32_t w = i < nwords ? bm[i] : 0u;
    unsigned ex, total;
    Scan(ts).ExclusiveSum((unsigned)__popc(w), ex, total);
    if (total) {  // CTA-uniform
      if (threadIdx.x == 0) s_base = atomicAdd(&ctrl->bm_ctr, total);
      const uint32_t id0 = (uint32_t)(i * 32);
      for (uint32_t x = w; x; x &= x - 1u) s_ids[ex++] = id0 + (uint32_t)(__ffs(x) - 1);
      if (w) bm[i] = 0u;
      __syncthreads();
      const unsigned base = s_base;
      for (unsigned j = threadIdx.x; j < total; j += kBmBlock) q[base + j] = s_ids[j];
    }
    __syncthreads();  // scan storage / s_ids / s_base reuse
  }
}

// HP id-ordered super-lists: the list a window sub-iteration 0 reads is
// exactly {v : cell tag == the super-iteration's generation} (every push of a
// super-iteration carries its generation), so a frontier holding >= N/8 nodes
// is rebuilt in id order from the cells -- same set and length, checked --
// like WD's dense scans (packed cells; not right after a 24-bit
// renormalisation).  A warp turns 1024 consecutive cells into 32 bitmap words
// with coalesced loads and ballots; then as k_bm_compact.
template <typename D>
__global__ void __launch_bounds__(kBmBlock) k_tag_compact(const CellS<D>* __restrict__ cells,
                                                          DevCtrl* ctrl) {
  if (!ctrl->hp_dense) return;
  using Scan = cub::BlockScan<unsigned, kBmBlock>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ uint32_t s_ids[kBmBlock * 32];
  __shared__ unsigned s_base;
  const long long nn = ctrl->n_nodes;
  const long long nwords = (nn + 31) / 32;
  const uint32_t in_gen = Cell<D>::tag(ctrl->gen - 1u);
  uint32_t* __restrict__ q = ctrl->qptr[ctrl->in];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  for (long long b = (long long)blockIdx.x * kBmBlock; b < nwords; b += (long long)gridDim.x * kBmBlock) {
    const long long wbase = b + (long long)warp * 32;  // this warp's 32 words
    uint32_t w = 0;
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      const long long id = (wbase + k) * 32 + lane;
      const bool m = id < nn && Cell<D>::gen(cells[id]) == in_gen;
      const unsigned bits = __ballot_sync(0xffffffffu, m);
      if (lane == (unsigned)k) w = bits;
    }
    const long long i = wbase + lane;  // word index of this thread
    unsigned ex, total;
    Scan(ts).ExclusiveSum((unsigned)__popc(w), ex, total);
    if (total) {  // CTA-uniform
      if (threadIdx.x == 0) s_base = atomicAdd(&ctrl->tag_ctr, total);
      const uint32_t id0 = (uint32_t)(i * 32);
      for (uint32_t x = w; x; x &= x - 1u) s_ids[ex++] = id0 + (uint32_t)(__ffs(x) - 1);
      __syncthreads();
      const unsigned base = s_base;
      for (unsigned j = threadIdx.x; j < total; j += kBmBlock) q[base + j] = s_ids[j];
    }
    __syncthreads();
  }
}

// ============================================================ EP (K2) ===
// Edge worklist; improved destinations reserve their whole out-edge range.
// Ranges are collected per CTA (one global reservation per CTA round) and
// written by warps, lanes on consecutive slots.
constexpr int kEpRanges = 1024;
struct EpRanges {
  long long lo[kEpRanges];
  unsigned int len[kEpRanges];
  unsigned int off[kEpRanges];
  unsigned int count;
  unsigned int total;
  unsigned int base;
};

template <typename D, bool W, bool CHUNKED>
__global__ void __launch_bounds__(kBlock) k_ep_relax(const long long* __restrict__ row,
                                                     const uint32_t* __restrict__ src,
                                                     Relaxer<D, W> rx0, DevCtrl* ctrl,
                                                     CtlTail tail) {
  __shared__ EpRanges rg;
  const unsigned n = ctrl->qcount[ctrl->in];
  if (blockIdx.x * kBlock >= n) {  // idle CTA
    ctl_tail(tail, ctrl);
    return;
  }
  timer_begin(ctrl->t_relax);
  if (threadIdx.x == 0) rg.count = rg.total = 0;
  __syncthreads();
  const Relaxer<D, W> rx = bind(rx0, ctrl);
  const uint32_t* __restrict__ qin = ctrl->qptr[ctrl->in];
  ThreadCounters c;
  constexpr int K = 4;
  const unsigned stride = gridDim.x * kBlock;
  const unsigned long long pol = l2_evict_first();
  for (unsigned base = blockIdx.x * kBlock; base < n; base += stride * K) {
    uint32_t e[K], u[K], v[K], w[K];
    D du[K], cur[K], cand[K];
    unsigned valid = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const unsigned i = base + k * stride + threadIdx.x;
      if (i < n) {
        valid |= 1u << k;
        e[k] = qin[i];
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (valid >> k & 1u) {
        u[k] = ld_stream_pol(src + e[k], pol);
        v[k] = ld_stream_pol(rx.col + e[k], pol);
        w[k] = W ? ld_stream_pol(rx.wt + e[k], pol) : 1u;
      }
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (valid >> k & 1u) {
        du[k] = rx.dist(u[k]);
        cur[k] = rx.dist(v[k]);
      }
    unsigned want = 0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (valid >> k & 1u) {
        ++c.work;
        if (du[k] == DistTraits<D>::kInf) continue;
        ++c.relax;
        if (make_cand<D>(du[k], w[k], cand[k], rx.ovf) && cand[k] < cur[k]) want |= 1u << k;
      }
    CellS<D> old[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (want >> k & 1u) old[k] = atomicMin(rx.cells + v[k], Cell<D>::make(cand[k], rx.gen));
    bool pushk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      pushk[k] = false;
      if ((want >> k & 1u) && cand[k] < Cell<D>::dist(old[k]))
        pushk[k] = rx.claim_push(v[k], Cell<D>::gen(old[k]) != Cell<D>::tag(rx.gen));
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!pushk[k]) continue;
      const long long lo = row[v[k]];
      const unsigned len = (unsigned)(row[v[k] + 1] - lo);
      if (len == 0) continue;
      if (CHUNKED) {  // one reservation for the whole range (worklist.py:84-104)
        ++c.push;
        const unsigned slot = atomicAdd(&rg.count, 1u);
        if (slot < (unsigned)kEpRanges) {
          rg.lo[slot] = lo;
          rg.len[slot] = len;
          rg.off[slot] = atomicAdd(&rg.total, len);
        } else {
          const unsigned g = atomicAdd(rx.nout, len);
          for (unsigned j = 0; j < len; ++j) rx.qout[g + j] = (uint32_t)(lo + j);
        }
      } else {  // one reservation per edge
        for (unsigned j = 0; j < len; ++j) {
          ++c.push;
          rx.qout[atomicAdd(rx.nout, 1u)] = (uint32_t)(lo + j);
        }
      }
    }
    if (CHUNKED) {
      __syncthreads();
      const unsigned nr = rg.count < (unsigned)kEpRanges ? rg.count : (unsigned)kEpRanges;
      if (threadIdx.x == 0) rg.base = rg.total ? atomicAdd(rx.nout, rg.total) : 0u;
      __syncthreads();
      const unsigned gb = rg.base;
      for (unsigned r = threadIdx.x >> 5; r < nr; r += kBlock / 32) {
        const long long lo = rg.lo[r];
        const unsigned len = rg.len[r], off = gb + rg.off[r];
        for (unsigned j = lane_id(); j < len; j += 32) rx.qout[off + j] = (uint32_t)(lo + j);
      }
      __syncthreads();
      if (threadIdx.x == 0) rg.count = rg.total = 0;
      __syncthreads();
    }
  }
  flush_counters(ctrl, c);
  timer_end(ctrl->t_relax);
  ctl_tail(tail, ctrl);
}

// ====================================================== WD (K4 + K5/K6) ===
constexpr int kWdIPT = 8;                     // frontier items per thread in the scan
constexpr int kWdScanTile = kBlock * kWdIPT;  // 2048 items per scan tile
#ifndef GLB_WD_EPL
#define GLB_WD_EPL 8
#endif
constexpr int kWdEPL = GLB_WD_EPL;            // edges per lane of a warp tile
constexpr int kWdTile = 32 * kWdEPL;          // 256 edges per warp tile
static_assert(kWdEPL % 4 == 0, "head flags are handled in int4 groups");
constexpr int kWdWarpQ = 256;                 // per-warp push buffer (smem entries)

// One compacted frontier item of a WD invocation (16 B, one 128-bit load):
// its first active edge `pre` in the invocation's edge space, `base` = CSR
// index of that edge minus `pre` (mod 2^32: edge ids are < 2^32), and the node.
struct __align__(16) WdItem {
  uint32_t pre, base, node, pad;
};

// Remaining degree of every frontier item (minus the HP base offset
// min(window, deg), hierarchical.py:69-72), scanned as {edges, non-empty}.
// Non-empty items are compacted to j = exclusive count (items[j]), and
// tile_first[b] = the item holding active edge b*kWdTile -- the per-thread
// start of find_offsets (workload.py:45-72) at warp-tile granularity.
template <typename D>
__global__ void __launch_bounds__(kBlock) k_wd_scan(const long long* __restrict__ row,
                                                    const CellS<D>* __restrict__ cells,
                                                    LookbackState<2> lb, DevCtrl* ctrl) {
  pdl_trigger();
  WdItem* __restrict__ items = reinterpret_cast<WdItem*>(ctrl->wd_items_buf[ctrl->wd_cur]);
  unsigned int* __restrict__ tile_first = ctrl->wd_tf_buf[ctrl->wd_cur];
  using TS = TileScan<2, kBlock>;
  __shared__ typename TS::Storage st;
  __shared__ long long s_tile;
  // Dense frontier (a large fraction of all nodes): the worklist is exactly
  // {v : cell generation == the generation that pushed it}, so scan the nodes
  // in id order instead of the queue.  Items then come out sorted, their
  // CSR segments touch, and the relax kernel's col / weight reads become
  // contiguous runs instead of one partial sector per short segment.
  const bool dense = ctrl->wd_dense != 0;
  const uint32_t in_gen = Cell<D>::tag(ctrl->gen - 1u);
  const long long n = dense ? ctrl->n_nodes : ctrl->qcount[ctrl->in];
  const long long ntiles = (n + kWdScanTile - 1) / kWdScanTile;
  if (ntiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctrl->wd_total = 0;
      ctrl->wd_items = 0;
    }
    return;
  }
  if (blockIdx.x >= ntiles) return;  // idle CTA
  timer_begin(ctrl->t_scan);
  const uint32_t* __restrict__ q = ctrl->qptr[ctrl->in];
  const long long window = ctrl->window;
  const unsigned epoch = ctrl->scan_epoch;
  // Tiles are handed out in ticket order, so every predecessor of a tile is
  // already owned by a running (or finished) CTA: the look-back always makes
  // progress, whatever the residency.
  while (true) {
    if (threadIdx.x == 0) s_tile = (long long)atomicAdd(&ctrl->scan_ticket, 1ull);
    __syncthreads();
    const long long t = s_tile;
    if (t >= ntiles) break;
    const long long first = t * kWdScanTile + (long long)threadIdx.x * kWdIPT;
    uint32_t v[kWdIPT];
    long long beg[kWdIPT], rem[kWdIPT];
    Vec<2> sum;
    unsigned act = 0xFFu;
    if (dense) {
#pragma unroll
      for (int k = 0; k < kWdIPT; ++k) {
        v[k] = (uint32_t)(first + k);
        if (first + k >= n || Cell<D>::gen(cells[first + k]) != in_gen) act &= ~(1u << k);
      }
    } else if (first + kWdIPT <= n) {  // two 128-bit loads of worklist items
      const uint4 a = *reinterpret_cast<const uint4*>(q + first);
      const uint4 b = *reinterpret_cast<const uint4*>(q + first + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < kWdIPT; ++k) v[k] = first + k < n ? q[first + k] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kWdIPT; ++k) {
      rem[k] = 0;
      if (first + k < n && (act >> k & 1u)) {
        const long long lo = row[v[k]], hi = row[v[k] + 1];
        const long long b = hi - lo < window ? hi - lo : window;
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
        const long long j = ex.w[1], pre = ex.w[0];
        WdItem it;
        it.pre = (uint32_t)pre;
        it.base = (uint32_t)beg[k] - (uint32_t)pre;
        it.node = v[k];
        it.pad = 0;
        items[j] = it;
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
  timer_end(ctrl->t_scan);
}

// Warp-private push buffer in shared memory, flushed to the global worklist
// with one reservation per kWdWarpQ entries (no CTA barriers anywhere).
__device__ __forceinline__ void wq_flush(uint32_t* buf, unsigned& cnt, uint32_t* qout,
                                         unsigned int* nout) {
  __syncwarp();
  unsigned base = 0;
  if (lane_id() == 0 && cnt) base = atomicAdd(nout, cnt);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (unsigned i = lane_id(); i < cnt; i += 32) qout[base + i] = buf[i];
  __syncwarp();
  cnt = 0;
}

// Fused WD push (all 32 lanes): lane nodes with `has` become WdItems of the
// next step's list, appended in lane order with ONE 64-bit atomic on the
// (items << 32 | edges) counter -- the exclusive scan of workload.py:99-103
// done at push time -- plus the tile_first entry of every 256-edge tile
// boundary the item covers.  Zero-degree nodes are only counted.
__device__ __forceinline__ void wd_push_items(bool has, uint32_t v,
                                              const long long* __restrict__ row,
                                              WdItem* __restrict__ out,
                                              unsigned int* __restrict__ tf,
                                              unsigned long long* next_ctr,
                                              unsigned int* zero_ctr) {
  constexpr unsigned FULL = 0xffffffffu;
  const unsigned lane = lane_id();
  long long lo = 0, hi = 0;
  if (has) {
    lo = row[v];
    hi = row[v + 1];
  }
  const uint32_t deg = (uint32_t)(hi - lo);
  const bool item = has && deg > 0;
  unsigned ci = item ? 1u : 0u, ce = item ? deg : 0u;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned a = __shfl_up_sync(FULL, ci, off), b = __shfl_up_sync(FULL, ce, off);
    if (lane >= (unsigned)off) {
      ci += a;
      ce += b;
    }
  }
  const unsigned ti = __shfl_sync(FULL, ci, 31), te = __shfl_sync(FULL, ce, 31);
  const unsigned zeros = __popc(__ballot_sync(FULL, has && deg == 0));
  unsigned long long base = 0;
  if (lane == 0) {
    if (ti) base = atomicAdd(next_ctr, ((unsigned long long)ti << 32) | te);
    if (zeros) atomicAdd(zero_ctr, zeros);
  }
  base = __shfl_sync(FULL, base, 0);
  if (item) {
    const unsigned slot = (unsigned)(base >> 32) + ci - 1u;
    const uint32_t pre = (uint32_t)base + ce - deg;
    WdItem it;
    it.pre = pre;
    it.base = (uint32_t)lo - pre;
    it.node = v;
    it.pad = 0;
    out[slot] = it;
    for (uint32_t b = (pre + kWdTile - 1) / kWdTile; (unsigned long long)b * kWdTile < (unsigned long long)pre + deg; ++b)
      tf[b] = slot;
  }
}

// Flush of a warp push buffer as fused WD items.
__device__ __forceinline__ void wq_flush_items(uint32_t* buf, unsigned& cnt,
                                               const long long* __restrict__ row, DevCtrl* ctrl) {
  __syncwarp();
  const int nb = ctrl->wd_cur ^ 1;
  WdItem* out = reinterpret_cast<WdItem*>(ctrl->wd_items_buf[nb]);
  unsigned int* tf = ctrl->wd_tf_buf[nb];
  for (unsigned c0 = 0; c0 < cnt; c0 += 32) {
    const unsigned i = c0 + lane_id();
    wd_push_items(i < cnt, i < cnt ? buf[i] : 0u, row, out, tf, &ctrl->wd_next,
                  &ctrl->wd_zero_next);
  }
  __syncwarp();
  cnt = 0;
}

// Equal-work warp tiles: warp tile t owns active edges [t*256, t*256+256) and
// lane l relaxes edges t*256 + k*32 + l (k < 8), so every lane gets the same
// edge count (workload.py:104-108) and every col / weight load
// instruction covers 32 consecutive edges.  Owners come from a head-flag
// array in the warp's shared memory: every item of the tile writes its index
// at its first edge, and a thread-local + warp max-scan carries it forward.
// The kernel is bound by random 32 B sector gathers through L1TEX (one per
// cycle per SM, measured by tools/gather_peak.cu), so the layout spends
// about one L1 wavefront per edge on the dist[dst] gather and ~1/8 on the
// streams.  The item's distance is read fresh from its cell when the
// tile starts (the reference re-reads dn at every node entry,
// workload.py:131,140).  No CTA-wide barriers: warps advance independently.
//
// Software pipeline: while tile t's col/weight -> dist -> atomic chain is in
// flight, the warp fetches tile t+stride's tile_first -> item -> item
// distance chain, so each tile costs about three memory round trips.
constexpr int kWdWarps = kBlock / 32;

constexpr int kWdPre = 2;  // items per lane prefetched for the next tile (64: degree >= 4)

template <typename D>
struct WdMeta {
  uint32_t j0, j1;        // first / last item of the tile
  uint32_t st[kWdPre];    // lane's items j0 + lane + 32 i: first edge relative to the tile
  uint32_t base[kWdPre];  // CSR index - pre
  D du[kWdPre];           // item distance
};

template <typename D, bool W>
__global__ void __launch_bounds__(kBlock, GLB_WD_MINB) k_wd_relax(
    Relaxer<D, W> rx0, const long long* __restrict__ row, DevCtrl* ctrl, CtlTail tail) {
  pdl_wait();
  const WdItem* __restrict__ items = reinterpret_cast<const WdItem*>(ctrl->wd_items_buf[ctrl->wd_cur]);
  const unsigned int* __restrict__ tile_first = ctrl->wd_tf_buf[ctrl->wd_cur];
  const bool fused = ctrl->wd_fused != 0;
  __shared__ uint32_t s_q[kWdWarps][kWdWarpQ];
  __shared__ __align__(16) int s_own[kWdWarps][kWdTile];
  __shared__ uint32_t s_base[kWdWarps][kWdTile + 1];
  __shared__ D s_dn[kWdWarps][kWdTile + 1];
  const long long total = ctrl->wd_total;
  const long long nitems = ctrl->wd_items;
  const long long ntiles = (total + kWdTile - 1) / kWdTile;
  if ((long long)blockIdx.x * kWdWarps >= ntiles) {  // idle CTA
    ctl_tail(tail, ctrl);
    return;
  }
  timer_begin(ctrl->t_relax);
  const Relaxer<D, W> rx = bind(rx0, ctrl);
  const unsigned lane = lane_id();
  const unsigned warp = threadIdx.x >> 5;
  uint32_t* wq = s_q[warp];
  int* own = s_own[warp];
  uint32_t* sbase = s_base[warp];
  D* sdn = s_dn[warp];
  unsigned qn = 0;
  unsigned long long n_work = 0, n_relax = 0, n_push = 0;
  constexpr unsigned FULL = 0xffffffffu;
  const long long stride = (long long)gridDim.x * kWdWarps;
  const uint32_t last_item = (uint32_t)(nitems - 1);
  const unsigned long long pol = l2_evict_first();

  auto load_items = [&](long long tt, WdMeta<D>& mm, uint32_t (&node)[kWdPre]) {
    const uint32_t te0 = (uint32_t)(tt * kWdTile);
#pragma unroll
    for (int i = 0; i < kWdPre; ++i) {
      mm.st[i] = 0xFFFFFFFFu;
      mm.base[i] = 0;
      node[i] = 0;
      const uint32_t j = mm.j0 + lane + 32u * i;
      if (j <= mm.j1) {
        const WdItem it = items[j];
        mm.st[i] = it.pre > te0 ? it.pre - te0 : 0u;
        mm.base[i] = it.base;
        node[i] = it.node;
      }
    }
  };
  auto load_dist = [&](WdMeta<D>& mm, const uint32_t (&node)[kWdPre]) {
#pragma unroll
    for (int i = 0; i < kWdPre; ++i)
      mm.du[i] = mm.st[i] != 0xFFFFFFFFu ? rx.dist(node[i]) : DistTraits<D>::kInf;
  };

  // ---- prologue: metadata of the warp's first tile
  long long t = (long long)blockIdx.x * kWdWarps + warp;
  WdMeta<D> m;
  {
    m.j0 = tile_first[t];
    m.j1 = t + 1 < ntiles ? tile_first[t + 1] : last_item;
    uint32_t node[kWdPre];
    load_items(t, m, node);
    load_dist(m, node);
  }

  while (t < ntiles) {
    const long long tn = t + stride;
    const bool has_next = tn < ntiles;  // warp-uniform
    const uint32_t e0 = (uint32_t)(t * kWdTile);
    const uint32_t ecount = (uint32_t)(total - (long long)e0 < kWdTile ? total - e0 : kWdTile);
    // ---- head flags: item i of the tile writes i at its first edge
    {
      int4* o4 = reinterpret_cast<int4*>(own + lane * kWdEPL);
#pragma unroll
      for (int q = 0; q < kWdEPL / 4; ++q) o4[q] = make_int4(0, 0, 0, 0);
    }
    __syncwarp();
    // (the tile's last item may start exactly at the next tile: st == 256)
#pragma unroll
    for (int i = 0; i < kWdPre; ++i)
      if (m.st[i] < (uint32_t)kWdTile) {
        const unsigned idx = lane + 32u * i;
        own[m.st[i]] = (int)idx;
        sbase[idx] = m.base[i];
        sdn[idx] = m.du[i];
      }
    for (uint32_t c0 = m.j0 + 32 * kWdPre; c0 <= m.j1; c0 += 32) {  // rare: > 64 items
      const uint32_t j = c0 + lane;
      const WdItem it = items[j <= m.j1 ? j : m.j1];
      if (j <= m.j1 && it.pre - e0 < (uint32_t)kWdTile) {
        const uint32_t idx = j - m.j0;
        own[it.pre - e0] = (int)idx;
        sbase[idx] = it.base;
        sdn[idx] = rx.dist(it.node);
      }
    }
    __syncwarp();
    // ---- owners: local max over the lane's 8 consecutive head slots, warp
    //      max-scan for the carry, scanned owners back to shared memory ...
    {
      int4* o4 = reinterpret_cast<int4*>(own + lane * kWdEPL);
      int o[kWdEPL];
#pragma unroll
      for (int q = 0; q < kWdEPL / 4; ++q) {
        const int4 a = o4[q];
        o[4 * q] = a.x;
        o[4 * q + 1] = a.y;
        o[4 * q + 2] = a.z;
        o[4 * q + 3] = a.w;
      }
#pragma unroll
      for (int k = 1; k < kWdEPL; ++k) o[k] = o[k] > o[k - 1] ? o[k] : o[k - 1];
      int carry = o[kWdEPL - 1];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(FULL, carry, off);
        if (lane >= (unsigned)off) carry = y > carry ? y : carry;
      }
      int prev = __shfl_up_sync(FULL, carry, 1);
      if (lane == 0) prev = 0;
#pragma unroll
      for (int k = 0; k < kWdEPL; ++k) o[k] = o[k] > prev ? o[k] : prev;
#pragma unroll
      for (int q = 0; q < kWdEPL / 4; ++q) o4[q] = make_int4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    }
    __syncwarp();
    // ... and read back so that lane l takes edges k*32 + l: each load
    //     instruction of the col / weight streams covers 32 consecutive edges
    uint32_t e[kWdEPL];
    D dn[kWdEPL];
    unsigned valid = 0, inf_edges = 0;
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k) {
      const uint32_t f = (uint32_t)k * 32u + lane;
      const int ok = own[f];
      e[k] = sbase[ok] + e0 + f;
      dn[k] = sdn[ok];
      if (f < ecount) {
        if (dn[k] != DistTraits<D>::kInf)
          valid |= 1u << k;
        else
          ++inf_edges;
      }
    }
    // ---- stage 1: this tile's col / weights  ||  next tile's tile_first
    uint32_t v[kWdEPL], w[kWdEPL];
#if GLB_WD_BRANCHLESS
    // invalid slots load edge 0 (always mapped): no divergent regions
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k) {
      const uint32_t ek = (valid >> k & 1u) ? e[k] : 0u;
      v[k] = ld_stream_pol(rx.col + ek, pol);
      w[k] = W ? ld_stream_pol(rx.wt + ek, pol) : 1u;
    }
#else
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k)
      if (valid >> k & 1u) {
        v[k] = ld_stream_pol(rx.col + e[k], pol);
        w[k] = W ? ld_stream_pol(rx.wt + e[k], pol) : 1u;
      }
#endif
    WdMeta<D> nm;
    nm.j0 = nm.j1 = 0;
    if (has_next) {
      nm.j0 = tile_first[tn];
      nm.j1 = tn + 1 < ntiles ? tile_first[tn + 1] : last_item;
    }
    // ---- stage 2: this tile's dist[dst]  ||  next tile's items
    D cur[kWdEPL];
#if GLB_WD_BRANCHLESS
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k) cur[k] = rx.dist(v[k]);  // v of an invalid slot is a node id
#else
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k)
      if (valid >> k & 1u) cur[k] = rx.dist(v[k]);
#endif
    uint32_t nnode[kWdPre];
#pragma unroll
    for (int i = 0; i < kWdPre; ++i) {
      nm.st[i] = 0xFFFFFFFFu;
      nnode[i] = 0;
    }
    if (has_next) load_items(tn, nm, nnode);
    // ---- stage 3: this tile's atomics  ||  next tile's item distances
    unsigned want = 0;
    D cand[kWdEPL];
#if GLB_WD_BRANCHLESS
    bool ovf = false;
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k) {
      const unsigned long long c64 = (unsigned long long)dn[k] + (unsigned long long)w[k];
      const bool big = c64 >= (unsigned long long)DistTraits<D>::kInf;
      cand[k] = (D)c64;
      const bool vk = (valid >> k & 1u) != 0;
      ovf |= vk && big;
      want |= (unsigned)(vk && !big && cand[k] < cur[k]) << k;
    }
    if (ovf) atomicOr(rx.ovf, 1u);
#else
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k)
      if (valid >> k & 1u) {
        if (make_cand<D>(dn[k], w[k], cand[k], rx.ovf) && cand[k] < cur[k]) want |= 1u << k;
      }
#endif
    CellS<D> old[kWdEPL];
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k)
      if (want >> k & 1u) old[k] = atomicMin(rx.cells + v[k], Cell<D>::make(cand[k], rx.gen));
    load_dist(nm, nnode);
    unsigned first = 0;
#pragma unroll
    for (int k = 0; k < kWdEPL; ++k)
      if ((want >> k & 1u) && cand[k] < Cell<D>::dist(old[k])) {
        if (Cell<D>::kPacked) {
          if (Cell<D>::gen(old[k]) != Cell<D>::tag(rx.gen)) first |= 1u << k;
        } else if (claim(rx.stamp, v[k], rx.gen)) {
          first |= 1u << k;
        }
      }
    const unsigned nv = __popc(valid);
    n_work += nv + inf_edges;
    n_relax += nv;
    // ---- warp-aggregated append of the improved destinations
    const unsigned mine = __popc(first);
    unsigned incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, off);
      if (lane >= (unsigned)off) incl += y;
    }
    const unsigned wtotal = __shfl_sync(FULL, incl, 31);
    if (wtotal) {
      if (qn + wtotal > (unsigned)kWdWarpQ) {
        if (fused)
          wq_flush_items(wq, qn, row, ctrl);
        else
          wq_flush(wq, qn, rx.qout, rx.nout);
      }
      unsigned pos = qn + incl - mine;
#pragma unroll
      for (int k = 0; k < kWdEPL; ++k)
        if (first >> k & 1u) wq[pos++] = v[k];
      qn += wtotal;
      n_push += mine;
    }
    __syncwarp();  // the head-flag array is rewritten by the next tile
    m = nm;
    t = tn;
  }
  if (fused)
    wq_flush_items(wq, qn, row, ctrl);
  else
    wq_flush(wq, qn, rx.qout, rx.nout);
  ThreadCounters c;
  c.work = n_work;
  c.relax = n_relax;
  c.push = n_push;
  flush_counters(ctrl, c);
  timer_end(ctrl->t_relax);
  ctl_tail(tail, ctrl);
}

// ============================================================ setup ===
template <typename D>
__global__ void k_init_dist(CellS<D>* cells, long long n) {
  const CellS<D> inf = Cell<D>::make_tag(DistTraits<D>::kInf, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    cells[i] = inf;
}

// Seed the first worklist: the source (+ its NS children at distance 0,
// splitting.py:123-126) for node worklists, or the source's out-edge range for
// the EP edge worklist (edge_based.py:55).
template <typename D>
__global__ void k_seed(CellS<D>* cells, uint32_t* q, unsigned int* nq, long long src,
                       long long kid_lo, long long kid_hi, long long edge_lo, long long edge_hi,
                       bool edges) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (tid == 0) cells[src] = Cell<D>::make_tag(0, 0);
  if (edges) {
    for (long long e = edge_lo + tid; e < edge_hi; e += stride) q[e - edge_lo] = (uint32_t)e;
    if (tid == 0) *nq = (unsigned)(edge_hi - edge_lo);
  } else {
    if (tid == 0) q[0] = (uint32_t)src;
    for (long long k = kid_lo + tid; k < kid_hi; k += stride) {
      cells[k] = Cell<D>::make_tag(0, 0);
      q[1 + k - kid_lo] = (uint32_t)k;
    }
    if (tid == 0) *nq = (unsigned)(1 + kid_hi - kid_lo);
  }
}

// packed cells -> u32 distances (INF becomes 0xFFFFFFFF; widened on the host)
template <typename D>
__global__ void k_dist_u32(const CellS<D>* __restrict__ cells, long long n,
                           uint32_t* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const D d = Cell<D>::dist(cells[i]);
    out[i] = d == DistTraits<D>::kInf ? 0xFFFFFFFFu : (uint32_t)d;
  }
}

// 24-bit tier: every tag is reset to 0 ("no generation") before a
// generation that is a multiple of 128 starts (Cell<dist24_t>).
__global__ void k_renorm(uint32_t* __restrict__ cells, long long n, DevCtrl* ctrl, CtlTail tail) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    cells[i] &= ~0xFFu;
  ctl_tail(tail, ctrl);
}

template <typename D>
__global__ void k_dist_out(const CellS<D>* __restrict__ cells, long long n,
                           long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const D d = Cell<D>::dist(cells[i]);
    out[i] = d == DistTraits<D>::kInf ? 0x7FFFFFFFFFFFFFFFll : (long long)d;
  }
}

}  // namespace glb
