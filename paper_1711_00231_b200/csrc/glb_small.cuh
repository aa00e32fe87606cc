// glb_small.cuh -- small-frontier iterations without a kernel launch each.
//
// High-diameter graphs (config C3: 8,191 BFS levels on the 4096^2 grid) and
// the tails of low-diameter traversals run long sequences of iterations whose
// worklists hold a few thousand nodes.  There, a step costs its launch and
// memory-latency chain (scan -> relax -> control, ~30 us), not its work.
// k_small_loop runs such iterations back to back inside ONE thread-block
// cluster (8 CTAs x 1024 threads, one per SM): every CTA keeps an identical
// copy of the control block in shared memory and applies the same
// transitions; iterations are separated by cluster barriers; the
// per-iteration counters meet in CTA 0 through distributed shared memory.
// Each iteration is the strategy's own decomposition at cluster scale,
//   * BS: thread per worklist node, all out-edges (node_based.py:43-67)
//   * NS: BS over the split graph + child mirroring (splitting.py:141-162)
//   * WD (and HP's super-list WD-fallback, hierarchical.py:55-61): frontier
//     scan into shared memory, then equal edge counts per thread with a
//     binary search for the owner (workload.py:75-159)
// and the iteration bookkeeping is the same k_control logic (records, stamp
// generation, worklist swap).  It returns to the grid-wide kernels as soon as
// a worklist outgrows the cluster (kSmallItems nodes, kSmallEdges WD edges).
//
// Distances and worklists are re-read with ld.global.cg inside the loop: L1
// is not coherent with the L2 atomics, and a node's distance must be fresh
// when it is expanded again in a later iteration of the same launch.
#pragma once

#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>

#include "glb_control.cuh"
#include "glb_internal.cuh"
#include "glb_relax.cuh"

namespace glb {

namespace cg = cooperative_groups;

#ifndef GLB_SMALL_CTAS
#define GLB_SMALL_CTAS 8
#endif
#ifndef GLB_SMALL_PRECHECK
#define GLB_SMALL_PRECHECK 1  // plain-load filter before the atomic inside the cluster loop
#endif
#ifndef GLB_SMALL_BRANCHLESS
#define GLB_SMALL_BRANCHLESS 1  // small_relax without divergent regions (C3 BFS BS 79.5 -> 75.1 ms)
#endif
// Cluster size: 8 CTAs (the portable maximum) or 16 (non-portable opt-in),
// a template parameter of the kernel; the driver picks per strategy.
constexpr int kSmallCtas = GLB_SMALL_CTAS;        // the default / BS / NS cluster size
constexpr int kSmallThreads = 1024;               // threads per CTA
constexpr int kSmallItems = kSmallItemsCtl;       // worklist nodes one iteration may hold
constexpr long long kSmallEdges = kSmallEdgesCtl;  // WD: active edges one iteration may hold

// dynamic shared memory of k_small_loop (the WD item table, replicated per CTA)
template <typename D>
constexpr size_t small_smem_bytes() {
  return (size_t)(kSmallItems + 1) * 4 + (size_t)kSmallItems * 4 + (size_t)kSmallItems * sizeof(D);
}

template <typename D>
__device__ __forceinline__ D dist_cg(const CellS<D>* cells, uint32_t v) {
  return Cell<D>::dist(__ldcg(cells + v));
}

// Warp-aggregated append to a global worklist cursor.
__device__ __forceinline__ void g_append(uint32_t* q, unsigned int* cursor, uint32_t item) {
  q_append(q, cursor, item);
}

// Relax one batch of K edges; improved destinations are appended to the
// global out-list (its cursor lives in the global control block).
// Fused WD pushes (WdItems of the next list) instead of node appends; every
// lane of the warp must call small_relax together when it is set.
struct SmallPush {
  const long long* row;
  WdItem* out;
  unsigned int* tf;
  unsigned long long* next_ctr;
  unsigned int* zero_ctr;
};

template <int K, bool PRE = true, typename D, bool W>
__device__ __forceinline__ unsigned small_relax(const Relaxer<D, W>& rx, unsigned* cursor,
                                                uint32_t* qout, const uint32_t (&e)[K],
                                                const D (&dn)[K], unsigned valid,
                                                ThreadCounters& c, uint32_t (&v)[K],
                                                D (&cand)[K], const SmallPush* fused = nullptr) {
  uint32_t w[K];
  unsigned want = 0;
#if GLB_SMALL_BRANCHLESS
  // invalid slots load edge 0 / gather its head (always mapped): no divergent regions
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t ek = (valid >> k & 1u) ? e[k] : 0u;
    v[k] = __ldg(rx.col + ek);
    w[k] = W ? __ldg(rx.wt + ek) : 1u;
  }
  D cur[K];
#pragma unroll
  for (int k = 0; k < K; ++k) cur[k] = PRE && GLB_SMALL_PRECHECK ? dist_cg<D>(rx.cells, v[k]) : DistTraits<D>::kInf;
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
#else
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (valid >> k & 1u) {
      v[k] = __ldg(rx.col + e[k]);
      w[k] = W ? __ldg(rx.wt + e[k]) : 1u;
    }
  D cur[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (valid >> k & 1u) cur[k] = dist_cg<D>(rx.cells, v[k]);
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (valid >> k & 1u) {
      ++c.work;
      ++c.relax;
      if (make_cand<D>(dn[k], w[k], cand[k], rx.ovf) && cand[k] < cur[k]) want |= 1u << k;
    }
#endif
  unsigned won = 0, first = 0;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (want >> k & 1u) {
      const CellS<D> old = atomicMin(rx.cells + v[k], Cell<D>::make(cand[k], rx.gen));
      if (cand[k] < Cell<D>::dist(old)) {
        won |= 1u << k;
        if (Cell<D>::kPacked ? Cell<D>::gen(old) != Cell<D>::tag(rx.gen)
                             : atomicExch(rx.stamp + v[k], rx.gen) != rx.gen)
          first |= 1u << k;
      }
    }
  if (fused) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      wd_push_items((first >> k) & 1u, v[k], fused->row, fused->out, fused->tf, fused->next_ctr,
                    fused->zero_ctr);
    c.push += __popc(first);
    return won;
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (first >> k & 1u) {
      g_append(qout, cursor, v[k]);
      ++c.push;
    }
  return won;
}

// Equal edges per thread across the cluster (f = gt + r * 8192) over the item
// table (s_pre: first edge of every item, s_pre[n_items] = total).  The loop
// bound is warp-uniform so fused pushes can use warp collectives.
template <int ALL, typename D, bool W>
__device__ __forceinline__ void wd_tiles(const Relaxer<D, W>& rx, unsigned* cursor, uint32_t* qout,
                                         const uint32_t* s_pre, const uint32_t* s_base,
                                         const D* s_dn, int n_items, uint32_t total, unsigned gt,
                                         ThreadCounters& c, const SmallPush* fused) {
  constexpr int K = 4;
  const unsigned lane = lane_id();
  for (uint32_t fb = gt - lane; fb < total; fb += (uint32_t)K * ALL) {
    uint32_t e[K];
    D d[K];
    unsigned valid = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint32_t f = fb + lane + (uint32_t)k * ALL;
      if (f < total) {
        int lo = 0, hi = n_items;  // last item with s_pre <= f
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_pre[mid] <= f)
            lo = mid;
          else
            hi = mid;
        }
        e[k] = s_base[lo] + f;
        d[k] = s_dn[lo];
        if (d[k] != DistTraits<D>::kInf)
          valid |= 1u << k;
        else
          ++c.work;
      }
    }
    uint32_t v[K];
    D cand[K];
    small_relax<K>(rx, cursor, qout, e, d, valid, c, v, cand, fused);
  }
}

template <typename D, bool W, int CTAS>
__global__ void __cluster_dims__(CTAS, 1, 1) __launch_bounds__(kSmallThreads, 1)
    k_small_loop(const long long* __restrict__ row, const long long* __restrict__ cs,
                 long long n_orig, const uint32_t* __restrict__ ep_src, bool ep_chunked,
                 Relaxer<D, W> rx0, DevCtrl* gctrl, CtlTail tail) {
  constexpr int kSmallAll = CTAS * kSmallThreads;  // threads of the cluster
  extern __shared__ __align__(16) unsigned char s_dyn[];
  D* s_dn = reinterpret_cast<D*>(s_dyn);                                   // [kSmallItems]
  uint32_t* s_pre = reinterpret_cast<uint32_t*>(s_dyn + kSmallItems * sizeof(D));  // [+1]
  uint32_t* s_base = s_pre + kSmallItems + 1;                              // [kSmallItems]
  using LScan = cub::BlockScan<long long, kSmallThreads, cub::BLOCK_SCAN_WARP_SCANS>;
  using IScan = cub::BlockScan<int, kSmallThreads, cub::BLOCK_SCAN_WARP_SCANS>;
  __shared__ union {
    typename LScan::TempStorage l;
    typename IScan::TempStorage i;
  } s_scan;
  __shared__ DevCtrl sc;                 // this CTA's copy of the control block
  // CTA 0 holds the cluster's per-iteration cursors and counters in THREE
  // rotating slots: iteration k uses slot k % 3, all CTAs read it after the
  // one cluster barrier of iteration k, and rank 0 clears slot (k + 2) % 3
  // (read by everybody before that barrier, next written after the next one)
  // -- one barrier per iteration instead of two.
  __shared__ unsigned int s_cur[3];            // out-list cursor
  __shared__ unsigned int s_nxt[3];            // HP: next-sublist cursor (unfinished windows)
  __shared__ unsigned long long s_acc[3][4];   // work, relax, push, work^2
  __shared__ unsigned int s_max[3];            // per-thread work maximum (native 32-bit atomicMax)
  __shared__ unsigned long long s_wdn[3];      // fused WD: (items << 32) | edges appended
  __shared__ unsigned int s_wdz[3];            // fused WD: zero-degree pushes
  __shared__ long long s_total;
  __shared__ int s_go;
  __shared__ unsigned long long s_t0;

  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const unsigned tid = threadIdx.x;
  const unsigned gt = rank * kSmallThreads + tid;
  unsigned int* cur0 = cluster.map_shared_rank(s_cur, 0);
  unsigned long long* acc0 = cluster.map_shared_rank(&s_acc[0][0], 0);
  unsigned int* max0 = cluster.map_shared_rank(s_max, 0);
  unsigned int* nxt0 = cluster.map_shared_rank(s_nxt, 0);
  unsigned long long* wdn0 = cluster.map_shared_rank(s_wdn, 0);
  unsigned int* wdz0 = cluster.map_shared_rank(s_wdz, 0);

  if (tid == 0) {
    sc = *gctrl;
    s_go = small_eligible(&sc);
    s_t0 = gtime();
  }
  if (tid < 3) {
    s_cur[tid] = 0;
    s_nxt[tid] = 0;
    s_max[tid] = 0;
    s_wdn[tid] = 0;
    s_wdz[tid] = 0;
    for (int k = 0; k < 4; ++k) s_acc[tid][k] = 0;
  }
  cluster.sync();
#ifdef GLB_SMALL_TRACE
  unsigned long long tr[4] = {0, 0, 0, 0}, tr_n = 0, tr_t = gtime();
#endif
  for (unsigned it = 0; s_go; ++it) {
    const unsigned slot = it % 3u;
    const unsigned n = sc.qcount[sc.in];
    const uint32_t* qin = sc.qptr[sc.in];
    // appends go after what the out list already holds (HP's super-out list
    // accumulates over the sub-iterations of a super-iteration)
    uint32_t* qout = sc.qptr[sc.out] + sc.qcount[sc.out];
    unsigned* cursor = cur0 + slot;
    Relaxer<D, W> rx = rx0;
    rx.gen = sc.gen;
    ThreadCounters c;
    bool ran = true;
    SmallPush push;
    const SmallPush* fused = nullptr;
    if (sc.wd_fused || sc.wd_fused_small) {
      push.row = row;
      push.out = reinterpret_cast<WdItem*>(sc.wd_items_buf[sc.wd_cur ^ 1]);
      push.tf = sc.wd_tf_buf[sc.wd_cur ^ 1];
      push.next_ctr = wdn0 + slot;
      push.zero_ctr = wdz0 + slot;
      fused = &push;
    }
    if (sc.mode == kModeWDF) {
      // ---- the item list the previous step appended: load it as the table
      const WdItem* it_in = reinterpret_cast<const WdItem*>(sc.wd_items_buf[sc.wd_cur]);
      const int ni = (int)sc.wd_items;
      for (int j = tid; j < ni; j += kSmallThreads) {
        const WdItem it = it_in[j];
        s_pre[j] = it.pre;
        s_base[j] = it.base;
        s_dn[j] = dist_cg<D>(rx.cells, it.node);  // dn at node entry (workload.py:131,140)
      }
      if (tid == 0) {
        s_pre[ni] = (uint32_t)sc.wd_total;
        s_total = sc.wd_total;
      }
      __syncthreads();
      wd_tiles<kSmallAll, D, W>(rx, cursor, qout, s_pre, s_base, s_dn, ni, (uint32_t)sc.wd_total, gt, c,
                     fused);
    } else if (sc.mode == kModeWD) {
      // ---- scan of remaining degrees, replicated in every CTA (items
      //      contiguous per thread), so each holds the whole item table
      const long long window = sc.window;
      const unsigned ipt = (n + kSmallThreads - 1) / kSmallThreads;
      const unsigned i0 = tid * ipt;
      long long rem_sum = 0;
      int cnt = 0;
      for (unsigned k = 0; k < ipt; ++k) {
        const unsigned i = i0 + k;
        if (i < n) {
          const uint32_t u = __ldcg(qin + i);
          const long long lo = row[u], hi = row[u + 1];
          const long long b = hi - lo < window ? hi - lo : window;
          rem_sum += hi - lo - b;
          cnt += hi - lo - b > 0;
        }
      }
      long long ex_e, tot_e;
      int ex_i, tot_i;
      LScan(s_scan.l).ExclusiveSum(rem_sum, ex_e, tot_e);
      __syncthreads();
      IScan(s_scan.i).ExclusiveSum(cnt, ex_i, tot_i);
      if (tid == 0) s_total = tot_e;
      if (tot_e > kSmallEdges) {  // too big for the cluster: the grid kernels take this step
        ran = false;
      } else if (tot_e > 0) {
        for (unsigned k = 0; k < ipt; ++k) {
          const unsigned i = i0 + k;
          if (i < n) {
            const uint32_t u = __ldcg(qin + i);
            const long long lo = row[u], hi = row[u + 1];
            const long long b = hi - lo < window ? hi - lo : window;
            const long long r = hi - lo - b;
            if (r > 0) {
              s_pre[ex_i] = (uint32_t)ex_e;
              s_base[ex_i] = (uint32_t)(lo + b) - (uint32_t)ex_e;
              s_dn[ex_i] = dist_cg<D>(rx.cells, u);  // dn at node entry (workload.py:131,140)
              ++ex_i;
              ex_e += r;
            }
          }
        }
        if (tid == 0) s_pre[tot_i] = (uint32_t)tot_e;
        __syncthreads();
        wd_tiles<kSmallAll, D, W>(rx, cursor, qout, s_pre, s_base, s_dn, tot_i, (uint32_t)tot_e, gt, c,
                       fused);
      }
    } else if (sc.mode == kModeHP) {
      // ---- HP window sub-iteration (hierarchical.py:95-120): thread per
      //      sublist node relaxes [s*mdt, (s+1)*mdt) of its edges; nodes with
      //      edges left carry into the next sublist
      uint32_t* qnext = sc.qptr[sc.next] + sc.qcount[sc.next];
      unsigned* ncur = nxt0 + slot;
      const long long window = sc.window, mdt = sc.mdt;
      for (unsigned i = gt; i < n; i += kSmallAll) {
        const uint32_t u = __ldcg(qin + i);
        const long long r0 = row[u], r1 = row[u + 1];
        const long long start = r0 + window;
        if (start >= r1) continue;
        const long long end = start + mdt < r1 ? start + mdt : r1;
        if (end < r1) {
          g_append(qnext, ncur, u);
          ++c.push;
        }
        const D du = dist_cg<D>(rx.cells, u);
        if (du == DistTraits<D>::kInf) continue;
        constexpr int K = 4;
        for (uint32_t b = (uint32_t)start; b < (uint32_t)end; b += K) {
          uint32_t e[K];
          D d[K];
          unsigned valid = 0;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            e[k] = b + k;
            d[k] = du;
            if (b + k < (uint32_t)end) valid |= 1u << k;
          }
          uint32_t v[K];
          D cand[K];
          small_relax<K>(rx, cursor, qout, e, d, valid, c, v, cand);
        }
      }
    } else if (ep_src) {
      // ---- EP (edge_based.py:70-87): thread per worklist edge; an improved
      //      destination appends its whole out-edge range with one
      //      reservation (work chunking) or one per edge
      // Unweighted graphs: every source of a listed edge was pushed with its
      // final level (all candidates of a level-synchronous step are equal),
      // so the level travels with the edge (ep_dn, written at push time) and
      // the walk goes edge -> column -> atomic, without the src / dist loads
      // and the pre-check (two dependent round trips less per level).  Lists
      // this launch did not write (iteration 0) load the level.
      const bool carry = !W && sc.ep_dn[0] != nullptr;
      const uint32_t* dn_in = carry && it > 0 ? sc.ep_dn[sc.in] : nullptr;
      uint32_t* dn_out = carry ? sc.ep_dn[sc.out] + sc.qcount[sc.out] : nullptr;
      for (unsigned i = gt; i < n; i += kSmallAll) {
        const uint32_t e = __ldcg(qin + i);
        uint32_t v, w = 1u;
        D du, dv;
        if (dn_in) {
          const uint32_t dc = __ldcg(dn_in + i);
          v = __ldg(rx.col + e);
          du = (D)dc;
          dv = DistTraits<D>::kInf;
        } else {
          const uint32_t u = __ldg(ep_src + e);
          v = __ldg(rx.col + e);
          if (W) w = __ldg(rx.wt + e);
          du = dist_cg<D>(rx.cells, u);
          dv = dist_cg<D>(rx.cells, v);  // in flight with du
        }
        ++c.work;
        if (du == DistTraits<D>::kInf) continue;
        ++c.relax;
        D cand;
        if (!make_cand<D>(du, w, cand, rx.ovf) || cand >= dv) continue;
        const long long lo = row[v], hi = row[v + 1];  // the push's range, in flight with the atomic
        const CellS<D> old = atomicMin(rx.cells + v, Cell<D>::make(cand, rx.gen));
        if (cand >= Cell<D>::dist(old)) continue;
        const bool first = Cell<D>::kPacked ? Cell<D>::gen(old) != Cell<D>::tag(rx.gen)
                                            : atomicExch(rx.stamp + v, rx.gen) != rx.gen;
        if (!first) continue;
        const unsigned len = (unsigned)(hi - lo);
        if (len == 0) continue;
        if (ep_chunked) {
          ++c.push;
          const unsigned b = atomicAdd(cursor, len);
          for (unsigned j = 0; j < len; ++j) qout[b + j] = (uint32_t)(lo + j);
          if (dn_out)
            for (unsigned j = 0; j < len; ++j) dn_out[b + j] = (uint32_t)cand;
        } else {
          for (unsigned j = 0; j < len; ++j) {
            ++c.push;
            const unsigned b = atomicAdd(cursor, 1u);
            qout[b] = (uint32_t)(lo + j);
            if (dn_out) dn_out[b] = (uint32_t)cand;
          }
        }
      }
    } else {
      // ---- BS / NS: thread per worklist node (node i -> cluster thread i mod 8192)
      // BS / NS id-ordered frontiers: the list a grid step handed over has its
      // bits set -- clear them; the cluster's own lists carry no bits
      // (bm_valid is dropped on exit), so its pushes stay off the bitmap
      uint32_t* bm_in = it == 0 && sc.bm_thr && sc.bm_valid[sc.in] ? sc.bm[sc.in] : nullptr;
      for (unsigned i = gt; i < n; i += kSmallAll) {
        const uint32_t u = __ldcg(qin + i);
        if (bm_in) bm_in[u >> 5] = 0u;
        const uint32_t lo = (uint32_t)row[u], hi = (uint32_t)row[u + 1];  // in flight with du
        const D du = dist_cg<D>(rx.cells, u);
        if (du == DistTraits<D>::kInf) continue;
        constexpr int K = 4;
        for (uint32_t b = lo; b < hi; b += K) {
          uint32_t e[K];
          D d[K];
          unsigned valid = 0;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            e[k] = b + k;
            d[k] = du;
            if (b + k < hi) valid |= 1u << k;
          }
          uint32_t v[K];
          D cand[K];
          // unweighted BS / NS walks go straight to the atomic: one dependent
          // round trip less per level (C3 BFS BS -6 %); weighted ones keep the
          // filter (C3 SSSP BS +4 % without it: 32K-node lists of atomics)
          const unsigned won = small_relax<K, W>(rx, cursor, qout, e, d, valid, c, v, cand);
          if (cs) {  // NS: mirror improved parents onto their children (splitting.py:154-160)
#pragma unroll
            for (int k = 0; k < K; ++k) {
              if (!(won >> k & 1u) || v[k] >= n_orig) continue;
              const long long k1 = cs[v[k] + 1];
              for (long long ch = cs[v[k]]; ch < k1; ++ch) {
                const uint32_t child = (uint32_t)(n_orig + ch);
                ++c.relax;
                bool first = false;
                if (relax_cell<D>(rx.cells, child, cand[k], rx.gen, &first) &&
                    rx.claim_push(child, first)) {
                  g_append(qout, cursor, child);
                  ++c.push;
                }
              }
            }
          }
        }
      }
    }
#ifdef GLB_SMALL_TRACE
    if (tid == 0) { const unsigned long long t = gtime(); tr[0] += t - tr_t; tr_t = t; }
#endif
    // ---- counters of the iteration meet in CTA 0 (distributed shared memory)
    if (ran && sc.ptw && c.work && sc.ptw_off + gt < sc.ptw_cap)
      sc.ptw[sc.ptw_off + gt] = c.work > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c.work;
    if (ran) {
      unsigned long long w = c.work, r = c.relax, p = c.push, sq = c.work * c.work, mx = c.work;
      constexpr unsigned FULL = 0xffffffffu;
      if (!__any_sync(FULL, ((c.work | c.relax | c.push) >> 13) != 0)) {
        // small per-thread counts (every lane < 2^13, so 32 squares sum below
        // 2^31): single-instruction warp reductions
        w = __reduce_add_sync(FULL, (unsigned)c.work);
        r = __reduce_add_sync(FULL, (unsigned)c.relax);
        p = __reduce_add_sync(FULL, (unsigned)c.push);
        sq = __reduce_add_sync(FULL, (unsigned)(c.work * c.work));
        mx = __reduce_max_sync(FULL, (unsigned)c.work);
      } else {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          w += __shfl_xor_sync(FULL, w, off);
          r += __shfl_xor_sync(FULL, r, off);
          p += __shfl_xor_sync(FULL, p, off);
          sq += __shfl_xor_sync(FULL, sq, off);
          const unsigned long long o = __shfl_xor_sync(FULL, mx, off);
          mx = o > mx ? o : mx;
        }
      }
      if (lane_id() == 0) {
        unsigned long long* a = acc0 + slot * 4;
        if (w) atomicAdd(&a[0], w);
        if (r) atomicAdd(&a[1], r);
        if (p) atomicAdd(&a[2], p);
        if (sq) atomicAdd(&a[3], sq);
        if (mx) atomicMax(max0 + slot, mx > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)mx);
      }
    }
#ifdef GLB_SMALL_TRACE
    if (tid == 0) { const unsigned long long t = gtime(); tr[1] += t - tr_t; tr_t = t; }
#endif
    cluster.sync();  // every push and counter of the iteration has landed
#ifdef GLB_SMALL_TRACE
    if (tid == 0) { const unsigned long long t = gtime(); tr[2] += t - tr_t; tr_t = t; }
#endif
    if (tid == 0) {
      DevCtrl* cc = &sc;
      if (!ran) {
        s_go = 0;
      } else {
        const unsigned produced = *(volatile unsigned*)cursor;
        cc->qcount[cc->out] += produced;
        if (cc->mode == kModeHP) cc->qcount[cc->next] += *(volatile unsigned*)(nxt0 + slot);
        const bool wd_empty = (cc->mode == kModeWD || cc->mode == kModeWDF) && s_total == 0;
        if (rank == 0 && !wd_empty && cc->nrec < cc->rec_cap) {
          DevRecord& rec = cc->recs[cc->nrec];
          rec.iteration = cc->iteration;
          rec.sub = cc->sub;
          rec.tag = cc->tag;
          rec.active = n;
          rec.threads = kSmallAll;
          rec.work = (long long)s_acc[slot][0];
          rec.relax = (long long)s_acc[slot][1];
          rec.push = (long long)s_acc[slot][2];
          rec.work_max = (long long)s_max[slot];
          rec.work_sumsq = (double)s_acc[slot][3];
          rec.k0 = s_t0;
          rec.k1 = gtime();
          rec.o0 = rec.o1 = 0;
        }
        // every CTA advances its copy of the list cursor identically
        if (!wd_empty && cc->nrec < cc->rec_cap) {
          const long long off = ctl_ptw_take(cc, kSmallAll);
          if (rank == 0) cc->recs[cc->nrec].ptw_off = off;
        }
        if (!wd_empty) cc->nrec += 1;
        if (cc->strategy == GLB_HP) {  // hierarchical.py:54-136
          ctl_hp_after_step(cc);
        } else if (wd_empty) {
          cc->done = 1;
        } else if (cc->wd_fused || (cc->wd_fused_small && cc->strategy == GLB_WD)) {
          ctl_wd_fused_advance(cc, *(volatile unsigned long long*)(wdn0 + slot),
                               *(volatile unsigned*)(wdz0 + slot));
        } else {
          ctl_simple_advance(cc);
        }
        if (cc->done) cc->mode = kModeDone;
        ctl_check_renorm(cc);
        s_go = small_eligible(cc);
        if (rank == 0) {  // clear the slot of iteration it + 2 (see above)
          const unsigned z = (it + 2u) % 3u;
          s_cur[z] = 0;
          s_nxt[z] = 0;
          s_max[z] = 0;
          s_wdn[z] = 0;
          s_wdz[z] = 0;
          for (int k = 0; k < 4; ++k) s_acc[z][k] = 0;
          s_t0 = gtime();
        }
      }
    }
    __syncthreads();  // this CTA's threads see the transition (identical in every CTA)
#ifdef GLB_SMALL_TRACE
    if (tid == 0) { const unsigned long long t = gtime(); tr[3] += t - tr_t; tr_t = t; ++tr_n; }
#endif
  }
  cluster.sync();  // no CTA leaves while others may still read its shared memory
#ifdef GLB_SMALL_TRACE
  if (rank == 0 && tid == 0 && tr_n)
    printf("small_loop trace: %llu iters  relax %.2f  counters %.2f  barrier %.2f  control %.2f us/iter\n",
           tr_n, tr[0] / 1e3 / tr_n, tr[1] / 1e3 / tr_n, tr[2] / 1e3 / tr_n, tr[3] / 1e3 / tr_n);
#endif
  if (rank == 0 && tid == 0) {
    sc.overflow |= __ldcg(&gctrl->overflow);  // make_cand's flag lives in the global block
    sc.small_exit = 1;
    sc.use_small = 0;
    sc.bm_valid[0] = sc.bm_valid[1] = 0;  // both bitmaps are zero now
    ctl_reset_timers(&sc);
    *gctrl = sc;
  }
  if (tail.on) {
    cluster.sync();  // the control block is written back before any CTA counts itself out
    ctl_tail(tail, gctrl);
  }
}

}  // namespace glb
