// glb_bins.cuh -- degree-binned relaxation of edge windows: the kernels of
// hierarchical processing (HP, hierarchical.py:95-120) and node splitting
// (NS, splitting.py:141-162).
//
// A step hands every lane of a warp chunk (32 worklist items, claimed by
// ticket) one edge window [lo, lo + len) relaxed from distance dn -- HP: the
// sub-iteration window [s*mdt, (s+1)*mdt) of a sublist node; NS: the whole
// out-range of a split-graph node.  Windows are binned by length:
//
//   thread bin  len <= 32       one lane's window;
//   warp bin    32 < len < 2048 a window its warp walks lane-consecutively;
//                               both bins stay with the warp that drew the
//                               items (32 per warp ticket): the warp walks the
//                               concatenation of its lanes' windows (exclusive
//                               warp scan of the lengths; an edge's owner lane
//                               by a 5-step shuffle search), 32 consecutive
//                               edges per load instruction and K per lane in
//                               flight, so a thread-bin window never idles 31
//                               lanes and a warp-bin window never idles the
//                               tail of its last pass;
//   CTA bin     len >= 2048     appended to the grid-wide bin (one 64-bit
//                               atomic reserves the entry and its 2048-edge
//                               pieces); the step's second kernel (k_bigbin,
//                               a programmatic dependent launch) lets every
//                               CTA claim pieces by ticket and stages each
//                               piece's columns / weights into shared memory
//                               with 1-D TMA bulk copies (cp.async.bulk +
//                               mbarrier), double-buffered: the next piece's
//                               copy is in flight while the current one is
//                               relaxed, so the dependent chain per edge is
//                               smem -> dist gather -> atomic.
//
// NS wraps the relaxation with the reference's child mirroring: an improved
// original node writes its value onto its split children (NsMirror).
#pragma once

#include "glb_relax.cuh"

#ifndef GLB_BIN_MINB
#define GLB_BIN_MINB 3  // CTAs per SM the window kernels are register-capped for
#endif

namespace glb {

constexpr unsigned kBinThreadMax = 32;   // thread bin: windows of at most 32 edges
#ifndef GLB_BIN_CTA_MIN
#define GLB_BIN_CTA_MIN 512  // C4 A/B: 2048 -> 512 took HP BFS 1.36 -> 1.09 ms, NS 2.06 -> 1.69 ms
#endif
constexpr long long kBinCtaMin = GLB_BIN_CTA_MIN;  // CTA bin: windows of at least this many edges
constexpr long long kBinPiece = 2048;    // edges per CTA-bin piece (one TMA stage)
constexpr int kBinBuf = (int)kBinPiece + 4;  // a piece plus the 16-byte alignment slack
#ifndef GLB_BIN_K
#define GLB_BIN_K 4
#endif
constexpr int kBinK = GLB_BIN_K;         // edges in flight per lane

// -------------------------------------------------------------- sinks ---
// Warp-private push buffer in shared memory, flushed with one global
// reservation per kBinWarpQ entries: the warps of a CTA never wait for each
// other (all 32 lanes call push / flush together).
constexpr int kBinWarps = kBlock / 32;
constexpr int kBinWarpQ = 256;
struct WarpSink {
  uint32_t* buf;
  unsigned n;
  uint32_t* qout;
  unsigned int* nout;
  uint32_t* bm = nullptr;  // NS: the out list's member bitmap (id-ordered frontiers)
  __device__ __forceinline__ void flush() {
    __syncwarp();
    unsigned base = 0;
    if (lane_id() == 0 && n) base = atomicAdd(nout, n);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (unsigned i = lane_id(); i < n; i += 32) {
      const uint32_t v = buf[i];
      qout[base + i] = v;
      if (bm) bm_set(bm, v);
    }
    __syncwarp();
    n = 0;
  }
  template <int K>
  __device__ __forceinline__ void push(unsigned first, const uint32_t (&v)[K], ThreadCounters& c) {
    constexpr unsigned FULL = 0xffffffffu;
    const unsigned mine = __popc(first), lane = lane_id();
    unsigned incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, off);
      if (lane >= (unsigned)off) incl += y;
    }
    const unsigned total = __shfl_sync(FULL, incl, 31);
    if (!total) return;
    if (n + total > (unsigned)kBinWarpQ) flush();
    unsigned pos = n + incl - mine;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (first >> k & 1u) buf[pos++] = v[k];
    n += total;
    c.push += mine;
  }
};

// -------------------------------------------------------------- mirrors ---
struct NoMirror {
  __device__ __forceinline__ void bind_bm(uint32_t*) {}
  template <int K, typename D, bool W>
  __device__ __forceinline__ void operator()(const Relaxer<D, W>&, unsigned,
                                             const uint32_t (&)[K], const D (&)[K],
                                             ThreadCounters&) const {}
};

// splitting.py:154-160: a strict improvement of original node v is written
// onto its children n_orig + cs[v] .. n_orig + cs[v+1] (contiguous ids);
// pushes go straight to the out list (warp-aggregated, divergence-safe).
struct NsMirror {
  const long long* __restrict__ cs;
  long long n_orig;
  uint32_t* bm = nullptr;  // the out list's member bitmap (bound per step on the device)
  __device__ __forceinline__ void bind_bm(uint32_t* b) { bm = b; }
  template <int K, typename D, bool W>
  __device__ __forceinline__ void operator()(const Relaxer<D, W>& rx, unsigned won,
                                             const uint32_t (&v)[K], const D (&cand)[K],
                                             ThreadCounters& c) const {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!(won >> k & 1u) || v[k] >= n_orig) continue;
      const long long k1 = cs[v[k] + 1];
      for (long long ch = cs[v[k]]; ch < k1; ++ch) {
        const uint32_t child = (uint32_t)(n_orig + ch);
        ++c.relax;
        bool first = false;
        if (relax_cell<D>(rx.cells, child, cand[k], rx.gen, &first) && rx.claim_push(child, first)) {
          q_append(rx.qout, rx.nout, child);
          if (bm) bm_set(bm, child);
          ++c.push;
        }
      }
    }
  }
};

// ------------------------------------------------------ TMA / mbarrier ---
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "GLB_MBAR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra GLB_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completing on `bar`; the
// source lines are fetched L2 evict-first (single-use edge streams).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------- binned windows ---
// Reserve a CTA-bin entry with its pieces (grid-wide; k_bigbin relaxes it).
template <typename D>
__device__ __forceinline__ void cta_bin_push(DevCtrl* ctrl, long long lo, long long len, D dn) {
  const unsigned pieces = (unsigned)((len + kBinPiece - 1) / kBinPiece);
  const unsigned long long r = atomicAdd(&ctrl->hp_big_ctr, (1ull << 32) | (unsigned long long)pieces);
  const unsigned e = (unsigned)(r >> 32);
  HpBig* b = ctrl->hp_big + e;
  b->dn = (unsigned long long)dn;
  b->lo = lo;
  b->hi = lo + len;
  b->qbase = (unsigned)r;
  // piece -> window table: k_bigbin finds a claimed piece's window in one read
  for (unsigned k = 0; k < pieces; ++k) ctrl->hp_owner[(unsigned)r + k] = e;
}

// The windows of a warp's 32 lanes (len 0 = none; all lanes call it).
template <typename D, bool W, class M>
__device__ __forceinline__ void warp_windows(const Relaxer<D, W>& rx, WarpSink& sink, long long lo,
                                             long long len, D dn, const M& mirror, DevCtrl* ctrl,
                                             ThreadCounters& c) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int K = kBinK;
  const unsigned lane = lane_id();
  if (len >= kBinCtaMin) {  // CTA bin
    cta_bin_push<D>(ctrl, lo, len, dn);
    len = 0;
  }
  const unsigned tl = (unsigned)len;
  unsigned incl = tl;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned y = __shfl_up_sync(FULL, incl, off);
    if (lane >= (unsigned)off) incl += y;
  }
  const unsigned total = __shfl_sync(FULL, incl, 31);
  const unsigned pre = incl - tl;
  const uint32_t base32 = (uint32_t)lo - pre;  // edge of flat slot f: base32 + f (edge ids < 2^32)
  const unsigned long long pol = l2_evict_first();
  for (unsigned f0 = 0; f0 < total; f0 += 32u * K) {
    uint32_t v[K], w[K];
    D d[K];
    unsigned valid = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const unsigned f = f0 + (unsigned)k * 32u + lane;
      int o = 0;  // last lane whose window starts at or before f
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const unsigned p = __shfl_sync(FULL, pre, o + step);
        if (p <= f) o += step;
      }
      const uint32_t e = __shfl_sync(FULL, base32, o) + f;
      d[k] = shfl_dist(dn, o);
#if GLB_RELAX_BRANCHLESS
      valid |= (unsigned)(f < total) << k;
      const uint32_t ek = f < total ? e : 0u;  // invalid slots load edge 0 (always mapped)
      v[k] = ld_stream_pol(rx.col + ek, pol);
      w[k] = W ? ld_stream_pol(rx.wt + ek, pol) : 1u;
#else
      v[k] = 0;
      w[k] = 1u;
      if (f < total) {
        valid |= 1u << k;
        v[k] = ld_stream_pol(rx.col + e, pol);
        if (W) w[k] = ld_stream_pol(rx.wt + e, pol);
      }
#endif
    }
    D cand[K];
    const unsigned won = relax_vals<K>(rx, sink, v, w, d, valid, c, cand);
    mirror(rx, won, v, cand, c);
  }
}

// Items per warp claim: 32, or fewer when the list would not give every
// warp of the grid a full chunk -- then a warp's edges come from fewer,
// longer windows and its lanes still walk 32 consecutive edges per load
// (HP sub-iterations s >= 1 hold a few thousand windows of ~mdt edges; with
// 32 per warp they ran as long serial chains on a fraction of the warps).
__device__ __forceinline__ int bin_chunk(long long n) {
  const long long warps = (long long)gridDim.x * kBinWarps;
  if (n >= 32 * warps) return 32;
  const long long c = n / warps;
  int p = 1;
  while (p * 2 <= c) p *= 2;
  return p;
}

// Claim the next `chunk` items of the step for this warp (dynamic: warps
// that drew light items take more).  Returns the first item, or -1 when done.
__device__ __forceinline__ long long warp_next_chunk(DevCtrl* ctrl, long long n, int chunk) {
  unsigned long long t = 0;
  if (lane_id() == 0) t = atomicAdd(&ctrl->relax_ticket, (unsigned long long)chunk);
  t = __shfl_sync(0xffffffffu, t, 0);
  return (long long)t < n ? (long long)t : -1;
}

// ============================================================ HP (K10) ===
// Sub-iteration window [s*mdt, (s+1)*mdt) of every sublist node
// (hierarchical.py:95-120); unfinished nodes are carried to the next sublist.
template <typename D, bool W>
__global__ void __launch_bounds__(kBlock, GLB_BIN_MINB) k_hp_window(const long long* __restrict__ row,
                                                                    Relaxer<D, W> rx0, DevCtrl* ctrl,
                                                                    CtlTail tail) {
  pdl_trigger();
  __shared__ uint32_t s_wq[kBinWarps][kBinWarpQ];
  const long long n = ctrl->qcount[ctrl->in];
  if (blockIdx.x == 0 && threadIdx.x == 0 && ctrl->hp_dense) {  // k_tag_compact rebuilt the list
    if (ctrl->tag_ctr != (unsigned)n) ctrl->bm_err = 1;
    ctrl->tag_ctr = 0;
  }
  const int chunk = bin_chunk(n);
  if (blockIdx.x * (long long)kBinWarps * chunk >= n) {  // idle CTA
    ctl_tail(tail, ctrl);
    return;
  }
  timer_begin(ctrl->t_relax);
  const Relaxer<D, W> rx = bind(rx0, ctrl);
  WarpSink sink{s_wq[threadIdx.x >> 5], 0u, rx.qout, rx.nout};
  const uint32_t* __restrict__ qin = ctrl->qptr[ctrl->in];
  uint32_t* qnext = ctrl->qptr[ctrl->next];
  unsigned int* nnext = &ctrl->qcount[ctrl->next];
  const long long window = ctrl->window, mdt = ctrl->mdt;
  ThreadCounters c;
  for (long long base; (base = warp_next_chunk(ctrl, n, chunk)) >= 0;) {
    const long long i = lane_id() < (unsigned)chunk ? base + lane_id() : n;
    long long lo = 0, len = 0;
    D dn = DistTraits<D>::kInf;
    if (i < n) {
      const uint32_t u = qin[i];
      const long long r0 = row[u], r1 = row[u + 1];
      const D du = rx.dist(u);  // dn at window entry (hierarchical.py:108), in flight with the row
      const long long start = r0 + window;
      if (start < r1) {
        const long long end = start + mdt < r1 ? start + mdt : r1;
        dn = du;
        if (dn != DistTraits<D>::kInf) {
          lo = start;
          len = end - start;
        }
        if (end < r1) {  // unfinished: carry into the next sublist
          q_append(qnext, nnext, u);
          ++c.push;
        }
      }
    }
    warp_windows(rx, sink, lo, len, dn, NoMirror{}, ctrl, c);
  }
  sink.flush();
  flush_counters(ctrl, c);
  timer_end(ctrl->t_relax);
  ctl_tail(tail, ctrl);  // on only when no window can reach the CTA bin (no k_bigbin)
}

// ============================================================ NS (K9) ===
// BS over the split graph (every node's out-degree is at most mdt), each
// node's range binned like an HP window, plus child mirroring.
template <typename D, bool W>
__global__ void __launch_bounds__(kBlock, GLB_BIN_MINB) k_ns_relax(const long long* __restrict__ row,
                                                                   NsMirror mirror, Relaxer<D, W> rx0,
                                                                   DevCtrl* ctrl, CtlTail tail) {
  pdl_trigger();
  __shared__ uint32_t s_wq[kBinWarps][kBinWarpQ];
  const long long n = ctrl->qcount[ctrl->in];
  // id-ordered frontiers (as k_bs_relax): clear the in list's words unless
  // k_bm_compact rebuilt it; this step's pushes set the out list's bits
  const unsigned bm_thr = ctrl->bm_thr;
  const bool bm_valid_in = bm_thr && ctrl->bm_valid[ctrl->in];
  uint32_t* bm_clear = bm_valid_in && n < bm_thr ? ctrl->bm[ctrl->in] : nullptr;
  uint32_t* bm_out = bm_thr ? ctrl->bm[ctrl->out] : nullptr;
  if (bm_thr && blockIdx.x == 0 && threadIdx.x == 0) {
    if (bm_valid_in && n >= bm_thr && ctrl->bm_ctr != (unsigned)n) ctrl->bm_err = 1;
    ctrl->bm_ctr = 0;
    ctrl->bm_valid[ctrl->out] = 1;
  }
  const int chunk = bin_chunk(n);
  if (blockIdx.x * (long long)kBinWarps * chunk >= n) {  // idle CTA
    ctl_tail(tail, ctrl);
    return;
  }
  timer_begin(ctrl->t_relax);
  const Relaxer<D, W> rx = bind(rx0, ctrl);
  WarpSink sink{s_wq[threadIdx.x >> 5], 0u, rx.qout, rx.nout, bm_out};
  mirror.bind_bm(bm_out);
  const uint32_t* __restrict__ qin = ctrl->qptr[ctrl->in];
  ThreadCounters c;
  for (long long base; (base = warp_next_chunk(ctrl, n, chunk)) >= 0;) {
    const long long i = lane_id() < (unsigned)chunk ? base + lane_id() : n;
    long long lo = 0, len = 0;
    D dn = DistTraits<D>::kInf;
    if (i < n) {
      const uint32_t u = qin[i];
      if (bm_clear) bm_clear[u >> 5] = 0u;
      const long long r0 = row[u], r1 = row[u + 1];  // in flight with dn
      dn = rx.dist(u);
      if (dn != DistTraits<D>::kInf) {
        lo = r0;
        len = r1 - r0;
      }
    }
    warp_windows(rx, sink, lo, len, dn, mirror, ctrl, c);
  }
  sink.flush();
  flush_counters(ctrl, c);
  timer_end(ctrl->t_relax);
  ctl_tail(tail, ctrl);  // on only when no split node can reach the CTA bin (no k_bigbin)
}

// ======================================================== CTA bin (TMA) ===
// Every CTA claims 2048-edge pieces of the step's long windows by ticket; a
// piece's window is found by binary search over the windows' first pieces.
// Thread 0 claims piece i+1 and issues its bulk copies into the other buffer
// before the CTA relaxes piece i out of shared memory.
template <typename D>
struct BigPiece {
  long long lo, hi, a_lo;
  D dn;
  int valid;
};

template <typename D, bool W, class M>
__global__ void __launch_bounds__(kBlock) k_bigbin(Relaxer<D, W> rx0, M mirror, DevCtrl* ctrl,
                                                   CtlTail tail) {
  pdl_wait();
  __shared__ __align__(128) uint32_t s_col[2][kBinBuf];
  __shared__ __align__(128) uint32_t s_wt[W ? 2 : 1][W ? kBinBuf : 4];
  __shared__ __align__(8) unsigned long long s_bar[2];
  __shared__ BigPiece<D> s_pc[2];
  __shared__ uint32_t s_q[kQCap];
  __shared__ BlockQ bq;
  const unsigned long long bc = ctrl->hp_big_ctr;
  const unsigned npieces = (unsigned)bc;  // (entries << 32 | pieces)
  if (npieces == 0 || blockIdx.x >= npieces) {
    ctl_tail(tail, ctrl);
    return;
  }
  timer_begin(ctrl->t_relax);
  const Relaxer<D, W> rx = bind(rx0, ctrl);
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  // NS id-ordered frontiers: the step's pushes set the out list's bits (HP runs have bm_thr 0)
  uint32_t* bm_out = ctrl->bm_thr ? ctrl->bm[ctrl->out] : nullptr;
  mirror.bind_bm(bm_out);
  bq_init(bq, s_q, bm_out);  // barrier: the mbarriers are ready
  const unsigned long long pol = l2_evict_first();
  // thread 0: claim a piece into buffer b and start its copies
  auto claim = [&](int b) {
    const unsigned t = atomicAdd(&ctrl->hp_piece_next, 1u);
    BigPiece<D>& pc = s_pc[b];
    if (t >= npieces) {
      pc.valid = 0;
      return;
    }
    const HpBig w = ctrl->hp_big[ctrl->hp_owner[t]];
    const long long lo = w.lo + (long long)(t - w.qbase) * kBinPiece;
    const long long hi = lo + kBinPiece < w.hi ? lo + kBinPiece : w.hi;
    const long long a_lo = lo & ~3ll;  // 16-byte aligned source (arrays carry a 64 B tail pad)
    const unsigned bytes = (unsigned)(((hi - a_lo + 3) & ~3ll) * 4);
    fence_proxy_async();  // the buffer's previous contents were read by the generic proxy
    mbar_expect_tx(&s_bar[b], W ? 2 * bytes : bytes);
    bulk_g2s(s_col[b], rx.col + a_lo, bytes, &s_bar[b], pol);
    if (W) bulk_g2s(s_wt[b], rx.wt + a_lo, bytes, &s_bar[b], pol);
    pc.lo = lo;
    pc.hi = hi;
    pc.a_lo = a_lo;
    pc.dn = (D)w.dn;
    pc.valid = 1;
  };
  if (threadIdx.x == 0) claim(0);
  __syncthreads();
  ThreadCounters c;
  constexpr int K = kBinK;
  for (unsigned it = 0;; ++it) {
    const int b = (int)(it & 1u);
    if (!s_pc[b].valid) break;
    if (threadIdx.x == 0) claim(b ^ 1);  // buffer b^1 was released by the last barrier
    const long long lo = s_pc[b].lo, hi = s_pc[b].hi, a_lo = s_pc[b].a_lo;
    const D dn = s_pc[b].dn;
    mbar_wait(&s_bar[b], (it >> 1) & 1u);
    for (long long f0 = lo; f0 < hi; f0 += (long long)K * kBlock) {
      uint32_t v[K], w[K];
      D d[K];
      unsigned valid = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const long long e = f0 + (long long)k * kBlock + threadIdx.x;
        d[k] = dn;
        v[k] = 0;
        w[k] = 1u;
        if (e < hi) {
          valid |= 1u << k;
          v[k] = s_col[b][e - a_lo];
          if (W) w[k] = s_wt[b][e - a_lo];
        }
      }
      D cand[K];
      const unsigned won = relax_vals<K>(rx, bq, v, w, d, valid, c, cand);
      mirror(rx, won, v, cand, c);
    }
    bq_flush(bq, rx.qout, rx.nout);  // barriers: piece b is consumed, s_pc[b^1] is visible
  }
  flush_counters(ctrl, c);
  timer_end(ctrl->t_relax);
  ctl_tail(tail, ctrl);
}

}  // namespace glb

namespace glb {
// ====================================================== BS, warp sinks ===
// Node-based relaxation (node_based.py:43-67), thread per worklist node and
// all its out-edges, with pushes through a warp-private buffer instead of the
// CTA queue: no CTA barrier between grid-stride rounds, so warps of a CTA
// never wait for each other.  The batch loop runs to the warp's longest
// node (what SIMT execution of the per-thread loop does anyway).
template <typename D, bool W>
__global__ void __launch_bounds__(kBlock) k_bs_warp(const long long* __restrict__ row,
                                                    Relaxer<D, W> rx0, DevCtrl* ctrl,
                                                    CtlTail tail) {
  __shared__ uint32_t s_wq[kBinWarps][kBinWarpQ];
  const unsigned n = ctrl->qcount[ctrl->in];
  if (blockIdx.x * kBlock >= n) {  // idle CTA
    ctl_tail(tail, ctrl);
    return;
  }
  timer_begin(ctrl->t_relax);
  const Relaxer<D, W> rx = bind(rx0, ctrl);
  WarpSink sink{s_wq[threadIdx.x >> 5], 0u, rx.qout, rx.nout};
  const uint32_t* __restrict__ qin = ctrl->qptr[ctrl->in];
  ThreadCounters c;
  constexpr int K = 4;
  for (unsigned base = blockIdx.x * kBlock; base < n; base += gridDim.x * kBlock) {
    const unsigned i = base + threadIdx.x;
    long long lo = 0, hi = 0;
    D du = DistTraits<D>::kInf;
    if (i < n) {
      const uint32_t u = qin[i];
      du = rx.dist(u);
      if (du != DistTraits<D>::kInf) {
        lo = row[u];
        hi = row[u + 1];
      }
    }
    long long mx = hi - lo;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const long long o = __shfl_xor_sync(0xffffffffu, mx, off);
      mx = o > mx ? o : mx;
    }
    for (long long b = 0; b < mx; b += K) {
      uint32_t v[K], w[K];
      D d[K];
      unsigned valid = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const long long e = lo + b + k;
        const bool ok = e < hi;
        valid |= (unsigned)ok << k;
        const long long ek = ok ? e : 0ll;  // edge 0 is always mapped
        v[k] = __ldg(rx.col + ek);
        w[k] = W ? __ldg(rx.wt + ek) : 1u;
        d[k] = du;
      }
      D cand[K];
      relax_vals<K>(rx, sink, v, w, d, valid, c, cand);
    }
  }
  sink.flush();
  flush_counters(ctrl, c);
  timer_end(ctrl->t_relax);
  ctl_tail(tail, ctrl);
}
}  // namespace glb
