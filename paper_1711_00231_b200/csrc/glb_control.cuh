// glb_control.cuh -- the strategy drivers' host loops (node_based.py:33-80,
// edge_based.py:58-100, workload.py:175-189, splitting.py:129-175,
// hierarchical.py:54-136) restated as a device-side state machine.
//
// k_control_init picks the first step; k_control runs after every step: it
// turns the step's counters into a record, rotates the worklists, advances
// the stamp generation and decides the next step -- including HP's choice
// between a window sub-iteration and the WD fallback.  Under the CUDA-graph
// loop it also drives the conditional WHILE (continue?) and SWITCH (which
// step kernels?) nodes, so a whole traversal runs without the host.
#pragma once

#include "glb_internal.cuh"

namespace glb {

// Sharded runs stop at the iteration boundary (before the worklist swap) so
// the host can exchange remote updates; k_shard_advance resumes.
__device__ __forceinline__ bool ctl_pause(DevCtrl* c) {
  if (!c->shard_mode) return false;
  c->paused = 1;
  c->done = 1;
  return true;
}

__device__ __forceinline__ void ctl_simple_advance(DevCtrl* c) {
  // wl_in.clear(); swap(wl_in, wl_out)  (node_based.py:75-79)
  const unsigned produced = c->qcount[c->out];
  c->qcount[c->in] = 0;
  const int t = c->in;
  c->in = c->out;
  c->out = t;
  c->gen += 1;
  c->iteration += 1;
  c->done = produced == 0;
}

__device__ __forceinline__ void hp_end_super(DevCtrl* c);
__device__ __forceinline__ void hp_decide_sub(DevCtrl* c);

// 24-bit tier: before every generation g with g % 128 == 0 starts, all
// tags are reset to 0 (k_renorm) -- Cell<dist24_t>'s tag (g % 128) + 1 then
// grows monotonically through the next 128 generations.  The interrupted
// step resumes after it.
__device__ __forceinline__ void ctl_check_renorm(DevCtrl* c) {
  if (c->tag_bits == 8 && !c->done && (c->gen & 127u) == 0 && c->mode != kModeRenorm &&
      c->renorm_gen != c->gen) {  // once per generation (HP sub-iterations share one)
    c->saved_mode = c->mode;
    c->mode = kModeRenorm;
    c->renorm_gen = c->gen;
  }
}

// HP after a step (hierarchical.py:54-136): a WD-fallback step finishes the
// super-iteration; a window sub-iteration hands its unfinished nodes to the
// next sublist.
__device__ __forceinline__ void ctl_hp_after_step(DevCtrl* c) {
  if (c->mode == kModeWD) {
    if (c->in != c->sup_in) c->qcount[c->in] = 0;
    hp_end_super(c);
  } else {
    if (c->cur != c->sup_in) c->qcount[c->cur] = 0;
    c->cur = c->spare;
    c->spare = c->cur == 2 ? 3 : 2;
    c->s += 1;
    hp_decide_sub(c);
  }
}

// WD with fused pushes: the next step's item list is the one just appended
// (run_wd's loop, workload.py:175-189; it ends when the list has no edges,
// workload.py:181-183).
__device__ __forceinline__ void ctl_wd_fused_advance(DevCtrl* c, unsigned long long next,
                                                     unsigned zeros) {
  const unsigned items = (unsigned)(next >> 32);
  c->qcount[c->out] = items + zeros;  // the worklist length the record reports
  ctl_simple_advance(c);
  c->wd_total = (long long)(next & 0xFFFFFFFFull);
  c->wd_items = items;
  c->wd_cur ^= 1;
  c->wd_next = 0;
  c->wd_zero_next = 0;
  c->mode = kModeWDF;
  if (c->wd_total == 0) c->done = 1;
}

__device__ __forceinline__ void hp_decide_sub(DevCtrl* c);

__device__ __forceinline__ void hp_begin_super(DevCtrl* c) {
  c->qcount[c->sup_out] = 0;
  const unsigned n = c->qcount[c->sup_in];
  if (c->hp_fallback && (long long)n < c->hp_threshold) {  // hierarchical.py:55-61
    c->mode = kModeWD;
    c->tag = GLB_TAG_WD_FALLBACK;
    c->in = c->sup_in;
    c->out = c->sup_out;
    c->window = 0;
    c->sub = -1;
  } else {
    c->cur = c->sup_in;
    c->spare = 2;
    c->s = 0;
    hp_decide_sub(c);
  }
}

__device__ __forceinline__ void hp_end_super(DevCtrl* c) {
  if (ctl_pause(c)) return;
  // super_in.clear(); swap(super_in, super_out)  (hierarchical.py:134-137)
  const unsigned produced = c->qcount[c->sup_out];
  c->qcount[c->sup_in] = 0;
  const int t = c->sup_in;
  c->sup_in = c->sup_out;
  c->sup_out = t;
  c->gen += 1;
  c->iteration += 1;
  if (produced == 0) {
    c->done = 1;
    c->mode = kModeDone;
  } else {
    hp_begin_super(c);
  }
}

__device__ __forceinline__ void hp_decide_sub(DevCtrl* c) {
  const unsigned n = c->qcount[c->cur];
  if (n == 0) {
    hp_end_super(c);
    return;
  }
  c->in = c->cur;
  c->out = c->sup_out;
  c->window = c->s * c->mdt;
  c->sub = (int)c->s;
  if (c->hp_fallback && c->s > 0 && (long long)n < c->hp_threshold) {  // hierarchical.py:67-81
    c->mode = kModeWD;
    c->tag = GLB_TAG_WD_FALLBACK;
  } else {
    c->mode = kModeHP;
    c->tag = GLB_HP;
    c->next = c->spare;
    c->qcount[c->spare] = 0;
  }
}

// WD over a frontier holding at least 1/dense_ok of the nodes scans the
// cells in id order (packed cells only: the generation marks the worklist).
// 24-bit tier: not right after a renormalisation (it reset the in list's tags).
// HP: the same for the super-list a window sub-iteration 0 reads (k_tag_compact).
__device__ __forceinline__ void ctl_choose_dense(DevCtrl* c) {
  const bool tags = c->dense_ok && (c->tag_bits == 32 || (c->tag_bits == 8 && c->renorm_gen != c->gen)) &&
                    !c->use_small && (long long)c->qcount[c->in] * c->dense_ok >= c->n_nodes;
  c->wd_dense = tags && c->strategy == GLB_WD && c->mode == kModeWD;
  c->hp_dense = tags && c->strategy == GLB_HP && c->mode == kModeHP && c->s == 0;
}

__device__ __forceinline__ int ctl_step_kind(const DevCtrl* c) {
  return c->use_small ? (int)kModeSmall : c->mode;
}

// The loop graph's WHILE body chains kGraphUnroll SWITCH nodes (one step
// each); every step's control sets all of their handles to the next step's
// kind, so whichever SWITCH runs next picks it up (a finished run selects
// kModeDone, which has no branch, for the rest of the body).
constexpr int kGraphUnroll = 4;
struct ModeHandles {
  cudaGraphConditionalHandle h[kGraphUnroll];
};

__device__ __forceinline__ void ctl_set_conditionals(DevCtrl* c, cudaGraphConditionalHandle h_loop,
                                                     const ModeHandles& h_mode,
                                                     int graph_mode) {
  if (graph_mode) {
    cudaGraphSetConditional(h_loop, c->done ? 0u : 1u);
    const unsigned kind = (unsigned)ctl_step_kind(c);
#pragma unroll
    for (int u = 0; u < kGraphUnroll; ++u)
      if (h_mode.h[u]) cudaGraphSetConditional(h_mode.h[u], kind);
  }
}

// Small-frontier steps that k_small_loop (glb_small.cuh) can run: BS / NS
// node steps, WD steps, and HP's super-list WD-fallback.
constexpr int kSmallItemsCtl = 8192;
#ifndef GLB_SMALL_EDGES
#define GLB_SMALL_EDGES 16384
#endif
constexpr long long kSmallEdgesCtl = GLB_SMALL_EDGES;  // WD: active edges one cluster iteration takes
constexpr long long kSmallMaxWindow = 64;   // HP: thread-per-node windows the cluster walks
constexpr long long kSmallHpEdgesCtl = 16384;  // HP: window edges (items x mdt) of a cluster step
constexpr long long kSmallNsMaxDeg = 1024;  // NS: split-node degree (mdt) a cluster thread walks
constexpr unsigned kSmallListCtl = 32768;    // BS / NS / EP / HP-window worklists (no item table)
__device__ __forceinline__ bool small_eligible(const DevCtrl* c) {
  if (!c->small_ok || c->done || c->shard_mode) return false;
  const bool table = c->mode == kModeWD || c->mode == kModeWDF;  // WD builds an smem item table
  if (c->qcount[c->in] > (table ? (unsigned)kSmallItemsCtl : kSmallListCtl)) return false;
  switch (c->strategy) {
    case GLB_BS:
    case GLB_EP:
      return c->mode == kModeRelax;
    case GLB_NS:  // thread-per-node in the cluster: only while split nodes are short
      return c->mode == kModeRelax && c->mdt <= kSmallNsMaxDeg;
    case GLB_WD:
      return c->mode == kModeWD || (c->mode == kModeWDF && c->wd_total <= kSmallEdgesCtl);
    case GLB_HP:  // WD-fallback steps, and window sub-iterations of few, short windows
      // (a cluster thread walks its window serially: thousands of mdt-long
      // windows are a long chain per thread there, the grid kernel spreads them)
      return c->mode == kModeWD ||
             (c->mode == kModeHP && c->mdt <= kSmallMaxWindow &&
              (long long)c->qcount[c->in] * c->mdt <= kSmallHpEdgesCtl);
    default:
      return false;
  }
}

// Slots of the per-thread work list of the record being written; -1 when the
// run is not instrumented or the list buffer is full.
__device__ __forceinline__ long long ctl_ptw_take(DevCtrl* c, unsigned long long threads) {
  if (!c->ptw) return -1;
  const unsigned long long off = c->ptw_off;
  c->ptw_off = off + threads;
  return off + threads <= c->ptw_cap ? (long long)off : -1;
}

__device__ __forceinline__ void ctl_reset_timers(DevCtrl* c) {
  c->t_relax.start = c->t_scan.start = ~0ull;
  c->t_relax.end = c->t_scan.end = 0;
  c->scan_ticket = c->relax_ticket = 0;
  c->hp_big_ctr = 0;
  c->hp_piece_next = 0;
}

// The host has written the static fields (qptr, strategy, mdt, thresholds,
// thread counts, record buffer, stamp generation base, scan epoch) and the
// seed kernel has filled list 0.
__global__ void k_control_init(DevCtrl* c, cudaGraphConditionalHandle h_loop,
                               ModeHandles h_mode, int graph_mode) {
  if (threadIdx.x != 0) return;
  const int strategy = c->strategy;
  c->in = 0;
  c->out = 1;
  c->next = 2;
  c->qcount[1] = c->qcount[2] = c->qcount[3] = 0;
  c->gen += 1;
  c->iteration = 0;
  c->sub = -1;
  c->window = 0;
  c->done = c->qcount[0] == 0;
  c->nrec = 0;
  ctl_reset_timers(c);
  switch (strategy) {
    case GLB_WD:
      c->mode = kModeWD;
      c->tag = GLB_WD;
      break;
    case GLB_HP:
      c->sup_in = 0;
      c->sup_out = 1;
      hp_begin_super(c);
      break;
    default:
      c->mode = kModeRelax;
      c->tag = strategy;
      break;
  }
  if (c->shard_mode) c->done = 0;  // every shard steps, even with an empty frontier
  if (c->done) c->mode = kModeDone;
  c->small_exit = 0;
  c->kernels = 1;
  c->tail_done = 0;
  ctl_check_renorm(c);
  c->use_small = small_eligible(c);
  ctl_set_conditionals(c, h_loop, h_mode, graph_mode);
}

// One warp: reduce the step's counters into a record, then transition.
// `fused`: running as the tail of the step's last kernel (ctl_tail), so no
// control kernel of its own was launched.
__device__ __forceinline__ void control_warp(DevCtrl* c, cudaGraphConditionalHandle h_loop,
                                             const ModeHandles& h_mode, int graph_mode,
                                             int fused) {
  const unsigned lane = threadIdx.x & 31u;
  StatSlot& sl = c->ls->slot[lane];
  unsigned long long w = __ldcg(&sl.work), r = __ldcg(&sl.relax), p = __ldcg(&sl.push),
                     mx = __ldcg(&sl.work_max);
  double sq = (double)__ldcg(&sl.work_sq);
  sl.work = sl.relax = sl.push = sl.work_sq = sl.work_max = 0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    w += __shfl_xor_sync(0xffffffffu, w, off);
    r += __shfl_xor_sync(0xffffffffu, r, off);
    p += __shfl_xor_sync(0xffffffffu, p, off);
    sq += __shfl_xor_sync(0xffffffffu, sq, off);
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = o > mx ? o : mx;
  }
  if (lane != 0) return;
  // this control kernel + the step's kernels (WD: scan + relax)
  // (two-kernel steps: WD scan + relax, HP window + CTA bin, NS relax + CTA bin)
  // (+1: the id-ordered frontier compaction before a BS / NS relax step)
  const bool two = c->mode == kModeWD ||
                   (c->bins_two && (c->mode == kModeHP ||
                                    (c->mode == kModeRelax && c->strategy == GLB_NS)));
  // (+1: HP window steps of a run with id-ordered super-lists start with k_tag_compact)
  const int bm = (c->bm_thr && c->mode == kModeRelax) ||
                 (c->dense_ok && c->strategy == GLB_HP && c->mode == kModeHP) ? 1 : 0;
  c->kernels += (c->small_exit || c->done ? 2 : (two ? 3 : 2) + bm) - (fused ? 1 : 0);
  const unsigned long long wd_next = c->wd_next;
  const unsigned wd_zero = c->wd_zero_next;
  if (c->small_exit) {  // k_small_loop recorded and advanced its own iterations
    c->small_exit = 0;
    c->use_small = 0;
    ctl_choose_dense(c);
    ctl_set_conditionals(c, h_loop, h_mode, graph_mode);
    return;
  }
  if (c->mode == kModeRenorm) {  // cells retagged: resume the interrupted step
    c->mode = c->saved_mode;
    c->use_small = small_eligible(c);
    ctl_choose_dense(c);
    ctl_set_conditionals(c, h_loop, h_mode, graph_mode);
    return;
  }
  if (c->done) {  // nothing ran (already finished)
    ctl_set_conditionals(c, h_loop, h_mode, graph_mode);
    return;
  }
  const bool wd_empty = (c->mode == kModeWD || c->mode == kModeWDF) && c->wd_total == 0;
  if (!wd_empty && c->nrec < c->rec_cap) {  // decompose_invocation returns None: no record
    DevRecord& rec = c->recs[c->nrec];
    rec.iteration = c->iteration;
    rec.sub = c->sub;
    rec.tag = c->tag;
    rec.active = c->qcount[c->in];
    rec.threads = c->mode == kModeHP ? c->hp_threads : c->relax_threads;
    rec.work = (long long)w;
    rec.relax = (long long)r;
    rec.push = (long long)p;
    rec.work_max = (long long)mx;
    rec.work_sumsq = sq;
    rec.k0 = c->t_relax.start;
    rec.k1 = c->t_relax.end;
    rec.o0 = c->mode == kModeWD ? c->t_scan.start : 0;
    rec.o1 = c->mode == kModeWD ? c->t_scan.end : 0;
    rec.ptw_off = ctl_ptw_take(c, (unsigned long long)rec.threads);
  }
  if (!wd_empty) c->nrec += 1;
  if (c->mode == kModeWD) c->scan_epoch += 1;
  ctl_reset_timers(c);
  switch (c->strategy) {
    case GLB_WD:
      if (ctl_pause(c)) break;
      if (wd_empty) {  // active nodes have no out-edges (workload.py:181-183)
        c->done = 1;
      } else if (c->wd_fused) {
        ctl_wd_fused_advance(c, wd_next, wd_zero);
      } else {
        ctl_simple_advance(c);
        c->mode = kModeWD;  // a relax-only step on the cluster loop's item list pushed nodes
      }
      break;
    case GLB_HP:
      ctl_hp_after_step(c);
      break;
    default:
      if (!ctl_pause(c)) ctl_simple_advance(c);
      break;
  }
  if (c->done && !c->paused) c->mode = kModeDone;
  ctl_check_renorm(c);
  c->use_small = small_eligible(c);
  ctl_choose_dense(c);
  ctl_set_conditionals(c, h_loop, h_mode, graph_mode);
}

__global__ void k_control(DevCtrl* c, cudaGraphConditionalHandle h_loop, ModeHandles h_mode,
                          int graph_mode) {
  control_warp(c, h_loop, h_mode, graph_mode, 0);
}

// Control fused into the step's last kernel (graph loop): every CTA counts
// itself out; the last one copies the control block into shared memory
// (L2 reads: its L1 may hold lines from the kernel's start), runs
// control_warp on the copy and writes it back.  Saves the k_control launch
// of every iteration.  All threads of the CTA call it (CTA-uniform exits).
struct CtlTail {
  cudaGraphConditionalHandle h_loop;
  ModeHandles h_mode;
  int on;
};

__device__ __noinline__ void ctl_tail_last(const CtlTail& t, DevCtrl* g) {
  __shared__ __align__(16) DevCtrl s_ctl;
  constexpr unsigned kWords = sizeof(DevCtrl) / 8;
  static_assert(sizeof(DevCtrl) % 8 == 0, "DevCtrl is copied in 8-byte words");
  __threadfence();
  for (unsigned i = threadIdx.x; i < kWords; i += blockDim.x)
    reinterpret_cast<unsigned long long*>(&s_ctl)[i] =
        __ldcg(reinterpret_cast<const unsigned long long*>(g) + i);
  __syncthreads();
  if (threadIdx.x < 32) control_warp(&s_ctl, t.h_loop, t.h_mode, 1, 1);
  __syncthreads();
  if (threadIdx.x == 0) s_ctl.tail_done = 0;
  __syncthreads();
  for (unsigned i = threadIdx.x; i < kWords; i += blockDim.x)
    reinterpret_cast<unsigned long long*>(g)[i] = reinterpret_cast<unsigned long long*>(&s_ctl)[i];
}

__device__ __forceinline__ void ctl_tail(const CtlTail& t, DevCtrl* g) {
  if (!t.on) return;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    s_last = atomicAdd(&g->tail_done, 1u) == total - 1u;
  }
  __syncthreads();
  if (s_last) ctl_tail_last(t, g);
}


// Resume a paused sharded run: the deferred worklist swap / super-iteration
// switch.  Global termination is the host's all-reduce, not `produced`.
__global__ void k_shard_advance(DevCtrl* c) {
  if (threadIdx.x != 0) return;
  c->paused = 0;
  c->done = 0;
  if (c->strategy == GLB_HP) {
    c->qcount[c->sup_in] = 0;
    const int t = c->sup_in;
    c->sup_in = c->sup_out;
    c->sup_out = t;
    c->gen += 1;
    c->iteration += 1;
    hp_begin_super(c);
  } else {
    ctl_simple_advance(c);
    c->done = 0;
    c->mode = c->strategy == GLB_WD ? kModeWD : kModeRelax;
    c->tag = c->strategy;
    c->sub = -1;
    c->window = 0;
  }
  ctl_check_renorm(c);  // 24-bit tier: retag before every 128th generation
}

// Re-enter the loop graph of a sharded run after the exchange (the state
// k_shard_advance left), instead of k_control_init's fresh start.
__global__ void k_control_resume(DevCtrl* c, cudaGraphConditionalHandle h_loop, ModeHandles h_mode,
                                 int graph_mode) {
  if (threadIdx.x != 0) return;
  c->kernels += 1;
  c->tail_done = 0;
  c->use_small = small_eligible(c);
  ctl_set_conditionals(c, h_loop, h_mode, graph_mode);
}

}  // namespace glb
