// glb_driver.cu -- strategy drivers behind glb_run (run_strategy,
// strategies/__init__.py:17-41).  Each driver restates the reference's host
// loop ("while the worklist is non-empty: launch, swap") over device-resident
// worklists; only the worklist sizes cross back to the host, once per launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "glb_internal.cuh"
#include "glb_relax.cuh"
#include "glb_scan.cuh"

namespace glb {

void split_device(glb_graph* g, long long mdt, long long totals_out[4]);
void coo_src(glb_graph* g, uint32_t* d_src);
void histogram(glb_graph* g, const long long* row, long long n, unsigned long long max_deg,
               int bins, int64_t* counts_out, int32_t* arg_max_bin, int64_t* mdt);

namespace {

constexpr int kStatRing = 64;  // LaunchStats slots cycled by the host loop

struct OverflowRestart {};  // a u32 candidate reached INF: re-run in u64

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void* ensure_zero(DevBuf& b, size_t bytes, cudaStream_t s, bool* fresh = nullptr) {
  bool grow = b.bytes < (bytes ? bytes : 16);
  void* p = ensure(b, bytes);
  if (grow) GLB_CUDA_TRY(cudaMemsetAsync(p, 0, b.bytes, s));
  if (fresh) *fresh = grow;
  return p;
}

struct HostMirror {  // pinned layout of g->host_ctrl
  DevCtrl ctrl;
  LaunchStats stats[2];
};

template <typename D, bool W>
class Runner {
 public:
  Runner(glb_graph* g, const glb_run_params& p, std::vector<glb_record>& recs)
      : g_(g), p_(p), recs_(recs), s_(g->stream) {}

  // Returns the number of output distances written to dist_out.
  void run(int64_t* dist_out, glb_run_stats* st) {
    double t_setup0 = now_ms();
    GLB_CUDA_TRY(cudaEventRecord(g_->ev[0], s_));
    n_out_ = g_->n;
    row_ = g_->row;
    col_ = g_->col;
    wt_ = g_->wt;
    n_all_ = g_->n;
    mdt_ = 0;
    const int strat = p_.strategy;
    if (strat == GLB_NS || strat == GLB_HP) {
      if (p_.mdt > 0) {
        mdt_ = p_.mdt;
      } else {
        int64_t m = 1;
        histogram(g_, g_->row, g_->n, (unsigned long long)g_->max_degree, p_.bins, nullptr,
                  nullptr, &m);
        mdt_ = m;
      }
    }
    if (strat == GLB_NS) {
      long long tot[4];
      split_device(g_, mdt_, tot);
      n_all_ = g_->n + tot[0];
      row_ = (const long long*)g_->ws.ns_row.p;
      col_ = (const uint32_t*)g_->ws.ns_col.p;
      wt_ = g_->wt ? (const uint32_t*)g_->ws.ns_w.p : nullptr;
      cs_ = (const long long*)g_->ws.ns_cs.p;
      st->num_children = tot[0];
      st->num_split_nodes = tot[3];
      st->split_fraction = g_->n ? (double)tot[3] / (double)g_->n : 0.0;
    }
    if (strat == GLB_EP) {
      src_ = (uint32_t*)ensure(g_->ws.ep_src, (size_t)std::max<long long>(g_->m, 1) * 4);
      coo_src(g_, src_);
    }
    alloc_state();
    setup_ms_ = now_ms() - t_setup0;

    switch (strat) {
      case GLB_BS: loop_node(false); break;
      case GLB_NS: loop_node(true); break;
      case GLB_EP: loop_ep(); break;
      case GLB_WD: loop_wd(); break;
      case GLB_HP: loop_hp(); break;
      default: throw Error{GLB_EINVAL, "unknown strategy"};
    }

    long long* out = (long long*)ensure(g_->ws.out64, (size_t)std::max<long long>(n_out_, 1) * 8);
    if (n_out_ > 0) {
      k_dist_out<D><<<grid_for(n_out_, kBlock, g_->num_sms * 8), kBlock, 0, s_>>>(dist_, n_out_,
                                                                                   out);
      GLB_CHECK_LAUNCH();
    }
    GLB_CUDA_TRY(cudaEventRecord(g_->ev[1], s_));
    if (n_out_ > 0 && dist_out)
      GLB_CUDA_TRY(cudaMemcpyAsync(dist_out, out, (size_t)n_out_ * 8, cudaMemcpyDeviceToHost, s_));
    GLB_CUDA_TRY(cudaStreamSynchronize(s_));
    float dev_ms = 0;
    GLB_CUDA_TRY(cudaEventElapsedTime(&dev_ms, g_->ev[0], g_->ev[1]));
    finish(st, dev_ms);
  }

 private:
  glb_graph* g_;
  const glb_run_params& p_;
  std::vector<glb_record>& recs_;
  cudaStream_t s_;
  long long n_out_ = 0, n_all_ = 0, mdt_ = 0;
  const long long* row_ = nullptr;
  const uint32_t* col_ = nullptr;
  const uint32_t* wt_ = nullptr;
  const long long* cs_ = nullptr;
  uint32_t* src_ = nullptr;
  D* dist_ = nullptr;
  uint32_t* stamp_ = nullptr;
  uint32_t* q_[4] = {nullptr, nullptr, nullptr, nullptr};
  DevCtrl* ctrl_ = nullptr;
  LaunchStats* ring_ = nullptr;
  HostMirror* h_ = nullptr;
  int ring_next_ = 0;
  double setup_ms_ = 0;
  double kernel_ms_ = 0;
  long long iterations_ = 0;
  // per-launch timing events (pairs), reused from g->ev_pool
  size_t ev_used_ = 0;

  cudaEvent_t event() {
    if (ev_used_ == g_->ev_pool.size()) {
      cudaEvent_t e;
      GLB_CUDA_TRY(cudaEventCreate(&e));
      g_->ev_pool.push_back(e);
    }
    return g_->ev_pool[ev_used_++];
  }

  void alloc_state() {
    Workspace& ws = g_->ws;
    size_t nb = (size_t)std::max<long long>(n_all_, 1);
    dist_ = (D*)ensure(ws.dist, nb * sizeof(D));
    bool fresh = false;
    stamp_ = (uint32_t*)ensure_zero(ws.stamp, nb * 4, s_, &fresh);
    if (g_->stamp_epoch > 0xF0000000u) {
      GLB_CUDA_TRY(cudaMemsetAsync(stamp_, 0, ws.stamp.bytes, s_));
      g_->stamp_epoch = 0;
    }
    if (p_.strategy == GLB_EP) {
      size_t eb = (size_t)std::max<long long>(g_->m, 1) * 4;
      q_[0] = (uint32_t*)ensure(ws.eq[0], eb);
      q_[1] = (uint32_t*)ensure(ws.eq[1], eb);
    } else {
      int nq = p_.strategy == GLB_HP ? 4 : 2;
      for (int i = 0; i < nq; ++i) q_[i] = (uint32_t*)ensure(ws.q[i], nb * 4);
    }
    ctrl_ = (DevCtrl*)ensure(ws.ctrl, sizeof(DevCtrl));
    ring_ = (LaunchStats*)ensure(ws.stats, sizeof(LaunchStats) * kStatRing);
    h_ = (HostMirror*)g_->host_ctrl;
    GLB_CUDA_TRY(cudaMemsetAsync(ctrl_, 0, sizeof(DevCtrl), s_));
    // distances: INF everywhere, then the seeds
    k_init_dist<D><<<grid_for((long long)nb, kBlock, g_->num_sms * 8), kBlock, 0, s_>>>(
        dist_, (long long)nb);
    GLB_CHECK_LAUNCH();
    long long src = p_.source;
    long long klo = 0, khi = 0, elo = 0, ehi = 0;
    bool edges = p_.strategy == GLB_EP;
    long long seeds = 1;
    if (p_.strategy == GLB_NS) {
      long long h2[2];
      GLB_CUDA_TRY(cudaMemcpyAsync(h2, cs_ + src, 16, cudaMemcpyDeviceToHost, s_));
      GLB_CUDA_TRY(cudaStreamSynchronize(s_));
      klo = g_->n + h2[0];
      khi = g_->n + h2[1];
      seeds = 1 + khi - klo;
    }
    if (edges) {
      long long h2[2];
      GLB_CUDA_TRY(cudaMemcpyAsync(h2, row_ + src, 16, cudaMemcpyDeviceToHost, s_));
      GLB_CUDA_TRY(cudaStreamSynchronize(s_));
      elo = h2[0];
      ehi = h2[1];
      seeds = ehi - elo;
    }
    seed_count_ = seeds;
    k_seed<D><<<grid_for(std::max<long long>(seeds, 1), kBlock, g_->num_sms * 4), kBlock, 0, s_>>>(
        dist_, q_[0], &ctrl_->qcount[0], src, klo, khi, elo, ehi, edges);
    GLB_CHECK_LAUNCH();
  }
  long long seed_count_ = 0;

  LaunchStats* next_slot() {
    LaunchStats* ls = ring_ + (ring_next_++ % kStatRing);
    GLB_CUDA_TRY(cudaMemsetAsync(ls, 0, sizeof(LaunchStats), s_));
    return ls;
  }

  Relaxer<D, W> relaxer(uint32_t gen, uint32_t* qout, unsigned* nout) {
    Relaxer<D, W> rx;
    rx.col = col_;
    rx.wt = wt_;
    rx.dist = dist_;
    rx.stamp = stamp_;
    rx.gen = gen;
    rx.qout = qout;
    rx.nout = nout;
    rx.ovf = &ctrl_->overflow;
    return rx;
  }

  int cap(const void* kernel) { return max_resident_blocks(kernel, kBlock, 0, g_->num_sms); }

  // Bring back the control block and the launch's counters (one round trip).
  void sync_back(LaunchStats* ls) {
    GLB_CUDA_TRY(cudaMemcpyAsync(&h_->ctrl, ctrl_, sizeof(DevCtrl), cudaMemcpyDeviceToHost, s_));
    if (ls)
      GLB_CUDA_TRY(cudaMemcpyAsync(&h_->stats[0], ls, sizeof(LaunchStats), cudaMemcpyDeviceToHost,
                                   s_));
    GLB_CUDA_TRY(cudaStreamSynchronize(s_));
    if (h_->ctrl.overflow) throw OverflowRestart{};
  }

  void add_record(int it, int sub, int tag, long long active, long long threads, cudaEvent_t k0,
                  cudaEvent_t k1, cudaEvent_t o0, cudaEvent_t o1) {
    glb_record r;
    std::memset(&r, 0, sizeof(r));
    r.iteration = it;
    r.sub_iteration = sub;
    r.tag = tag;
    r.active_items = active;
    r.threads = threads;
    const LaunchStats& ls = h_->stats[0];
    double sq = 0;
    for (int i = 0; i < kStatSlots; ++i) {
      const StatSlot& s = ls.slot[i];
      r.work_total += (int64_t)s.work;
      r.relax_ops += (int64_t)s.relax;
      r.push_ops += (int64_t)s.push;
      sq += (double)s.work_sq;
      r.work_max = std::max<int64_t>(r.work_max, (int64_t)s.work_max);
    }
    r.work_sumsq = sq;
    float ms = 0;
    if (k0 && k1 && cudaEventElapsedTime(&ms, k0, k1) == cudaSuccess) r.kernel_ms = ms;
    if (o0 && o1 && cudaEventElapsedTime(&ms, o0, o1) == cudaSuccess) r.overhead_ms = ms;
    kernel_ms_ += r.kernel_ms;
    recs_.push_back(r);
  }

  uint32_t next_gen() { return ++g_->stamp_epoch; }

  // ---------------------------------------------------------- BS / NS ---
  void loop_node(bool ns) {
    const void* kfn = ns ? (const void*)k_ns_relax<D, W> : (const void*)k_bs_relax<D, W>;
    const int kcap = std::max(cap(kfn), g_->num_sms * 8);
    int in = 0;
    long long h_in = seed_count_;
    int it = 0;
    while (h_in > 0) {
      const int out = in ^ 1;
      uint32_t gen = next_gen();
      GLB_CUDA_TRY(cudaMemsetAsync(&ctrl_->qcount[out], 0, 4, s_));
      LaunchStats* ls = next_slot();
      unsigned grid = grid_for(h_in, kBlock, kcap);
      Relaxer<D, W> rx = relaxer(gen, q_[out], &ctrl_->qcount[out]);
      cudaEvent_t k0 = event(), k1 = event();
      GLB_CUDA_TRY(cudaEventRecord(k0, s_));
      if (ns)
        k_ns_relax<D, W><<<grid, kBlock, 0, s_>>>(row_, cs_, g_->n, rx, q_[in], &ctrl_->qcount[in],
                                                  ls);
      else
        k_bs_relax<D, W><<<grid, kBlock, 0, s_>>>(row_, rx, q_[in], &ctrl_->qcount[in], ls);
      GLB_CHECK_LAUNCH();
      GLB_CUDA_TRY(cudaEventRecord(k1, s_));
      sync_back(ls);
      add_record(it, -1, ns ? GLB_NS : GLB_BS, h_in, (long long)grid * kBlock, k0, k1, nullptr,
                 nullptr);
      ev_used_ = 0;
      h_in = h_->ctrl.qcount[out];
      in = out;
      ++it;
    }
    iterations_ = it;
  }

  // --------------------------------------------------------------- EP ---
  void loop_ep() {
    const void* kfn = p_.chunked ? (const void*)k_ep_relax<D, W, true>
                                 : (const void*)k_ep_relax<D, W, false>;
    const int kcap = std::max(cap(kfn), g_->num_sms * 8);
    int in = 0;
    long long h_in = seed_count_;
    int it = 0;
    while (h_in > 0) {
      const int out = in ^ 1;
      uint32_t gen = next_gen();
      GLB_CUDA_TRY(cudaMemsetAsync(&ctrl_->qcount[out], 0, 4, s_));
      LaunchStats* ls = next_slot();
      unsigned grid = grid_for(h_in, kBlock, kcap);
      Relaxer<D, W> rx = relaxer(gen, q_[out], &ctrl_->qcount[out]);
      cudaEvent_t k0 = event(), k1 = event();
      GLB_CUDA_TRY(cudaEventRecord(k0, s_));
      if (p_.chunked)
        k_ep_relax<D, W, true><<<grid, kBlock, 0, s_>>>(row_, src_, rx, q_[in],
                                                        &ctrl_->qcount[in], ls);
      else
        k_ep_relax<D, W, false><<<grid, kBlock, 0, s_>>>(row_, src_, rx, q_[in],
                                                         &ctrl_->qcount[in], ls);
      GLB_CHECK_LAUNCH();
      GLB_CUDA_TRY(cudaEventRecord(k1, s_));
      sync_back(ls);
      add_record(it, -1, GLB_EP, h_in, (long long)grid * kBlock, k0, k1, nullptr, nullptr);
      ev_used_ = 0;
      h_in = h_->ctrl.qcount[out];
      in = out;
      ++it;
    }
    iterations_ = it;
  }

  // --------------------------------------------------------------- WD ---
  // One decomposition invocation (workload.py:75-159) over q_[in] with base
  // offset `window`, pushing improved nodes to q_[out] (stamped `gen`).
  // Returns false when the active nodes have no edges left (no record).
  bool wd_invocation(int in, long long h_in, long long window, int out, uint32_t gen, int it,
                     int sub, int tag) {
    Workspace& ws = g_->ws;
    size_t nb = (size_t)std::max<long long>(h_in, 1);
    long long* c_pre = (long long*)ensure(ws.c_pre, (size_t)std::max<long long>(n_all_, 1) * 8);
    long long* c_base = (long long*)ensure(ws.c_base, (size_t)std::max<long long>(n_all_, 1) * 8);
    uint32_t* c_node = (uint32_t*)ensure(ws.c_node, (size_t)std::max<long long>(n_all_, 1) * 4);
    long long max_tiles = (g_->m + kWdTile - 1) / kWdTile + 2;
    unsigned* tile_first = (unsigned*)ensure(ws.tile_first, (size_t)max_tiles * 4);
    long long stiles = ((long long)nb + kWdScanTile - 1) / kWdScanTile;
    long long max_stiles = (std::max<long long>(n_all_, 1) + kWdScanTile - 1) / kWdScanTile + 1;
    unsigned* flags = (unsigned*)ensure_zero(ws.scan_flags, (size_t)max_stiles * 4 + 4096, s_);
    size_t vb = (size_t)max_stiles * sizeof(Vec<2>);
    char* vals = (char*)ensure(ws.scan_vals, 2 * vb + 4096);
    LookbackState<2> lb{flags, (Vec<2>*)vals, (Vec<2>*)(vals + vb)};
    unsigned epoch = ++g_->scan_epoch;

    cudaEvent_t o0 = event(), o1 = event(), k0 = event(), k1 = event();
    GLB_CUDA_TRY(cudaEventRecord(o0, s_));
    static int scan_cap = 0;
    if (!scan_cap) scan_cap = cap((const void*)k_wd_scan);
    k_wd_scan<<<grid_for(stiles, 1, scan_cap), kBlock, 0, s_>>>(
        row_, q_[in], &ctrl_->qcount[in], window, lb, epoch, c_pre, c_base, c_node, tile_first,
        ctrl_);
    GLB_CHECK_LAUNCH();
    GLB_CUDA_TRY(cudaEventRecord(o1, s_));
    LaunchStats* ls = next_slot();
    Relaxer<D, W> rx = relaxer(gen, q_[out], &ctrl_->qcount[out]);
    static int relax_cap = 0;
    if (!relax_cap) relax_cap = cap((const void*)k_wd_relax<D, W>);
    GLB_CUDA_TRY(cudaEventRecord(k0, s_));
    k_wd_relax<D, W><<<relax_cap, kBlock, 0, s_>>>(rx, c_pre, c_base, c_node, tile_first, ctrl_, ls);
    GLB_CHECK_LAUNCH();
    GLB_CUDA_TRY(cudaEventRecord(k1, s_));
    sync_back(ls);
    if (h_->ctrl.wd_total == 0) return false;
    add_record(it, sub, tag, h_in, (long long)relax_cap * kBlock, k0, k1, o0, o1);
    return true;
  }

  void loop_wd() {
    int in = 0;
    long long h_in = seed_count_;
    int it = 0;
    while (h_in > 0) {
      const int out = in ^ 1;
      uint32_t gen = next_gen();
      GLB_CUDA_TRY(cudaMemsetAsync(&ctrl_->qcount[out], 0, 4, s_));
      bool ok = wd_invocation(in, h_in, 0, out, gen, it, -1, GLB_WD);
      ev_used_ = 0;
      if (!ok) break;  // active nodes have no out-edges (workload.py:181-183)
      h_in = h_->ctrl.qcount[out];
      in = out;
      ++it;
    }
    iterations_ = it;
  }

  // --------------------------------------------------------------- HP ---
  void loop_hp() {
    const long long thr = p_.block_size;
    const bool fb = p_.hp_fallback != 0;
    const int kcap = std::max(cap((const void*)k_hp_window<D, W>), g_->num_sms * 8);
    int sup_in = 0, sup_out = 1;
    long long h_super = seed_count_;
    int it = 0;
    while (h_super > 0) {
      uint32_t gen = next_gen();
      GLB_CUDA_TRY(cudaMemsetAsync(&ctrl_->qcount[sup_out], 0, 4, s_));
      if (fb && h_super < thr) {
        wd_invocation(sup_in, h_super, 0, sup_out, gen, it, -1, GLB_TAG_WD_FALLBACK);
      } else {
        int cur = sup_in;
        long long h_cur = h_super;
        int spare = 2;
        long long s = 0;
        while (h_cur > 0) {
          if (fb && s > 0 && h_cur < thr) {
            wd_invocation(cur, h_cur, s * mdt_, sup_out, gen, it, (int)s, GLB_TAG_WD_FALLBACK);
            break;
          }
          GLB_CUDA_TRY(cudaMemsetAsync(&ctrl_->qcount[spare], 0, 4, s_));
          LaunchStats* ls = next_slot();
          unsigned grid = grid_for(h_cur, kBlock, kcap);
          Relaxer<D, W> rx = relaxer(gen, q_[sup_out], &ctrl_->qcount[sup_out]);
          cudaEvent_t k0 = event(), k1 = event();
          GLB_CUDA_TRY(cudaEventRecord(k0, s_));
          k_hp_window<D, W><<<grid, kBlock, 0, s_>>>(row_, rx, q_[cur], &ctrl_->qcount[cur],
                                                     s * mdt_, mdt_, q_[spare],
                                                     &ctrl_->qcount[spare], ls);
          GLB_CHECK_LAUNCH();
          GLB_CUDA_TRY(cudaEventRecord(k1, s_));
          sync_back(ls);
          add_record(it, (int)s, GLB_HP, h_cur, (long long)grid * kBlock, k0, k1, nullptr,
                     nullptr);
          ev_used_ = 0;
          h_cur = h_->ctrl.qcount[spare];
          cur = spare;                   // the unfinished nodes form the next sublist
          spare = (cur == 2) ? 3 : 2;    // sublists alternate (hierarchical.py:130-133)
          ++s;
        }
      }
      ev_used_ = 0;
      // read the super-out size (already in h_ from the last sync_back)
      GLB_CUDA_TRY(cudaMemcpyAsync(&h_->ctrl, ctrl_, sizeof(DevCtrl), cudaMemcpyDeviceToHost, s_));
      GLB_CUDA_TRY(cudaStreamSynchronize(s_));
      h_super = h_->ctrl.qcount[sup_out];
      std::swap(sup_in, sup_out);
      ++it;
    }
    iterations_ = it;
  }

  void finish(glb_run_stats* st, float dev_ms) {
    st->status = GLB_OK;
    st->dist_bits = (int)(sizeof(D) * 8);
    st->iterations = iterations_;
    st->launches = (int64_t)recs_.size();
    st->mdt = mdt_;
    st->sub_iterations = 0;
    st->relax_ops = st->push_ops = st->edges_examined = st->active_items = 0;
    for (const glb_record& r : recs_) {
      if (r.tag == GLB_HP) ++st->sub_iterations;
      st->relax_ops += r.relax_ops;
      st->push_ops += r.push_ops;
      st->edges_examined += r.work_total;
      st->active_items += r.active_items;
    }
    st->device_ms = dev_ms;
    st->kernel_ms = kernel_ms_;
    st->overhead_ms = std::max(0.0, (double)dev_ms - kernel_ms_);
    st->setup_ms = setup_ms_;
    st->n_records = (int64_t)recs_.size();
  }
};

template <typename D>
void run_typed(glb_graph* g, const glb_run_params& p, int64_t* dist_out, glb_run_stats* st,
               std::vector<glb_record>& recs) {
  const bool weighted = p.algo == GLB_SSSP && g->wt != nullptr;
  if (weighted) {
    Runner<D, true> r(g, p, recs);
    r.run(dist_out, st);
  } else {
    Runner<D, false> r(g, p, recs);
    r.run(dist_out, st);
  }
}

}  // namespace

void run(glb_graph* g, const glb_run_params& p, int64_t* dist_out, glb_run_stats* st,
         std::vector<glb_record>& recs) {
  std::memset(st, 0, sizeof(*st));
  st->split_fraction = -1.0;
  if (p.dist_bits == 64) {
    run_typed<unsigned long long>(g, p, dist_out, st, recs);
    return;
  }
  try {
    run_typed<uint32_t>(g, p, dist_out, st, recs);
  } catch (const OverflowRestart&) {
    if (p.dist_bits == 32) throw Error{GLB_EOVERFLOW, "distance exceeds the 32-bit range"};
    recs.clear();
    std::memset(st, 0, sizeof(*st));
    st->split_fraction = -1.0;
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
    try {
      run_typed<unsigned long long>(g, p, dist_out, st, recs);
    } catch (const OverflowRestart&) {
      throw Error{GLB_EOVERFLOW, "distance exceeds the 63-bit range"};
    }
  }
}

}  // namespace glb

extern "C" int glb_run(glb_graph* g, const glb_run_params* params, int64_t* dist_out,
                       glb_run_stats* stats, glb_record* records, int64_t records_capacity) {
  try {
    if (!g || !params || !stats) throw glb::Error{GLB_EINVAL, "graph/params/stats is NULL"};
    const glb_run_params& p = *params;
    if (p.strategy < GLB_BS || p.strategy > GLB_HP)
      throw glb::Error{GLB_EINVAL, "unknown strategy id " + std::to_string(p.strategy)};
    if (p.algo != GLB_BFS && p.algo != GLB_SSSP)
      throw glb::Error{GLB_EINVAL, "unknown relaxation kind"};
    if (p.source < 0 || p.source >= g->n)
      throw glb::Error{GLB_EINVAL, "source " + std::to_string(p.source) + " out of range for " +
                                       std::to_string(g->n) + " nodes"};
    if ((p.strategy == GLB_NS || p.strategy == GLB_HP) && p.mdt <= 0 && p.bins < 1)
      throw glb::Error{GLB_EINVAL, "bins must be >= 1"};
    if (p.block_size < 1) throw glb::Error{GLB_EINVAL, "block_size must be >= 1"};
    if (p.dist_bits != 0 && p.dist_bits != 32 && p.dist_bits != 64)
      throw glb::Error{GLB_EINVAL, "dist_bits must be 0, 32 or 64"};
    std::memset(stats, 0, sizeof(*stats));
    if (p.strategy == GLB_EP) {
      long long required = (g->weighted ? 3 : 2) * g->m;
      if (required > p.max_cells) {  // csr.py:155-167 -> edge_based.py:41-46
        stats->status = GLB_ECOO_CAPACITY;
        stats->split_fraction = -1.0;
        return GLB_OK;
      }
      if (g->m >= (int64_t)0xFFFFFFFFll)
        throw glb::Error{GLB_EINVAL, "EP edge worklists need num_edges < 2^32"};
    }
    std::lock_guard<std::mutex> lk(g->mu);
    int prev = -1;
    cudaGetDevice(&prev);
    GLB_CUDA_TRY(cudaSetDevice(g->device));
    std::vector<glb_record> recs;
    try {
      glb::run(g, p, dist_out, stats, recs);
    } catch (...) {
      if (prev >= 0) cudaSetDevice(prev);
      throw;
    }
    if (prev >= 0) cudaSetDevice(prev);
    if (records) {
      int64_t k = std::min<int64_t>(records_capacity, (int64_t)recs.size());
      if (k > 0) std::memcpy(records, recs.data(), (size_t)k * sizeof(glb_record));
    }
    stats->n_records = (int64_t)recs.size();
    g->last_records.swap(recs);
    return GLB_OK;
  } catch (const glb::Error& e) {
    glb::set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    glb::set_error(e.what());
    return GLB_ECUDA;
  }
}

extern "C" int glb_run_records(glb_graph* g, int64_t offset, glb_record* records,
                               int64_t capacity, int64_t* written) {
  if (!g || !written || (capacity > 0 && !records) || offset < 0 || capacity < 0) {
    glb::set_error("glb_run_records: invalid argument");
    return GLB_EINVAL;
  }
  std::lock_guard<std::mutex> lk(g->mu);
  int64_t total = (int64_t)g->last_records.size();
  int64_t k = offset >= total ? 0 : std::min<int64_t>(capacity, total - offset);
  if (k > 0) std::memcpy(records, g->last_records.data() + offset, (size_t)k * sizeof(glb_record));
  *written = k;
  return GLB_OK;
}
