// glb_driver.cu -- glb_run (run_strategy, strategies/__init__.py:17-41).
//
// A run = per-run preprocessing (histogram/MDT, split, COO: the reference's
// "setup overhead"), distance init + seed, then the strategy loop, then the
// int64 distances.  The loop is the device state machine of glb_control.cuh
// driven either
//   * by the host (GLB_LOOP_HOST): launch the step's kernels + k_control,
//     read the control block back, repeat -- exact per-launch CUDA events; or
//   * by the device (GLB_LOOP_GRAPH): one CUDA graph whose conditional WHILE
//     node repeats [step kernels, k_control] and whose SWITCH node picks the
//     HP step kind, so the host launches the whole traversal once.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <unordered_map>
#include <memory>
#include <mutex>
#include <vector>

#include "glb_control.cuh"
#include "glb_internal.cuh"
#include "glb_bins.cuh"
#include "glb_relax.cuh"
#include "glb_scan.cuh"
#include "glb_small.cuh"
#include "glb_peer.cuh"

namespace glb {

void split_device(glb_graph* g, long long mdt, long long totals_out[4]);
void coo_src(glb_graph* g, uint32_t* d_src);
void histogram(glb_graph* g, const long long* row, long long n, unsigned long long max_deg,
               int bins, int64_t* counts_out, int32_t* arg_max_bin, int64_t* mdt);

namespace {

constexpr unsigned kMaxRecords = 1u << 16;
constexpr unsigned kBmThrDefault = 32768;  // BS lists rebuilt in id order from this size
constexpr unsigned long long kPtwCap = 1ull << 27;  // per-thread work slots of one run (512 MB)

// a narrow candidate reached INF: re-run at the next distance tier.  Derived
// from std::exception so no C-ABI guard can let it escape an extern "C" call.
struct OverflowRestart : std::exception {
  const char* what() const noexcept override { return "distance overflow"; }
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}


struct HostMirror {  // pinned layout of g->host_ctrl
  DevCtrl ctrl;
};

template <typename D, bool W>
class Runner {
 public:
  Runner(glb_graph* g, const glb_run_params& p, std::vector<glb_record>& recs)
      : g_(g), p_(p), recs_(recs), s_(g->stream) {}

  void run(int64_t* dist_out, glb_run_stats* st) {
    {
      NvtxRange r("glb setup (histogram/MDT, split, COO, init)");
      prepare(st);
    }
    {
      NvtxRange r(p_.loop_mode == GLB_LOOP_GRAPH ? "glb traversal (graph loop)"
                                                  : "glb traversal (host loop)");
      if (p_.loop_mode == GLB_LOOP_GRAPH)
        loop_graph();
      else
        loop_host();
    }
    NvtxRange r("glb distances + records to host");
    finish_run(dist_out, st, 0, g_->n);
  }

 protected:
  // per-run preprocessing + state (the reference's "setup overhead")
  void prepare(glb_run_stats* st) {
    const double t0 = now_ms();
    GLB_CUDA_TRY(cudaEventRecord(g_->ev[0], s_));
    n_out_ = g_->n;
    row_ = g_->row;
    col_ = g_->col;
    wt_ = g_->wt;
    n_all_ = g_->n;
    const int strat = p_.strategy;
    if (strat == GLB_NS || strat == GLB_HP) {  // splitting.py:112-113, hierarchical.py:38-39
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
    if (strat == GLB_EP) {  // csr_to_coo inside run_ep (edge_based.py:41)
      src_ = (uint32_t*)ensure(g_->ws.ep_src, (size_t)std::max<long long>(g_->m, 1) * 4);
      coo_src(g_, src_);
    }
    alloc_state();
    setup_ms_ = now_ms() - t0;
  }

  // distances of ids [lo, hi) to the host, counters into records / stats
  void finish_run(int64_t* dist_out, glb_run_stats* st, long long lo, long long hi) {
    const long long cnt = std::max<long long>(hi - lo, 0);
    // 32-bit distances travel as u32 and are widened by the host workers;
    // 64-bit ones are widened to the int64 layout on the device
    constexpr bool kNarrow = sizeof(D) == 4;
    void* out = ensure(g_->ws.out64, (size_t)std::max<long long>(cnt, 1) * (kNarrow ? 4 : 8));
    if (cnt && dist_out) {
      if (kNarrow)
        k_dist_u32<D><<<grid_for(cnt, kBlock, g_->num_sms * 8), kBlock, 0, s_>>>(
            cells_ + lo, cnt, (uint32_t*)out);
      else
        k_dist_out<D><<<grid_for(cnt, kBlock, g_->num_sms * 8), kBlock, 0, s_>>>(
            cells_ + lo, cnt, (long long*)out);
      GLB_CHECK_LAUNCH();
    }
    GLB_CUDA_TRY(cudaEventRecord(g_->ev[1], s_));
    GLB_CUDA_TRY(cudaMemcpyAsync(&h_->ctrl, ctrl_, sizeof(DevCtrl), cudaMemcpyDeviceToHost, s_));
    GLB_CUDA_TRY(cudaStreamSynchronize(s_));
    if (p_.loop_mode == GLB_LOOP_GRAPH) count_launches(h_->ctrl.kernels);
    if (h_->ctrl.overflow) throw OverflowRestart{};
    if (h_->ctrl.bm_err) throw Error{GLB_ECUDA, "frontier bitmap out of step with its worklist"};
    if (cnt > 0 && dist_out) {
      if (kNarrow)
        download_dist_u32(s_, (const uint32_t*)out, cnt, dist_out);
      else
        GLB_CUDA_TRY(cudaMemcpy(dist_out, out, (size_t)cnt * 8, cudaMemcpyDeviceToHost));
    }
    g_->ptw_len = ptw_ ? (long long)std::min<unsigned long long>(h_->ctrl.ptw_off, kPtwCap) : 0;
    if (ptw_) g_->ptw_dirty = g_->ptw_len;
    g_->stamp_epoch = h_->ctrl.gen;
    g_->scan_epoch = h_->ctrl.scan_epoch;
    float dev_ms = 0;
    GLB_CUDA_TRY(cudaEventElapsedTime(&dev_ms, g_->ev[0], g_->ev[1]));
    collect_records();
    finish(st, dev_ms);
  }

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
  CellS<D>* cells_ = nullptr;
  uint32_t* stamp_ = nullptr;
  uint32_t* ptw_ = nullptr;
  uint32_t* q_[4] = {nullptr, nullptr, nullptr, nullptr};
  DevCtrl* ctrl_ = nullptr;
  LaunchStats* ls_ = nullptr;
  DevRecord* drecs_ = nullptr;
  HostMirror* h_ = nullptr;
  // WD workspace
  HpBig* hp_big_ = nullptr;
  unsigned* hp_owner_ = nullptr;
  WdItem* items_[2] = {nullptr, nullptr};
  unsigned* tile_first_[2] = {nullptr, nullptr};
  LookbackState<2> lb_{};
  // grids
  int cap_relax_ = 0, cap_scan_ = 0, cap_wd_ = 0, cap_hp_ = 0, cap_big_ = 0;
  // graph loop: the control step runs as the tail of each step's last kernel
  CtlTail tail_{0, {}, 0};
  bool fused_ctl_ = getenv("GLB_NO_FUSED_CTL") == nullptr;
  bool pdl_ = getenv("GLB_NO_PDL") == nullptr;
  // BS pushes through warp buffers (k_bs_warp): C2 SSSP BS -10 %, BFS -17 %, but
  // C3 SSSP +12 % (the CTA queue wins on degree-4 grids), so opt-in
  bool bs_warp_ = getenv("GLB_BS_WARP") != nullptr;
  // BS / NS id-ordered frontiers (k_bm_compact) for relax steps of >= bm_thr_
  // nodes (and >= 1/256 of the graph); GLB_BM_THR=t sets the threshold to t
  // exactly, GLB_BM_THR=0 turns them off
  unsigned bm_thr_ = getenv("GLB_BM_THR") ? (unsigned)atoll(getenv("GLB_BM_THR")) : kBmThrDefault;
  uint32_t* bm_[2] = {nullptr, nullptr};
  bool hp_dense_ = false;  // HP window steps start with k_tag_compact
  int small_ctas_ = kSmallCtas;  // cluster loop CTAs (8 or 16)
  uint32_t* ep_dn_[2] = {nullptr, nullptr};  // EP carried source levels (unweighted)
  long long bm_vec_ = 0;
  bool bm_on() const {
    return ((p_.strategy == GLB_BS && !bs_warp_) || p_.strategy == GLB_NS) && !shard_mode_ && bm_thr_ > 0;
  }
  int unroll_ = getenv("GLB_GRAPH_UNROLL") ? std::max(1, std::min(kGraphUnroll, atoi(getenv("GLB_GRAPH_UNROLL"))))
                                           : kGraphUnroll;
  double setup_ms_ = 0;
  long long seed_count_ = 0;
  bool shard_mode_ = false;
  bool resume_graph_ = false;  // the loop graph starts with k_control_resume
  // host-loop per-record event timing
  struct EvPair {
    cudaEvent_t k0, k1, o0, o1;
    long long threads;
  };
  std::vector<EvPair> ev_of_rec_;
  size_t ev_used_ = 0;

  cudaEvent_t event() {
    while (ev_used_ >= g_->ev_pool.size()) {
      cudaEvent_t e;
      GLB_CUDA_TRY(cudaEventCreate(&e));
      g_->ev_pool.push_back(e);
    }
    return g_->ev_pool[ev_used_++];
  }

  int cap(const void* kernel) { return max_resident_blocks(kernel, kBlock, 0, g_->num_sms); }

  const void* relax_kernel() const {
    switch (p_.strategy) {
      case GLB_BS:
        return bs_warp_ ? (const void*)k_bs_warp<D, W> : (const void*)k_bs_relax<D, W>;
      case GLB_NS: return (const void*)k_ns_relax<D, W>;
      case GLB_EP:
        return p_.chunked ? (const void*)k_ep_relax<D, W, true> : (const void*)k_ep_relax<D, W, false>;
      default: return nullptr;
    }
  }

  void alloc_state() {
    Workspace& ws = g_->ws;
    const size_t nb = (size_t)std::max<long long>(n_all_, 1);
    cells_ = (CellS<D>*)ensure(ws.dist, nb * sizeof(CellS<D>));
    stamp_ = (uint32_t*)ensure_zero(ws.stamp, nb * 4, s_);
    if (g_->stamp_epoch > 0xF0000000u) {
      GLB_CUDA_TRY(cudaMemsetAsync(stamp_, 0, ws.stamp.bytes, s_));
      g_->stamp_epoch = 0;
    }
    if (p_.strategy == GLB_EP) {
      const size_t eb = (size_t)std::max<long long>(g_->m, 1) * 4;
      q_[0] = (uint32_t*)ensure(ws.eq[0], eb);
      q_[1] = (uint32_t*)ensure(ws.eq[1], eb);
      ep_dn_[0] = ep_dn_[1] = nullptr;
      // carried levels skip the pre-check, which on R-MAT tails filters most
      // atomics (C1 BFS EP +18 %, C2 +5 %); on low-degree, high-diameter
      // graphs the shorter chain wins (C3 BFS EP 51.8 -> 49.1 ms): average
      // out-degree <= 8 only (GLB_EP_CARRY=0/1 forces)
      const char* ec = getenv("GLB_EP_CARRY");
      const bool carry = ec ? atoi(ec) != 0 : g_->m <= 8 * g_->n;
      if (!W && sizeof(D) == 4 && !shard_mode_ && carry) {  // levels fit u32
        ep_dn_[0] = (uint32_t*)ensure(ws.ep_dn[0], eb);
        ep_dn_[1] = (uint32_t*)ensure(ws.ep_dn[1], eb);
      }
      q_[2] = q_[3] = q_[1];
    } else {
      for (int i = 0; i < 4; ++i)
        q_[i] = (i < 2 || p_.strategy == GLB_HP) ? (uint32_t*)ensure(ws.q[i], nb * 4) : q_[1];
    }
    bm_[0] = bm_[1] = nullptr;
    if (bm_on()) {  // two member bitmaps, 16-byte vectors, zeroed per run
      bm_vec_ = ((long long)nb + 127) / 128;  // words / 4 (16-byte aligned halves)
      char* b = (char*)ensure(ws.bm, (size_t)bm_vec_ * 32);
      GLB_CUDA_TRY(cudaMemsetAsync(b, 0, (size_t)bm_vec_ * 32, s_));
      bm_[0] = (uint32_t*)b;
      bm_[1] = (uint32_t*)(b + (size_t)bm_vec_ * 16);
    }
    if (p_.strategy == GLB_WD || p_.strategy == GLB_HP) {
      items_[0] = (WdItem*)ensure(ws.wd_items[0], nb * sizeof(WdItem));
      items_[1] = (WdItem*)ensure(ws.wd_items[1], nb * sizeof(WdItem));
      const long long max_tiles = (g_->m + kWdTile - 1) / kWdTile + 2;
      tile_first_[0] = (unsigned*)ensure(ws.wd_tiles[0], (size_t)max_tiles * 4);
      tile_first_[1] = (unsigned*)ensure(ws.wd_tiles[1], (size_t)max_tiles * 4);
      const long long stiles = ((long long)nb + kWdScanTile - 1) / kWdScanTile + 1;
      unsigned* flags = (unsigned*)ensure_zero(ws.scan_flags, (size_t)stiles * 4 + 4096, s_);
      const size_t vb = (size_t)stiles * sizeof(Vec<2>);
      char* vals = (char*)ensure(ws.scan_vals, 2 * vb + 4096);
      lb_ = LookbackState<2>{flags, (Vec<2>*)vals, (Vec<2>*)(vals + vb)};
      cap_scan_ = cap((const void*)k_wd_scan<D>);
      cap_wd_ = cap((const void*)k_wd_relax<D, W>);
    }
    if (p_.strategy == GLB_HP)
      cap_hp_ = std::max(cap((const void*)k_hp_window<D, W>), g_->num_sms);
    if (p_.strategy == GLB_HP || p_.strategy == GLB_NS) {
      // CTA-bin entries: every long window holds >= kBinCtaMin edges
      const size_t entries = (size_t)g_->m / kBinCtaMin + 64;
      const size_t pieces = entries + (size_t)g_->m / kBinPiece + 64;
      hp_big_ = (HpBig*)ensure(ws.hp_big, entries * sizeof(HpBig) + pieces * 4);
      hp_owner_ = reinterpret_cast<unsigned*>(hp_big_ + entries);
      cap_big_ = std::max(p_.strategy == GLB_HP ? cap((const void*)k_bigbin<D, W, NoMirror>)
                                                : cap((const void*)k_bigbin<D, W, NsMirror>),
                          g_->num_sms);
    }
    // Cluster loop size: 16 CTAs (non-portable) for EP / HP -- C3 BFS EP
    // 58.8 -> 52.6 ms, C2 SSSP / BFS HP -2 / -3 % -- and for WD on graphs of
    // average out-degree <= 8 (C3 BFS WD 94.3 -> 85.0, SSSP 482 -> 461; on
    // R-MAT C2 BFS WD +2.7 %, so 8 there); 8 for BS / NS (C3 SSSP BS +2.4 %
    // at 16).  GLB_SMALL_CTAS=8|16 overrides.  16 needs the GPU to
    // co-schedule a 16-CTA cluster; otherwise 8.
    {
      const char* e = getenv("GLB_SMALL_CTAS");
      const bool wd16 = p_.strategy == GLB_WD && g_->m <= 8 * g_->n;
      int want = e ? atoi(e) : (p_.strategy == GLB_EP || p_.strategy == GLB_HP || wd16 ? 16 : kSmallCtas);
      if (want != 16) want = 8;
      GLB_CUDA_TRY(cudaFuncSetAttribute((const void*)k_small_loop<D, W, 8>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)small_smem_bytes<D>()));
      if (want == 16) {
        const void* k16 = (const void*)k_small_loop<D, W, 16>;
        int nclusters = 0;
        if (cudaFuncSetAttribute(k16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
            cudaFuncSetAttribute(k16, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)small_smem_bytes<D>()) == cudaSuccess) {
          cudaLaunchConfig_t lc = {};
          lc.gridDim = dim3(16);
          lc.blockDim = dim3(kSmallThreads);
          lc.dynamicSmemBytes = small_smem_bytes<D>();
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = 16;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          lc.attrs = at;
          lc.numAttrs = 1;
          if (cudaOccupancyMaxActiveClusters(&nclusters, k16, &lc) != cudaSuccess) nclusters = 0;
        }
        cudaGetLastError();
        if (nclusters < 1) want = 8;
      }
      small_ctas_ = want;
    }
    if (relax_kernel()) cap_relax_ = std::max(cap(relax_kernel()), g_->num_sms);
    pin_cells_in_l2(nb * sizeof(CellS<D>));
    ptw_ = nullptr;
    if (p_.instrument) {  // per-thread work lists: zeroed once, atomically accumulated
      // The list is accumulated with atomics, so it must start zeroed; only
      // the prefix the previous instrumented run used is dirty (a fresh or
      // recycled buffer is zeroed whole).
      const void* before = ws.ptw.p;
      ptw_ = (uint32_t*)ensure(ws.ptw, (size_t)kPtwCap * 4);
      const long long dirty = (before != ws.ptw.p || g_->ptw_dirty < 0) ? (long long)kPtwCap
                                                                         : g_->ptw_dirty;
      if (dirty > 0) GLB_CUDA_TRY(cudaMemsetAsync(ptw_, 0, (size_t)dirty * 4, s_));
      g_->ptw_dirty = -1;  // unknown until this run finishes
    }
    ctrl_ = (DevCtrl*)ensure(ws.ctrl, sizeof(DevCtrl));
    ls_ = (LaunchStats*)ensure_zero(ws.stats, sizeof(LaunchStats), s_);
    drecs_ = (DevRecord*)ensure(ws.recs, sizeof(DevRecord) * kMaxRecords);
    h_ = (HostMirror*)g_->host_ctrl;

    // static fields of the control block
    DevCtrl c;
    std::memset(&c, 0, sizeof(c));
    for (int i = 0; i < 4; ++i) c.qptr[i] = q_[i];
    c.strategy = p_.strategy;
    c.mdt = mdt_;
    c.hp_threshold = p_.block_size;
    c.hp_fallback = p_.hp_fallback ? 1 : 0;
    c.relax_threads =
        (long long)(p_.strategy == GLB_WD || p_.strategy == GLB_HP ? cap_wd_ : cap_relax_) * kBlock;
    c.hp_threads = (long long)cap_hp_ * kBlock;
    c.gen = g_->stamp_epoch;
    c.tag_bits = Cell<D>::kGenBits;
    c.renorm_gen = 0xFFFFFFFFu;
    c.scan_epoch = g_->scan_epoch + 1;
    c.rec_cap = kMaxRecords;
    c.shard_mode = shard_mode_ ? 1 : 0;
    c.small_ok = !shard_mode_ && !getenv("GLB_NO_SMALL") ? 1 : 0;
    for (int i = 0; i < 2; ++i) {
      c.wd_items_buf[i] = items_[i];
      c.wd_tf_buf[i] = tile_first_[i];
    }
    // Fused item pushes (no scan between WD steps) measured slower on C2 than
    // scan + relax (the pushes' row loads sit on the relax kernel's critical
    // path), so they are opt-in.
    c.hp_big = hp_big_;
    c.hp_owner = hp_owner_;
    c.bins_two = bins_two() ? 1 : 0;
    c.n_nodes = n_all_;
    // Dense-frontier scans (cells in id order, frontiers of >= N/8 nodes) speed
    // the relax kernel up per edge.  Where the cells fit L2 (32-bit tier) the
    // id-ordered processing does ~10 % more re-relaxation (C2), a wash, so
    // they are opt-in there; in the 24-bit tier (cells > 2x L2) they are the
    // default (C5 at 32 bits: SSSP 266 -> 200 ms, BFS 59.6 -> 48.7).
    // GLB_WD_DENSE=0 off, =1 on, =2 on for every frontier size (tests).
    {
      const char* e = getenv("GLB_WD_DENSE");
      const int mode = e ? atoi(e) : (Cell<D>::kGenBits == 8 ? 1 : 0);
      c.dense_ok = (p_.strategy == GLB_WD || p_.strategy == GLB_HP) && !shard_mode_ && Cell<D>::kPacked &&
                           mode > 0
                       ? (mode >= 2 ? (1 << 30) : 8)
                       : 0;
      hp_dense_ = p_.strategy == GLB_HP && c.dense_ok;
    }
    c.wd_fused = p_.strategy == GLB_WD && !shard_mode_ && getenv("GLB_WD_FUSED") ? 1 : 0;
    // Inside the cluster loop the fused pushes replace the scan that every CTA
    // of the cluster would otherwise replicate over the whole list (C3 BFS WD
    // 117 -> 96 ms); grid steps keep scan + relax.
    c.wd_fused_small = p_.strategy == GLB_WD && !shard_mode_ && !c.wd_fused &&
                       !getenv("GLB_NO_WD_FUSED_SMALL") ? 1 : 0;
    c.bm[0] = bm_[0];
    c.bm[1] = bm_[1];
    c.ep_dn[0] = p_.strategy == GLB_EP ? ep_dn_[0] : nullptr;
    c.ep_dn[1] = p_.strategy == GLB_EP ? ep_dn_[1] : nullptr;
    // a compaction reads the whole bitmap (n/8 bytes): worth it once the list
    // holds >= 1/256 of the nodes (C3 SSSP: 65,536 of 16.8M) and >= 32K of them
    c.bm_thr = !bm_on() ? 0u
               : getenv("GLB_BM_THR") ? bm_thr_
                                      : (unsigned)std::max<long long>(bm_thr_, n_all_ / 256);
    // the BS seed list's bit is set after the seed kernel; NS seeds the source's
    // children too, so its first list is taken in seed order
    c.bm_valid[0] = p_.strategy == GLB_BS ? 1 : 0;
    c.recs = drecs_;
    c.ls = ls_;
    c.ptw = ptw_;
    c.ptw_off = 0;
    c.ptw_cap = ptw_ ? kPtwCap : 0;
    h_->ctrl = c;
    GLB_CUDA_TRY(cudaMemcpyAsync(ctrl_, &h_->ctrl, sizeof(DevCtrl), cudaMemcpyHostToDevice, s_));

    // distances: INF everywhere, then the seeds
    k_init_dist<D><<<grid_for((long long)nb, kBlock, g_->num_sms * 8), kBlock, 0, s_>>>(
        cells_, (long long)nb);
    GLB_CHECK_LAUNCH();
    const long long src = p_.source;
    long long klo = 0, khi = 0, elo = 0, ehi = 0;
    const bool edges = p_.strategy == GLB_EP;
    long long seeds = 1;
    if (p_.strategy == GLB_NS || edges) {
      long long h2[2];
      GLB_CUDA_TRY(cudaMemcpyAsync(h2, (edges ? row_ : cs_) + src, 16, cudaMemcpyDeviceToHost, s_));
      GLB_CUDA_TRY(cudaStreamSynchronize(s_));
      if (edges) {
        elo = h2[0];
        ehi = h2[1];
        seeds = ehi - elo;
      } else {
        klo = g_->n + h2[0];
        khi = g_->n + h2[1];
        seeds = 1 + khi - klo;
      }
    }
    seed_count_ = seeds;
    k_seed<D><<<grid_for(std::max<long long>(seeds, 1), kBlock, g_->num_sms * 4), kBlock, 0, s_>>>(
        cells_, q_[0], &ctrl_->qcount[0], src, klo, khi, elo, ehi, edges);
    GLB_CHECK_LAUNCH();
    if (bm_[0] && p_.strategy == GLB_BS)  // the seed list's member bit
      GLB_CUDA_TRY(cudaMemsetAsync((char*)bm_[0] + (src >> 3), 1 << (src & 7), 1, s_));
  }

  // Keep the distance cells -- the randomly accessed array -- resident in L2
  // (persisting access-policy window on the library stream; captured into
  // the loop graph's kernel nodes).  Column / weight streams are loaded
  // evict-first, so they do not displace it.
  void pin_cells_in_l2(size_t bytes) {
    if (!g_->l2_persist_max || !g_->l2_window_max || !getenv("GLB_L2_PERSIST")) return;
    const size_t win = std::min(bytes, (size_t)g_->l2_window_max);
    cudaStreamAttrValue attr;
    std::memset(&attr, 0, sizeof(attr));
    attr.accessPolicyWindow.base_ptr = (void*)cells_;
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio =
        (float)std::min(1.0, (double)g_->l2_persist_max / (double)win);
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(s_, cudaStreamAttributeAccessPolicyWindow, &attr) != cudaSuccess)
      cudaGetLastError();  // advisory only
  }

  Relaxer<D, W> relaxer() const {
    Relaxer<D, W> rx;
    rx.col = col_;
    rx.wt = wt_;
    rx.cells = cells_;
    rx.stamp = stamp_;
    rx.gen = 0;
    rx.qout = nullptr;
    rx.nout = nullptr;
    rx.ovf = &ctrl_->overflow;
    return rx;
  }

  // ------------------------------------------------------ step launches ---
  // 24-bit tier: retag every cell (see ctl_check_renorm)
  void launch_renorm() {
    if constexpr (Cell<D>::kGenBits == 8) {
      k_renorm<<<grid_for(n_all_, kBlock, g_->num_sms * 8), kBlock, 0, s_>>>(cells_, n_all_, ctrl_,
                                                                             tail_);
      GLB_CHECK_LAUNCH();
    } else {
      throw Error{GLB_ECUDA, "renormalisation requested for a 32-bit-tag run"};
    }
  }

  void launch_relax(unsigned grid) {
    const Relaxer<D, W> rx = relaxer();
    switch (p_.strategy) {
      case GLB_BS:
        if (bs_warp_) {
          k_bs_warp<D, W><<<grid, kBlock, 0, s_>>>(row_, rx, ctrl_, tail_);
          break;
        }
        if (bm_[0]) {  // id-ordered in-list (no-op below the threshold).  Not a
                       // programmatic dependent launch: relax CTAs parked early
                       // starve the compaction (C5 SSSP BS 238 -> 455 ms)
          k_bm_compact<<<grid_for(bm_vec_ * 4, kBmBlock, g_->num_sms * 8), kBmBlock, 0, s_>>>(ctrl_,
                                                                                          bm_vec_ * 4);
          GLB_CHECK_LAUNCH();
        }
        k_bs_relax<D, W><<<grid, kBlock, 0, s_>>>(row_, rx, ctrl_, tail_);
        break;
      case GLB_NS:  // binned windows + the CTA bin of the long ones (TMA-staged)
        if (bm_[0]) {  // id-ordered in-list (no-op below the threshold)
          k_bm_compact<<<grid_for(bm_vec_ * 4, kBmBlock, g_->num_sms * 8), kBmBlock, 0, s_>>>(ctrl_,
                                                                                          bm_vec_ * 4);
          GLB_CHECK_LAUNCH();
        }
        if (!bins_two()) {  // split nodes all shorter than a CTA-bin window: one kernel
          k_ns_relax<D, W><<<grid, kBlock, 0, s_>>>(row_, ns_mirror(), rx, ctrl_, tail_);
          break;
        }
        k_ns_relax<D, W><<<grid, kBlock, 0, s_>>>(row_, ns_mirror(), rx, ctrl_, CtlTail{0, {}, 0});
        GLB_CHECK_LAUNCH();
        launch_dependent(k_bigbin<D, W, NsMirror>, (unsigned)cap_big_, rx, ns_mirror(), ctrl_, tail_);
        break;
      case GLB_EP:
        if (p_.chunked)
          k_ep_relax<D, W, true><<<grid, kBlock, 0, s_>>>(row_, src_, rx, ctrl_, tail_);
        else
          k_ep_relax<D, W, false><<<grid, kBlock, 0, s_>>>(row_, src_, rx, ctrl_, tail_);
        break;
      default: throw Error{GLB_EINVAL, "no relax kernel for this strategy"};
    }
    GLB_CHECK_LAUNCH();
  }
  void launch_wd_scan(unsigned grid) {
    k_wd_scan<D><<<grid, kBlock, 0, s_>>>(row_, cells_, lb_,
                                          ctrl_);
    GLB_CHECK_LAUNCH();
  }
  void launch_wd_relax(unsigned grid) {
    launch_dependent(k_wd_relax<D, W>, grid, relaxer(), row_, ctrl_, tail_);
    GLB_CHECK_LAUNCH();
  }
  // second kernel of a step: programmatic dependent launch on the first
  template <typename... KArgs, typename... Args>
  void launch_dependent(void (*kernel)(KArgs...), unsigned grid, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s_;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_ ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GLB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, args...));
  }
  // HP / NS windows never reach the CTA bin when mdt < kBinCtaMin: the
  // window kernel is then the step's only kernel (and runs the control tail)
  bool bins_two() const { return mdt_ >= kBinCtaMin; }
  void launch_hp(unsigned grid) {
    if (hp_dense_) {  // id-ordered super-list for window sub-iteration 0 (no-op otherwise)
      k_tag_compact<D><<<grid_for((n_all_ + 31) / 32, kBmBlock, g_->num_sms * 8), kBmBlock, 0, s_>>>(cells_,
                                                                                                   ctrl_);
      GLB_CHECK_LAUNCH();
    }
    if (!bins_two()) {
      k_hp_window<D, W><<<grid, kBlock, 0, s_>>>(row_, relaxer(), ctrl_, tail_);
      GLB_CHECK_LAUNCH();
      return;
    }
    k_hp_window<D, W><<<grid, kBlock, 0, s_>>>(row_, relaxer(), ctrl_, CtlTail{0, {}, 0});
    GLB_CHECK_LAUNCH();
    launch_dependent(k_bigbin<D, W, NoMirror>, (unsigned)cap_big_, relaxer(), NoMirror{}, ctrl_, tail_);
    GLB_CHECK_LAUNCH();
  }
  NsMirror ns_mirror() const { return NsMirror{cs_, g_->n}; }
  void launch_small() {
    const long long* cs = p_.strategy == GLB_NS ? cs_ : nullptr;
    const uint32_t* src = p_.strategy == GLB_EP ? src_ : nullptr;
    if (small_ctas_ == 16)
      k_small_loop<D, W, 16><<<16, kSmallThreads, small_smem_bytes<D>(), s_>>>(
          row_, cs, g_->n, src, p_.chunked != 0, relaxer(), ctrl_, tail_);
    else
      k_small_loop<D, W, 8><<<8, kSmallThreads, small_smem_bytes<D>(), s_>>>(
          row_, cs, g_->n, src, p_.chunked != 0, relaxer(), ctrl_, tail_);
    GLB_CHECK_LAUNCH();
  }
  void launch_control(cudaGraphConditionalHandle hl, const ModeHandles& hm, int gm) {
    k_control<<<1, 32, 0, s_>>>(ctrl_, hl, hm, gm);
    GLB_CHECK_LAUNCH();
  }

  void read_ctrl() {
    GLB_CUDA_TRY(cudaMemcpyAsync(&h_->ctrl, ctrl_, sizeof(DevCtrl), cudaMemcpyDeviceToHost, s_));
    GLB_CUDA_TRY(cudaStreamSynchronize(s_));
    if (h_->ctrl.overflow) throw OverflowRestart{};
  }

  // ------------------------------------------------------- host loop ---
  void loop_host() {
    k_control_init<<<1, 32, 0, s_>>>(ctrl_, 0, ModeHandles{}, 0);
    GLB_CHECK_LAUNCH();
    read_ctrl();
    step_host();
  }

  // launch steps until the control block reports done (or paused)
  void step_host() {
    const bool timing = p_.record_timing != 0;
    while (!h_->ctrl.done) {
      const DevCtrl& c = h_->ctrl;
      const long long n_in = c.qcount[c.in];
      const unsigned nrec0 = c.nrec;
      ev_used_ = ev_of_rec_.size() * 4;
      EvPair ev{nullptr, nullptr, nullptr, nullptr, 0};
      if (timing) {
        ev.k0 = event();
        ev.k1 = event();
      }
      switch (c.use_small ? (int)kModeSmall : c.mode) {
        case kModeSmall: {
          ev.threads = (long long)small_ctas_ * kSmallThreads;
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k0, s_));
          launch_small();
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k1, s_));
          break;
        }
        case kModeRelax: {
          const long long per = p_.strategy == GLB_EP ? 4LL * kBlock : kBlock;
          const unsigned grid = p_.strategy == GLB_NS ? (unsigned)cap_relax_  // as HP windows
                                                      : grid_for(n_in, (int)per, cap_relax_);
          ev.threads = (long long)grid * kBlock;
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k0, s_));
          launch_relax(grid);
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k1, s_));
          break;
        }
        case kModeWD: {
          if (timing) {
            ev.o0 = event();
            ev.o1 = event();
            GLB_CUDA_TRY(cudaEventRecord(ev.o0, s_));
          }
          launch_wd_scan(grid_for(c.wd_dense ? n_all_ : n_in, kWdScanTile, cap_scan_));
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.o1, s_));
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k0, s_));
          launch_wd_relax(cap_wd_);
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k1, s_));
          ev.threads = (long long)cap_wd_ * kBlock;
          break;
        }
        case kModeWDF: {  // fused WD: the item list is already built
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k0, s_));
          launch_wd_relax(cap_wd_);
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k1, s_));
          ev.threads = (long long)cap_wd_ * kBlock;
          break;
        }
        case kModeRenorm:
          launch_renorm();
          break;
        case kModeHP: {  // full grid: the window kernel sizes its warp chunks to the list
          const unsigned grid = (unsigned)cap_hp_;
          ev.threads = (long long)grid * kBlock;
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k0, s_));
          launch_hp(grid);
          if (timing) GLB_CUDA_TRY(cudaEventRecord(ev.k1, s_));
          break;
        }
        default: throw Error{GLB_ECUDA, "control block in an unknown mode"};
      }
      const bool small = c.use_small != 0;
      launch_control(0, ModeHandles{}, 0);
      read_ctrl();
      if (small) {  // several iterations in one launch: per-record device timers
        for (unsigned r = nrec0; r < h_->ctrl.nrec; ++r)
          ev_of_rec_.push_back(EvPair{nullptr, nullptr, nullptr, nullptr, (long long)small_ctas_ * kSmallThreads});
      } else if (h_->ctrl.nrec > nrec0) {
        ev_of_rec_.push_back(ev);
      }
    }
  }

  // ----------------------------------------------------- graph loop ---
  std::string graph_key() const {
    std::ostringstream k;
    k << g_->device << '|' << p_.strategy << '|' << bs_warp_ << '|' << fused_ctl_ << '|' << unroll_ << '|' << pdl_ << '|' << Cell<D>::kDistBits << '|' << W << '|' << p_.chunked << '|' << cap_relax_
      << '|' << cap_scan_ << '|' << cap_wd_ << '|' << cap_hp_ << '|' << cap_big_ << '|' << (const void*)row_ << '|'
      << (const void*)col_ << '|' << (const void*)wt_ << '|' << (const void*)cs_ << '|'
      << (const void*)src_ << '|' << (const void*)cells_ << '|' << (const void*)stamp_ << '|'
      << (const void*)ctrl_ << '|' << (const void*)items_[0] << '|' << (const void*)items_[1] << '|'
      << (const void*)tile_first_[0] << '|' << (const void*)tile_first_[1] << '|'
      << (const void*)lb_.flags << '|' << (const void*)lb_.aggs << '|' << g_->n << '|' << n_all_
      << '|' << mdt_ << '|' << resume_graph_ << '|' << (const void*)bm_[0] << '|' << bm_vec_ << '|' << hp_dense_ << '|' << small_ctas_;
    return k.str();
  }

  void capture_into(cudaGraph_t graph, const cudaGraphNode_t* deps, size_t ndeps) {
    GLB_CUDA_TRY(cudaStreamBeginCaptureToGraph(s_, graph, deps, nullptr, ndeps,
                                               cudaStreamCaptureModeThreadLocal));
  }
  void end_capture() {
    cudaGraph_t out = nullptr;
    GLB_CUDA_TRY(cudaStreamEndCapture(s_, &out));
  }
  static cudaGraphNode_t only_node(cudaGraph_t graph) {
    size_t n = 0;
    GLB_CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &n));
    if (n != 1) throw Error{GLB_ECUDA, "unexpected node count while building the loop graph"};
    cudaGraphNode_t node;
    GLB_CUDA_TRY(cudaGraphGetNodes(graph, &node, &n));
    return node;
  }

  cudaGraphExec_t build_graph() {
    cudaGraph_t graph;
    GLB_CUDA_TRY(cudaGraphCreate(&graph, 0));
    try {
      // fused control: kGraphUnroll SWITCH steps per WHILE iteration
      const int unroll = fused_ctl_ ? unroll_ : 1;
      cudaGraphConditionalHandle h_loop = 0;
      ModeHandles h_mode{};
      GLB_CUDA_TRY(cudaGraphConditionalHandleCreate(&h_loop, graph, 0, 0));
      for (int u = 0; u < unroll; ++u)
        GLB_CUDA_TRY(cudaGraphConditionalHandleCreate(&h_mode.h[u], graph, 0, 0));
      capture_into(graph, nullptr, 0);
      if (resume_graph_)  // sharded run: re-enter after the exchange
        k_control_resume<<<1, 32, 0, s_>>>(ctrl_, h_loop, h_mode, 1);
      else
        k_control_init<<<1, 32, 0, s_>>>(ctrl_, h_loop, h_mode, 1);
      GLB_CHECK_LAUNCH();
      end_capture();
      cudaGraphNode_t init = only_node(graph);

      alignas(cudaGraphNodeParams) unsigned char wbuf[sizeof(cudaGraphNodeParams)] = {};
      cudaGraphNodeParams& wp = *reinterpret_cast<cudaGraphNodeParams*>(wbuf);
      wp.type = cudaGraphNodeTypeConditional;
      wp.conditional.handle = h_loop;
      wp.conditional.type = cudaGraphCondTypeWhile;
      wp.conditional.size = 1;
      cudaGraphNode_t wnode;
      GLB_CUDA_TRY(cudaGraphAddNode(&wnode, graph, &init, 1, &wp));
      cudaGraph_t body = wp.conditional.phGraph_out[0];

      // SWITCH on the step kind (StepMode): the strategy's grid kernels or
      // the CTA-resident small-frontier loop
      if (fused_ctl_) tail_ = CtlTail{h_loop, h_mode, 1};
      cudaGraphNode_t snode = nullptr;
      for (int u = 0; u < unroll; ++u) {
        alignas(cudaGraphNodeParams) unsigned char sbuf[sizeof(cudaGraphNodeParams)] = {};
        cudaGraphNodeParams& sp = *reinterpret_cast<cudaGraphNodeParams*>(sbuf);
        sp.type = cudaGraphNodeTypeConditional;
        sp.conditional.handle = h_mode.h[u];
        sp.conditional.type = cudaGraphCondTypeSwitch;
        sp.conditional.size = kNumModes;
        cudaGraphNode_t prev = snode;
        GLB_CUDA_TRY(cudaGraphAddNode(&snode, body, prev ? &prev : nullptr, prev ? 1 : 0, &sp));
        if (p_.strategy == GLB_WD || p_.strategy == GLB_HP) {
          capture_into(sp.conditional.phGraph_out[kModeWD], nullptr, 0);
          launch_wd_scan(cap_scan_);
          launch_wd_relax(cap_wd_);
          end_capture();
        }
        if (p_.strategy == GLB_WD) {
          capture_into(sp.conditional.phGraph_out[kModeWDF], nullptr, 0);
          launch_wd_relax(cap_wd_);
          end_capture();
        }
        if (p_.strategy == GLB_HP) {
          capture_into(sp.conditional.phGraph_out[kModeHP], nullptr, 0);
          launch_hp(cap_hp_);
          end_capture();
        }
        if (relax_kernel()) {
          capture_into(sp.conditional.phGraph_out[kModeRelax], nullptr, 0);
          launch_relax(cap_relax_);
          end_capture();
        }
        capture_into(sp.conditional.phGraph_out[kModeSmall], nullptr, 0);
        launch_small();
        end_capture();
        if (Cell<D>::kGenBits == 8) {
          capture_into(sp.conditional.phGraph_out[kModeRenorm], nullptr, 0);
          launch_renorm();
          end_capture();
        }
      }
      tail_ = CtlTail{0, {}, 0};
      if (!fused_ctl_) {
        capture_into(body, &snode, 1);
        launch_control(h_loop, h_mode, 1);
        end_capture();
      }
      cudaGraphExec_t exec;
      GLB_CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      return exec;
    } catch (...) {
      tail_ = CtlTail{0, {}, 0};
      cudaStreamCaptureStatus cs;
      if (cudaStreamIsCapturing(s_, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(s_, &junk);
      }
      cudaGetLastError();
      cudaGraphDestroy(graph);
      throw;
    }
  }

  // Instantiated loop graphs are cached process-wide by everything captured
  // into them (device, strategy, widths, grids and every buffer pointer).
  // With the caching allocator a new graph of the same shape usually gets the
  // same buffers back, so create -> run -> destroy cycles reuse the exec.
  void loop_graph() { GLB_CUDA_TRY(cudaGraphLaunch(graph_exec(), s_)); }
  cudaGraphExec_t graph_exec() {
    const std::string key = graph_key();
    cudaGraphExec_t exec = nullptr;
    {
      std::lock_guard<std::mutex> lk(exec_cache_mu());
      auto it = exec_cache().find(key);
      if (it != exec_cache().end()) exec = it->second;
    }
    if (!exec) {
      exec = build_graph();
      std::lock_guard<std::mutex> lk(exec_cache_mu());
      exec_cache().emplace(key, exec);
    }
    return exec;
  }
  static std::mutex& exec_cache_mu() {
    static std::mutex* m = new std::mutex();
    return *m;
  }
  static std::unordered_map<std::string, cudaGraphExec_t>& exec_cache() {
    static auto* c = new std::unordered_map<std::string, cudaGraphExec_t>();
    return *c;
  }

  // ---------------------------------------------------------- results ---
  void collect_records() {
    const unsigned n = std::min(h_->ctrl.nrec, kMaxRecords);
    std::vector<DevRecord> dr(n);
    if (n)
      GLB_CUDA_TRY(cudaMemcpy(dr.data(), drecs_, sizeof(DevRecord) * n, cudaMemcpyDeviceToHost));
    recs_.clear();
    recs_.reserve(n);
    for (unsigned i = 0; i < n; ++i) {
      const DevRecord& d = dr[i];
      glb_record r;
      std::memset(&r, 0, sizeof(r));
      r.iteration = d.iteration;
      r.sub_iteration = d.sub;
      r.tag = d.tag;
      r.active_items = d.active;
      r.threads = d.threads;
      r.work_total = d.work;
      r.work_max = d.work_max;
      r.work_sumsq = d.work_sumsq;
      r.relax_ops = d.relax;
      r.push_ops = d.push;
      r.kernel_ms = d.k1 > d.k0 && d.k0 != ~0ull ? (double)(d.k1 - d.k0) * 1e-6 : 0.0;
      r.overhead_ms = d.o0 && d.o1 > d.o0 && d.o0 != ~0ull ? (double)(d.o1 - d.o0) * 1e-6 : 0.0;
      r.thread_work_offset = ptw_ ? d.ptw_off : -1;
      if (i < ev_of_rec_.size()) {  // host loop: CUDA-event times and the exact grid
        const EvPair& e = ev_of_rec_[i];
        float ms = 0;
        if (e.k0 && cudaEventElapsedTime(&ms, e.k0, e.k1) == cudaSuccess) r.kernel_ms = ms;
        if (e.o0 && cudaEventElapsedTime(&ms, e.o0, e.o1) == cudaSuccess) r.overhead_ms = ms;
        cudaGetLastError();
        r.threads = e.threads;
      }
      recs_.push_back(r);
    }
  }

  void finish(glb_run_stats* st, float dev_ms) {
    st->status = GLB_OK;
    st->dist_bits = Cell<D>::kDistBits;
    st->iterations = h_->ctrl.iteration;
    st->launches = (int64_t)recs_.size();
    st->mdt = mdt_;
    st->sub_iterations = 0;
    st->relax_ops = st->push_ops = st->edges_examined = st->active_items = 0;
    double kms = 0;
    for (const glb_record& r : recs_) {
      if (r.tag == GLB_HP) ++st->sub_iterations;
      st->relax_ops += r.relax_ops;
      st->push_ops += r.push_ops;
      st->edges_examined += r.work_total;
      st->active_items += r.active_items;
      kms += r.kernel_ms;
    }
    st->device_ms = dev_ms;
    st->kernel_ms = kms;
    st->overhead_ms = std::max(0.0, (double)dev_ms - kms);
    st->setup_ms = setup_ms_;
    st->n_records = (int64_t)h_->ctrl.nrec;
  }
};

// =========================================================== sharded run ===
// 1-D vertex partition: the shard is a graph over the GLOBAL id
// space whose rows outside [lo, hi) are empty, so every strategy kernel runs
// unchanged on the owned frontier.  Cells of remote vertices act as
// sender-side shadows: a candidate for remote v is atomically min-combined
// into cells[v], and v is pushed once per generation like any improvement.
// At the iteration boundary the out list is split by owner; remote entries
// (v, best candidate) go to per-owner send buckets that the host exchanges
// (NCCL all-to-all), and received updates are relaxed into the owner's cells
// with the same generation, so local and remote pushes deduplicate together.

__device__ __forceinline__ int owner_of(const long long* __restrict__ bounds, int parts,
                                        uint32_t v) {
  int lo = 0, hi = parts;  // bounds[0] = 0 <= v < bounds[parts]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((long long)v >= bounds[mid])
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

struct ShardBounds {
  long long b[65];
};

__global__ void k_shard_count(const DevCtrl* __restrict__ c, ShardBounds sb, int parts,
                              unsigned long long* __restrict__ counts) {
  __shared__ unsigned int s_cnt[64];
  if (threadIdx.x < 64) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int ol = c->strategy == GLB_HP ? c->sup_out : c->out;
  const uint32_t* q = c->qptr[ol];
  const unsigned n = c->qcount[ol];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&s_cnt[owner_of(sb.b, parts, q[i])], 1u);
  __syncthreads();
  if (threadIdx.x < parts && s_cnt[threadIdx.x])
    atomicAdd(counts + threadIdx.x, (unsigned long long)s_cnt[threadIdx.x]);
}

// cursors[o] start at the owner's offset in `send`; the local owner's cursor
// indexes `local_tmp`.
__global__ void k_shard_scatter(const DevCtrl* __restrict__ c, ShardBounds sb, int parts, int me,
                                const unsigned long long* __restrict__ cells,
                                unsigned long long* __restrict__ cursors,
                                unsigned long long* __restrict__ send,
                                uint32_t* __restrict__ local_tmp) {
  const int ol = c->strategy == GLB_HP ? c->sup_out : c->out;
  const uint32_t* q = c->qptr[ol];
  const unsigned n = c->qcount[ol];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = q[i];
    const int o = owner_of(sb.b, parts, v);
    const unsigned long long slot = atomicAdd(cursors + o, 1ull);
    if (o == me)
      local_tmp[slot] = v;
    else
      send[slot] = ((unsigned long long)Cell<uint32_t>::dist(cells[v]) << 32) | v;
  }
}

// received (dist << 32 | v) updates: relax with this iteration's generation
__global__ void k_shard_apply(DevCtrl* __restrict__ c, unsigned long long* __restrict__ cells,
                              const unsigned long long* __restrict__ recv, long long nrecv) {
  const int ol = c->strategy == GLB_HP ? c->sup_out : c->out;
  uint32_t* q = c->qptr[ol];
  unsigned int* nq = &c->qcount[ol];
  const uint32_t gen = c->gen;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nrecv;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long e = recv[i];
    const uint32_t v = (uint32_t)e, d = (uint32_t)(e >> 32);
    bool first = false;
    if (relax_cell<uint32_t>(cells, v, d, gen, &first) && first) q_append(q, nq, v);
  }
}

template <bool W>
class ShardSession : public ShardSessionBase, public Runner<uint32_t, W> {
  using R = Runner<uint32_t, W>;

 public:
  ShardSession(glb_graph* g, const glb_run_params& p, const long long* bounds, int parts, int rank)
      : R(g, params_, recs_), params_(p), parts_(parts), me_(rank) {
    for (int i = 0; i <= parts; ++i) sb_.b[i] = bounds[i];
    lo_ = bounds[rank];
    hi_ = bounds[rank + 1];
    this->shard_mode_ = true;
    std::memset(&stats_, 0, sizeof(stats_));
    stats_.split_fraction = -1.0;
    R::prepare(&stats_);
    if (p.source < lo_ || p.source >= hi_)  // not ours: start with an empty frontier
      GLB_CUDA_TRY(cudaMemsetAsync(&this->ctrl_->qcount[0], 0, 4, this->s_));
    k_control_init<<<1, 32, 0, this->s_>>>(this->ctrl_, 0, ModeHandles{}, 0);
    GLB_CHECK_LAUNCH();
    this->read_ctrl();
    counts_ = (unsigned long long*)ensure(g->ws.misc_small, 64 * 8 * 2);
    tmp_ = (uint32_t*)ensure(g->ws.shard_tmp, (size_t)std::max<long long>(g->n, 1) * 4);
  }

  void local(int64_t* send_counts, unsigned long long* send, long long cap,
             int64_t* local_next) override {
    this->step_host();  // until the control block pauses at the iteration boundary
    const DevCtrl& hc = this->h_->ctrl;
    const int ol = hc.strategy == GLB_HP ? hc.sup_out : hc.out;
    const long long n = hc.qcount[ol];
    cudaStream_t s = this->s_;
    GLB_CUDA_TRY(cudaMemsetAsync(counts_, 0, 64 * 8, s));
    const unsigned grid = grid_for(std::max<long long>(n, 1), kBlock, this->g_->num_sms * 4);
    k_shard_count<<<grid, kBlock, 0, s>>>(this->ctrl_, sb_, parts_, counts_);
    GLB_CHECK_LAUNCH();
    unsigned long long h[64];
    GLB_CUDA_TRY(cudaMemcpyAsync(h, counts_, 8 * parts_, cudaMemcpyDeviceToHost, s));
    GLB_CUDA_TRY(cudaStreamSynchronize(s));
    unsigned long long off[64], run = 0;
    for (int o = 0; o < parts_; ++o) {
      off[o] = o == me_ ? 0 : run;
      if (o != me_) run += h[o];
      send_counts[o] = o == me_ ? 0 : (int64_t)h[o];
    }
    if ((long long)run > cap) throw Error{GLB_ENOMEM, "shard send buffer too small"};
    GLB_CUDA_TRY(cudaMemcpyAsync(counts_ + 64, off, 8 * parts_, cudaMemcpyHostToDevice, s));
    k_shard_scatter<<<grid, kBlock, 0, s>>>(this->ctrl_, sb_, parts_, me_, this->cells_,
                                            counts_ + 64, send, tmp_);
    GLB_CHECK_LAUNCH();
    // the out list keeps only owned vertices
    const unsigned nlocal = (unsigned)h[me_];
    GLB_CUDA_TRY(cudaMemcpyAsync(this->q_[ol], tmp_, (size_t)nlocal * 4, cudaMemcpyDeviceToDevice, s));
    GLB_CUDA_TRY(cudaMemcpyAsync(&this->ctrl_->qcount[ol], &nlocal, 4, cudaMemcpyHostToDevice, s));
    GLB_CUDA_TRY(cudaStreamSynchronize(s));
    *local_next = nlocal;
  }

  void apply(const unsigned long long* recv, long long n) override {
    if (n > 0) {
      k_shard_apply<<<grid_for(n, kBlock, this->g_->num_sms * 4), kBlock, 0, this->s_>>>(
          this->ctrl_, this->cells_, recv, n);
      GLB_CHECK_LAUNCH();
    }
  }

  long long advance() override {
    k_shard_advance<<<1, 32, 0, this->s_>>>(this->ctrl_);
    GLB_CHECK_LAUNCH();
    this->read_ctrl();
    const DevCtrl& hc = this->h_->ctrl;
    return hc.strategy == GLB_HP ? hc.qcount[hc.sup_in] : hc.qcount[hc.in];
  }

  void finish(int64_t* dist_owned, glb_run_stats* st) override {
    R::finish_run(dist_owned, &stats_, lo_, hi_);
    *st = stats_;
  }

 private:
  glb_run_params params_;
  std::vector<glb_record> recs_;
  glb_run_stats stats_;
  ShardBounds sb_;
  int parts_, me_;
  long long lo_, hi_;
  unsigned long long* counts_ = nullptr;
  uint32_t* tmp_ = nullptr;
};

// ===================================================== peer-memory run ===
// The whole sharded BSP loop inside the library (glb_peer_run): local
// relaxation to the iteration boundary as the loop graph (one launch), then
// the peer exchange of glb_peer.cuh, then one control-block read-back that
// carries the global termination and overflow verdicts -- the only host
// synchronisation of an iteration.
class PeerRunBase {
 public:
  virtual ~PeerRunBase() {}
  virtual void issue(unsigned long long seq) = 0;
  virtual int complete() = 0;  // 0 continue, 1 globally done, 2 global overflow
  virtual void finish(int64_t* dist_owned, glb_run_stats* st, glb_peer_stats* xs) = 0;
};

__global__ void k_peer_begin(PeerTable* t, uint32_t* tmp) {
  if (threadIdx.x != 0) return;
  t->tmp = tmp;
  for (int o = 0; o < kPeerMaxParts; ++o) t->cursor[o] = 0;
  t->my_work = t->sent = t->recv = t->wait_ns = 0;
}

__global__ void k_peer_reset_cursors(PeerTable* t) {
  if (threadIdx.x < kPeerMaxParts) t->cursor[threadIdx.x] = 0;
}

template <typename D, bool W>
class PeerRun : public PeerRunBase, public Runner<D, W> {
  using R = Runner<D, W>;

 public:
  PeerRun(glb_peer* pr, const glb_run_params& p, std::vector<glb_record>& recs)
      : R(pr->g, params_, recs), params_(p), pr_(pr) {
    params_.loop_mode = GLB_LOOP_GRAPH;
    this->shard_mode_ = true;
    this->resume_graph_ = true;
    // The control step runs as its own kernel here, not as the last-CTA tail
    // of each step: with several processes time-sliced on one GPU (ranks
    // sharing a device) the fused tail was observed to stall the WD loop
    // graph (tools/peer_mp_probe.py: hangs with the tail, completes with
    // GLB_NO_FUSED_CTL), and the extra ~3 us per step is small next to the
    // exchange.
    this->fused_ctl_ = false;
    std::memset(&stats_, 0, sizeof(stats_));
    stats_.split_fraction = -1.0;
    lo_ = pr->bounds[pr->rank];
    hi_ = pr->bounds[pr->rank + 1];
    R::prepare(&stats_);
    cudaStream_t s = this->s_;
    if (p.source < lo_ || p.source >= hi_)  // not ours: start with an empty frontier
      GLB_CUDA_TRY(cudaMemsetAsync(&this->ctrl_->qcount[0], 0, 4, s));
    k_control_init<<<1, 32, 0, s>>>(this->ctrl_, 0, ModeHandles{}, 0);
    GLB_CHECK_LAUNCH();
    uint32_t* tmp = (uint32_t*)ensure(this->g_->ws.shard_tmp,
                                      (size_t)std::max<long long>(this->g_->n, 1) * 4);
    k_peer_begin<<<1, 32, 0, s>>>(pr->table, tmp);
    GLB_CHECK_LAUNCH();
    GLB_CUDA_TRY(cudaEventCreate(&ev_[0]));
    GLB_CUDA_TRY(cudaEventCreate(&ev_[1]));
    grid_ = (unsigned)this->g_->num_sms * 4;
    // Build, instantiate and upload the loop graph now, before any rank's
    // mailbox poll occupies the device: ranks sharing a GPU must never need
    // a module load or a graph upload while a peer's k_peer_wait spins.
    exec_ = R::graph_exec();
    GLB_CUDA_TRY(cudaGraphUpload(exec_, s));
    GLB_CUDA_TRY(cudaStreamSynchronize(s));
  }
  ~PeerRun() override {
    for (cudaEvent_t e : ev_)
      if (e) cudaEventDestroy(e);
  }

  void issue(unsigned long long seq) override {
    NvtxRange r("glb bsp iteration: local relaxation + peer exchange (issue)");
    const int parity = (int)(seq & 1ull);
    cudaStream_t s = this->s_;
    GLB_CUDA_TRY(cudaGraphLaunch(exec_, s));  // local relaxation, paused at the iteration boundary
    GLB_CHECK_LAUNCH();
    GLB_CUDA_TRY(cudaEventRecord(ev_[0], s));
    PeerTable* t = pr_->table;
    k_peer_scatter<D><<<grid_, kBlock, 0, s>>>(this->ctrl_, t, this->cells_, parity);
    GLB_CHECK_LAUNCH();
    k_peer_publish<<<1, 64, 0, s>>>(this->ctrl_, t, seq, parity);
    GLB_CHECK_LAUNCH();
    k_peer_wait<<<1, 32, 0, s>>>(this->ctrl_, t, seq, parity);
    GLB_CHECK_LAUNCH();
    k_peer_reset_cursors<<<1, kPeerMaxParts, 0, s>>>(t);
    GLB_CHECK_LAUNCH();
    k_peer_apply<D><<<grid_, kBlock, 0, s>>>(this->ctrl_, t, this->cells_, this->stamp_, parity);
    GLB_CHECK_LAUNCH();
    k_shard_advance<<<1, 32, 0, s>>>(this->ctrl_);
    GLB_CHECK_LAUNCH();
    GLB_CUDA_TRY(cudaEventRecord(ev_[1], s));
    GLB_CUDA_TRY(cudaMemcpyAsync(&this->h_->ctrl, this->ctrl_, sizeof(DevCtrl),
                                 cudaMemcpyDeviceToHost, s));
  }

  int complete() override {
    {
      NvtxRange r("glb bsp iteration: wait for the global verdict");
      GLB_CUDA_TRY(cudaStreamSynchronize(this->s_));
    }
    const DevCtrl& hc = this->h_->ctrl;
    if ((hc.bad_input & 0xFFFF0000u) == kPeerTimeoutFlag) {
      pr_->poisoned = true;
      throw Error{GLB_ECUDA, "peer exchange: rank " + std::to_string(hc.bad_input & 0xFFFFu) +
                                 " did not publish iteration " + std::to_string(bsp_ + 1) +
                                 " within the timeout (GLB_PEER_TIMEOUT_S)"};
    }
    float ms = 0;
    if (cudaEventElapsedTime(&ms, ev_[0], ev_[1]) == cudaSuccess) xms_ += ms;
    cudaGetLastError();
    ++bsp_;
    if (hc.overflow) return 2;
    return hc.aux[1] == 0 ? 1 : 0;
  }

  void finish(int64_t* dist_owned, glb_run_stats* st, glb_peer_stats* xs) override {
    R::finish_run(dist_owned, &stats_, lo_, hi_);
    *st = stats_;
    if (xs) {
      PeerTable ht;
      GLB_CUDA_TRY(cudaMemcpy(&ht, pr_->table, sizeof(PeerTable), cudaMemcpyDeviceToHost));
      std::memset(xs, 0, sizeof(*xs));
      xs->bsp_iterations = bsp_;
      xs->sent_entries = (int64_t)ht.sent;
      xs->recv_entries = (int64_t)ht.recv;
      xs->entry_bytes = (int32_t)PeerEntry<D>::kBytes;
      xs->parts = pr_->parts;
      xs->rank = pr_->rank;
      xs->transport = pr_->transport;
      xs->exchange_ms = xms_;
      xs->wait_ms = (double)ht.wait_ns * 1e-6;
    }
  }

 private:
  glb_run_params params_;
  glb_peer* pr_;
  glb_run_stats stats_;
  long long lo_ = 0, hi_ = 0;
  cudaEvent_t ev_[2] = {nullptr, nullptr};
  cudaGraphExec_t exec_ = nullptr;  // cached process-wide (Runner::graph_exec)
  unsigned grid_ = 148;
  long long bsp_ = 0;
  double xms_ = 0;
};

}  // namespace

// Load every exchange kernel into the context up front (lazy module loading
// would otherwise load them at first launch -- possibly while another rank's
// mailbox poll is spinning on the same GPU).
void preload_peer_kernels() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = -1;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  done.push_back(dev);
  {
    cudaFuncAttributes a;
    const void* ks[] = {
        (const void*)k_peer_scatter<dist24_t>, (const void*)k_peer_scatter<uint32_t>,
        (const void*)k_peer_scatter<unsigned long long>, (const void*)k_peer_apply<dist24_t>,
        (const void*)k_peer_apply<uint32_t>, (const void*)k_peer_apply<unsigned long long>,
        (const void*)k_peer_publish, (const void*)k_peer_wait, (const void*)k_peer_begin,
        (const void*)k_peer_reset_cursors, (const void*)k_shard_advance,
        (const void*)k_control_init, (const void*)k_control_resume};
    for (const void* k : ks) cudaFuncGetAttributes(&a, k);
    cudaGetLastError();
  }
}

namespace {
std::unique_ptr<PeerRunBase> make_peer_run(int bits, glb_peer* pr, const glb_run_params& p,
                                           std::vector<glb_record>& recs) {
  const bool w = p.algo == GLB_SSSP && pr->g->wt != nullptr;
  if (bits == 24)
    return w ? std::unique_ptr<PeerRunBase>(new PeerRun<dist24_t, true>(pr, p, recs))
             : std::unique_ptr<PeerRunBase>(new PeerRun<dist24_t, false>(pr, p, recs));
  if (bits == 32)
    return w ? std::unique_ptr<PeerRunBase>(new PeerRun<uint32_t, true>(pr, p, recs))
             : std::unique_ptr<PeerRunBase>(new PeerRun<uint32_t, false>(pr, p, recs));
  return w ? std::unique_ptr<PeerRunBase>(new PeerRun<unsigned long long, true>(pr, p, recs))
           : std::unique_ptr<PeerRunBase>(new PeerRun<unsigned long long, false>(pr, p, recs));
}

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

// An aborted run leaves stamps / look-back flags of generations the handle
// never recorded; clear both so the next run cannot mistake them for its own.
void reset_epochs(glb_graph* g) {
  cudaStreamSynchronize(g->stream);
  cudaGetLastError();
  if (g->ws.stamp.p) cudaMemsetAsync(g->ws.stamp.p, 0, g->ws.stamp.bytes, g->stream);
  if (g->ws.scan_flags.p) cudaMemsetAsync(g->ws.scan_flags.p, 0, g->ws.scan_flags.bytes, g->stream);
  g->stamp_epoch = 0;
  g->scan_epoch = 0;
  cudaStreamSynchronize(g->stream);
}

template <typename D>
void run_guarded(glb_graph* g, const glb_run_params& p, int64_t* dist_out, glb_run_stats* st,
                 std::vector<glb_record>& recs) {
  try {
    run_typed<D>(g, p, dist_out, st, recs);
  } catch (...) {
    reset_epochs(g);
    throw;
  }
}

}  // namespace

void reset_epochs_public(glb_graph* g) { reset_epochs(g); }

void run(glb_graph* g, const glb_run_params& p, int64_t* dist_out, glb_run_stats* st,
         std::vector<glb_record>& recs) {
  std::memset(st, 0, sizeof(*st));
  st->split_fraction = -1.0;
  // Tiers (dist_bits 0): 24-bit distances in u32 cells, then 32-bit in
  // packed u64 cells, then 64-bit; a tier that overflows re-runs at the next
  // one.  The handle remembers a 24-bit overflow per relaxation kind so
  // later runs on the same graph start at 32 bits.  The 24-bit tier is only
  // the first choice when the u64 cells are over twice the L2: with 8 cells
  // per 32-byte sector instead of 4, the relax kernels lose more to L2
  // sector contention between cell gathers and atomics than they gain from
  // the smaller array while either array mostly fits (C2 / C4 SSSP WD
  // +13..15 %, C3 mixed within +-8 %).
  const bool huge = g->n * 8LL > 2LL * g->l2_bytes;
  const int first = p.dist_bits ? p.dist_bits
                                : (!g->narrow_overflow[p.algo == GLB_SSSP] && huge ? 24 : 32);
  for (int bits = first;; bits = bits == 24 ? 32 : 64) {
    try {
      if (bits == 24)
        run_guarded<dist24_t>(g, p, dist_out, st, recs);
      else if (bits == 32)
        run_guarded<uint32_t>(g, p, dist_out, st, recs);
      else
        run_guarded<unsigned long long>(g, p, dist_out, st, recs);
      return;
    } catch (const OverflowRestart&) {
      if (bits == 64) throw Error{GLB_EOVERFLOW, "distance exceeds the 63-bit range"};
      if (p.dist_bits)
        throw Error{GLB_EOVERFLOW, "distance exceeds the " + std::to_string(bits) + "-bit range"};
      if (bits == 24) g->narrow_overflow[p.algo == GLB_SSSP] = true;
      recs.clear();
      const double sf = st->split_fraction;
      std::memset(st, 0, sizeof(*st));
      st->split_fraction = sf;
      GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
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
    if (p.dist_bits != 0 && p.dist_bits != 24 && p.dist_bits != 32 && p.dist_bits != 64)
      throw glb::Error{GLB_EINVAL, "dist_bits must be 0, 24, 32 or 64"};
    if (p.loop_mode != GLB_LOOP_HOST && p.loop_mode != GLB_LOOP_GRAPH)
      throw glb::Error{GLB_EINVAL, "loop_mode must be GLB_LOOP_HOST or GLB_LOOP_GRAPH"};
    std::memset(stats, 0, sizeof(*stats));
    if (p.strategy == GLB_EP) {
      const long long required = (g->weighted ? 3 : 2) * g->m;
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
      const int64_t k = std::min<int64_t>(records_capacity, (int64_t)recs.size());
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
  const int64_t total = (int64_t)g->last_records.size();
  const int64_t k = offset >= total ? 0 : std::min<int64_t>(capacity, total - offset);
  if (k > 0) std::memcpy(records, g->last_records.data() + offset, (size_t)k * sizeof(glb_record));
  *written = k;
  return GLB_OK;
}

extern "C" int glb_run_thread_work(glb_graph* g, int64_t offset, int64_t count, uint32_t* out,
                                   int64_t* total) {
  try {
    if (!g || offset < 0 || count < 0 || (count > 0 && !out))
      throw glb::Error{GLB_EINVAL, "glb_run_thread_work: invalid argument"};
    std::lock_guard<std::mutex> lk(g->mu);
    if (total) *total = g->ptw_len;
    if (count == 0) return GLB_OK;
    if (offset + count > g->ptw_len || !g->ws.ptw.p)
      throw glb::Error{GLB_ERANGE, "per-thread work range beyond the last instrumented run"};
    int prev = -1;
    cudaGetDevice(&prev);
    GLB_CUDA_TRY(cudaSetDevice(g->device));
    const cudaError_t e = cudaMemcpy(out, (const uint32_t*)g->ws.ptw.p + offset, (size_t)count * 4,
                                     cudaMemcpyDeviceToHost);
    if (prev >= 0) cudaSetDevice(prev);
    GLB_CUDA_TRY(e);
    return GLB_OK;
  } catch (const glb::Error& e) {
    glb::set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    glb::set_error(e.what());
    return GLB_ECUDA;
  }
}

// ============================================================ shard C-ABI ===
namespace {
template <typename F>
int shard_guard(glb_graph* g, F&& f) {
  try {
    if (!g) throw glb::Error{GLB_EINVAL, "graph is NULL"};
    std::lock_guard<std::mutex> lk(g->mu);
    int prev = -1;
    cudaGetDevice(&prev);
    GLB_CUDA_TRY(cudaSetDevice(g->device));
    try {
      f();
    } catch (...) {
      if (prev >= 0) cudaSetDevice(prev);
      throw;
    }
    if (prev >= 0) cudaSetDevice(prev);
    return GLB_OK;
  } catch (const glb::Error& e) {
    glb::set_error(e.msg);
    return e.code;
  } catch (const glb::OverflowRestart&) {
    // a sharded run has no automatic re-run at a wider tier: the caller
    // restarts with dist_bits 64 (sharded.run_sharded does)
    if (g) {
      delete g->shard;
      g->shard = nullptr;
      glb::reset_epochs_public(g);
    }
    glb::set_error("distance exceeds the 32-bit range of the sharded run");
    return GLB_EOVERFLOW;
  } catch (const std::exception& e) {
    glb::set_error(e.what());
    return GLB_ECUDA;
  }
}
}  // namespace

extern "C" int glb_shard_begin(glb_graph* g, const glb_run_params* p, const int64_t* bounds,
                               int parts, int rank) {
  return shard_guard(g, [&] {
    if (!p || !bounds) throw glb::Error{GLB_EINVAL, "params/bounds is NULL"};
    if (parts < 1 || parts > 64 || rank < 0 || rank >= parts)
      throw glb::Error{GLB_EINVAL, "parts must be in [1, 64] and 0 <= rank < parts"};
    if (bounds[0] != 0 || bounds[parts] != g->n)
      throw glb::Error{GLB_EINVAL, "bounds must start at 0 and end at num_nodes"};
    for (int i = 0; i < parts; ++i)
      if (bounds[i + 1] < bounds[i]) throw glb::Error{GLB_EINVAL, "bounds must be nondecreasing"};
    if (p->strategy != GLB_BS && p->strategy != GLB_WD && p->strategy != GLB_HP)
      throw glb::Error{GLB_EINVAL, "sharded runs support the BS, WD and HP strategies"};
    if (p->algo != GLB_BFS && p->algo != GLB_SSSP) throw glb::Error{GLB_EINVAL, "unknown algo"};
    if (p->source < 0 || p->source >= g->n)
      throw glb::Error{GLB_EINVAL, "source out of range"};
    if (p->block_size < 1) throw glb::Error{GLB_EINVAL, "block_size must be >= 1"};
    if (p->dist_bits == 64 || p->dist_bits == 24)
      throw glb::Error{GLB_EINVAL, "sharded runs use 32-bit distances (dist_bits 0 or 32)"};
    delete g->shard;
    g->shard = nullptr;
    const bool weighted = p->algo == GLB_SSSP && g->wt != nullptr;
    long long bb[65];
    for (int i = 0; i <= parts; ++i) bb[i] = bounds[i];
    if (weighted)
      g->shard = new glb::ShardSession<true>(g, *p, bb, parts, rank);
    else
      g->shard = new glb::ShardSession<false>(g, *p, bb, parts, rank);
  });
}

extern "C" int glb_shard_local(glb_graph* g, int64_t* send_counts, void* send_buf,
                               int64_t send_capacity, int64_t* local_next) {
  return shard_guard(g, [&] {
    if (!g->shard) throw glb::Error{GLB_EINVAL, "no sharded run in progress"};
    if (!send_counts || !local_next || (!send_buf && send_capacity > 0))
      throw glb::Error{GLB_EINVAL, "NULL argument"};
    g->shard->local(send_counts, (unsigned long long*)send_buf, send_capacity, local_next);
  });
}

extern "C" int glb_shard_apply(glb_graph* g, const void* recv_buf, int64_t nrecv) {
  return shard_guard(g, [&] {
    if (!g->shard) throw glb::Error{GLB_EINVAL, "no sharded run in progress"};
    if (nrecv < 0 || (nrecv > 0 && !recv_buf)) throw glb::Error{GLB_EINVAL, "bad receive buffer"};
    g->shard->apply((const unsigned long long*)recv_buf, nrecv);
  });
}

extern "C" int glb_shard_advance(glb_graph* g, int64_t* frontier) {
  return shard_guard(g, [&] {
    if (!g->shard) throw glb::Error{GLB_EINVAL, "no sharded run in progress"};
    const long long f = g->shard->advance();
    if (frontier) *frontier = f;
  });
}

extern "C" int glb_shard_finish(glb_graph* g, int64_t* dist_owned, glb_run_stats* stats) {
  return shard_guard(g, [&] {
    if (!g->shard) throw glb::Error{GLB_EINVAL, "no sharded run in progress"};
    glb_run_stats st;
    try {
      g->shard->finish(dist_owned, &st);
    } catch (...) {
      delete g->shard;
      g->shard = nullptr;
      glb::reset_epochs_public(g);
      throw;
    }
    if (stats) *stats = st;
    delete g->shard;
    g->shard = nullptr;
  });
}

// ============================================================= peer C-ABI ===
namespace {
template <typename F>
int peer_guard(F&& f) {
  try {
    f();
    return GLB_OK;
  } catch (const glb::Error& e) {
    glb::set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    glb::set_error(e.what());
    return GLB_ECUDA;
  }
}

struct DeviceScope {  // make `dev` current, restore the caller's device
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    GLB_CUDA_TRY(cudaSetDevice(dev));
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

unsigned long long peer_timeout_ns() {
  const char* e = getenv("GLB_PEER_TIMEOUT_S");
  const double s = e ? atof(e) : 120.0;
  return (unsigned long long)((s > 0 ? s : 120.0) * 1e9);
}

void peer_write_table(glb_peer* p) {
  glb::PeerTable ht;
  std::memset(&ht, 0, sizeof(ht));
  for (int r = 0; r < p->parts; ++r) {
    ht.base[r] = p->base[r];
    ht.seg[r] = p->bounds[r + 1] - p->bounds[r];
  }
  for (int r = 0; r <= p->parts; ++r) ht.bounds[r] = p->bounds[r];
  ht.parts = p->parts;
  ht.me = p->rank;
  ht.timeout_ns = peer_timeout_ns();
  GLB_CUDA_TRY(cudaMemcpy(p->table, &ht, sizeof(ht), cudaMemcpyHostToDevice));
}

void peer_check_params(glb_peer* p, const glb_run_params* q) {
  if (!p || !q) throw glb::Error{GLB_EINVAL, "peer/params is NULL"};
  if (!p->connected) throw glb::Error{GLB_EINVAL, "peer is not connected"};
  if (p->poisoned)
    throw glb::Error{GLB_ECUDA, "peer exchange lost lockstep (an earlier run timed out); recreate it"};
  if (q->strategy != GLB_BS && q->strategy != GLB_WD && q->strategy != GLB_HP)
    throw glb::Error{GLB_EINVAL, "sharded runs support the BS, WD and HP strategies"};
  if (q->algo != GLB_BFS && q->algo != GLB_SSSP) throw glb::Error{GLB_EINVAL, "unknown algo"};
  if (q->source < 0 || q->source >= p->g->n) throw glb::Error{GLB_EINVAL, "source out of range"};
  if (q->block_size < 1) throw glb::Error{GLB_EINVAL, "block_size must be >= 1"};
  if (q->dist_bits != 0 && q->dist_bits != 24 && q->dist_bits != 32 && q->dist_bits != 64)
    throw glb::Error{GLB_EINVAL, "dist_bits must be 0, 24, 32 or 64"};
}

// Run every rank in `ps` (one host thread): each iteration is issued on all
// ranks before any is waited for, so ranks sharing a GPU cannot deadlock.
// All ranks see the same global verdict after every iteration, so a tier
// change (overflow) happens on all of them at once.
void peer_run_all(glb_peer* const* ps, int n, const glb_run_params& q, int64_t* const* dist,
                  glb_run_stats* st, glb_peer_stats* xs) {
  glb_peer* p0 = ps[0];
  const bool sssp = q.algo == GLB_SSSP;
  const bool huge = p0->g->n * 8LL > 2LL * p0->g->l2_bytes;
  const int first = q.dist_bits ? q.dist_bits : (!p0->narrow_overflow[sssp] && huge ? 24 : 32);
  for (int bits = first;; bits = bits == 24 ? 32 : 64) {
    std::vector<std::vector<glb_record>> recs(n);
    std::vector<std::unique_ptr<glb::PeerRunBase>> runs(n);
    int verdict = 0;
    try {
      for (int r = 0; r < n; ++r) {
        DeviceScope ds(ps[r]->g->device);
        runs[r] = glb::make_peer_run(bits, ps[r], q, recs[r]);
      }
      while (verdict == 0) {
        for (int r = 0; r < n; ++r) {
          DeviceScope ds(ps[r]->g->device);
          runs[r]->issue(++ps[r]->seq);
        }
        int v0 = -1;
        for (int r = 0; r < n; ++r) {
          DeviceScope ds(ps[r]->g->device);
          const int v = runs[r]->complete();
          if (v0 >= 0 && v != v0) {
            for (int k = 0; k < n; ++k) ps[k]->poisoned = true;
            throw glb::Error{GLB_ECUDA, "peer exchange: ranks disagree on the global verdict"};
          }
          v0 = v;
        }
        verdict = v0;
      }
      if (verdict == 1) {
        for (int r = 0; r < n; ++r) {
          DeviceScope ds(ps[r]->g->device);
          runs[r]->finish(dist ? dist[r] : nullptr, &st[r], xs ? &xs[r] : nullptr);
          st[r].n_records = (int64_t)recs[r].size();
          ps[r]->g->last_records.swap(recs[r]);
        }
        return;
      }
    } catch (...) {
      runs.clear();
      for (int r = 0; r < n; ++r) {
        DeviceScope ds(ps[r]->g->device);
        glb::reset_epochs_public(ps[r]->g);
      }
      throw;
    }
    runs.clear();  // verdict 2: distance overflow somewhere -> next tier everywhere
    for (int r = 0; r < n; ++r) {
      DeviceScope ds(ps[r]->g->device);
      glb::reset_epochs_public(ps[r]->g);
    }
    if (bits == 64) throw glb::Error{GLB_EOVERFLOW, "distance exceeds the 63-bit range"};
    if (q.dist_bits)
      throw glb::Error{GLB_EOVERFLOW, "distance exceeds the " + std::to_string(bits) + "-bit range"};
    if (bits == 24)
      for (int r = 0; r < n; ++r) ps[r]->narrow_overflow[sssp] = true;
  }
}
}  // namespace

extern "C" int glb_peer_create(glb_graph* g, const int64_t* bounds, int parts, int rank,
                               glb_peer** out) {
  return peer_guard([&] {
    if (!g || !bounds || !out) throw glb::Error{GLB_EINVAL, "graph/bounds/out is NULL"};
    if (parts < 1 || parts > glb::kPeerMaxParts || rank < 0 || rank >= parts)
      throw glb::Error{GLB_EINVAL, "parts must be in [1, 64] and 0 <= rank < parts"};
    if (bounds[0] != 0 || bounds[parts] != g->n)
      throw glb::Error{GLB_EINVAL, "bounds must start at 0 and end at num_nodes"};
    for (int i = 0; i < parts; ++i)
      if (bounds[i + 1] < bounds[i]) throw glb::Error{GLB_EINVAL, "bounds must be nondecreasing"};
    DeviceScope ds(g->device);
    std::unique_ptr<glb_peer> p(new glb_peer());
    p->g = g;
    p->parts = parts;
    p->rank = rank;
    for (int i = 0; i <= parts; ++i) p->bounds[i] = bounds[i];
    const long long seg = std::max<long long>(bounds[rank + 1] - bounds[rank], 1);
    p->region_bytes = glb::kPeerHdrBytes + 2 * (size_t)parts * (size_t)seg * glb::kPeerEntryMax;
    GLB_CUDA_TRY(cudaMalloc((void**)&p->region, p->region_bytes));
    GLB_CUDA_TRY(cudaMemset(p->region, 0, glb::kPeerHdrBytes));
    cudaError_t e = cudaMalloc((void**)&p->table, sizeof(glb::PeerTable));
    if (e != cudaSuccess) {
      cudaFree(p->region);
      GLB_CUDA_TRY(e);
    }
    p->base[rank] = p->region;
    glb::preload_peer_kernels();
    *out = p.release();
  });
}

extern "C" int glb_peer_handle(glb_peer* p, void* handle_out) {
  return peer_guard([&] {
    if (!p || !handle_out) throw glb::Error{GLB_EINVAL, "peer/handle is NULL"};
    static_assert(sizeof(cudaIpcMemHandle_t) == GLB_PEER_HANDLE_BYTES, "IPC handle size");
    DeviceScope ds(p->g->device);
    cudaIpcMemHandle_t h;
    GLB_CUDA_TRY(cudaIpcGetMemHandle(&h, p->region));
    std::memcpy(handle_out, &h, sizeof(h));
  });
}

extern "C" int glb_peer_connect(glb_peer* p, const void* handles) {
  return peer_guard([&] {
    if (!p || !handles) throw glb::Error{GLB_EINVAL, "peer/handles is NULL"};
    if (p->connected) throw glb::Error{GLB_EINVAL, "peer is already connected"};
    DeviceScope ds(p->g->device);
    const char* hb = (const char*)handles;
    for (int r = 0; r < p->parts; ++r) {
      if (r == p->rank) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, hb + (size_t)r * GLB_PEER_HANDLE_BYTES, sizeof(h));
      void* ptr = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (int k = 0; k < r; ++k)
          if (p->ipc_opened[k]) {
            cudaIpcCloseMemHandle(p->base[k]);
            p->ipc_opened[k] = false;
            p->base[k] = nullptr;
          }
        throw glb::Error{GLB_ECUDA, "cudaIpcOpenMemHandle(rank " + std::to_string(r) +
                                        "): " + cudaGetErrorString(e)};
      }
      p->base[r] = (char*)ptr;
      p->ipc_opened[r] = true;
    }
    peer_write_table(p);
    p->transport = GLB_PEER_IPC;
    p->connected = true;
  });
}

extern "C" int glb_peer_connect_local(glb_peer* const* peers, int parts) {
  return peer_guard([&] {
    if (!peers || parts < 1) throw glb::Error{GLB_EINVAL, "peers is NULL"};
    for (int r = 0; r < parts; ++r) {
      if (!peers[r]) throw glb::Error{GLB_EINVAL, "NULL peer"};
      if (peers[r]->parts != parts || peers[r]->rank != r)
        throw glb::Error{GLB_EINVAL, "peers must be ranks 0..parts-1 of one partition"};
      if (peers[r]->connected) throw glb::Error{GLB_EINVAL, "peer is already connected"};
      for (int i = 0; i <= parts; ++i)
        if (peers[r]->bounds[i] != peers[0]->bounds[i])
          throw glb::Error{GLB_EINVAL, "peers were created with different bounds"};
    }
    for (int r = 0; r < parts; ++r) {
      glb_peer* p = peers[r];
      DeviceScope ds(p->g->device);
      for (int k = 0; k < parts; ++k) {
        p->base[k] = peers[k]->region;
        const int dk = peers[k]->g->device;
        if (dk != p->g->device) {  // direct loads/stores into the other GPU's HBM
          const cudaError_t e = cudaDeviceEnablePeerAccess(dk, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) GLB_CUDA_TRY(e);
          cudaGetLastError();
        }
      }
      peer_write_table(p);
      p->transport = GLB_PEER_LOCAL;
      p->connected = true;
    }
  });
}

extern "C" int glb_peer_run(glb_peer* p, const glb_run_params* params, int64_t* dist_owned,
                            glb_run_stats* stats, glb_peer_stats* xstats) {
  return peer_guard([&] {
    peer_check_params(p, params);
    if (!stats) throw glb::Error{GLB_EINVAL, "stats is NULL"};
    std::lock_guard<std::mutex> lk(p->g->mu);
    glb_peer* ps[1] = {p};
    int64_t* ds[1] = {dist_owned};
    peer_run_all(ps, 1, *params, ds, stats, xstats);
  });
}

extern "C" int glb_peer_run_local(glb_peer* const* peers, int parts, const glb_run_params* params,
                                  int64_t* const* dist_owned, glb_run_stats* stats,
                                  glb_peer_stats* xstats) {
  return peer_guard([&] {
    if (!peers || parts < 1 || !stats) throw glb::Error{GLB_EINVAL, "peers/stats is NULL"};
    std::vector<std::unique_lock<std::mutex>> locks;
    for (int r = 0; r < parts; ++r) {
      peer_check_params(peers[r], params);
      if (peers[r]->parts != parts || peers[r]->rank != r || peers[r]->transport != GLB_PEER_LOCAL)
        throw glb::Error{GLB_EINVAL, "glb_peer_run_local needs all ranks of a local connection"};
      for (int k = 0; k < r; ++k)
        if (peers[k]->g == peers[r]->g) throw glb::Error{GLB_EINVAL, "ranks share a graph handle"};
      locks.emplace_back(peers[r]->g->mu);
    }
    peer_run_all(peers, parts, *params, dist_owned, stats, xstats);
  });
}

extern "C" int glb_peer_destroy(glb_peer* p) {
  return peer_guard([&] {
    if (!p) return;
    DeviceScope ds(p->g->device);
    cudaStreamSynchronize(p->g->stream);
    for (int r = 0; r < p->parts; ++r)
      if (p->ipc_opened[r]) cudaIpcCloseMemHandle(p->base[r]);
    cudaFree(p->table);
    cudaFree(p->region);
    cudaGetLastError();
    delete p;
  });
}
