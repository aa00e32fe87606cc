// glb_internal.cuh -- shared device/host internals of libgraphlb_b200.so.
//
// Device layout of a graph:
//   row  : int64[n+1]   row offsets (kept 64-bit; csr.py:57 INDEX_DTYPE)
//   col  : uint32[m]    destinations (narrowed from int64 on upload)
//   wt   : uint32[m]    weights, or nullptr for an unweighted graph
//   dist : uint32[n]    INF = 0xFFFFFFFF (u64 variant: INF = 2^63-1, engine.py:27)
//   stamp: uint32[n]    "pushed in generation g" marks replacing the dedup
//                       flag array + clear() of worklist.py:26-81
//   queue: uint32[n]    node worklists (capacity n is overflow-free with dedup)
#pragma once

#include <initializer_list>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/graphlb_b200.h"

namespace glb {

constexpr int kBlock = 256;  // threads per CTA for every relax kernel
constexpr int kStatSlots = 32;  // spread of the per-launch counter atomics
// Tail padding of every u32 edge array (col / weights): the CTA bin's 1-D
// TMA copies read whole 16-byte units, up to 3 elements past the last edge.
constexpr size_t kEdgePad = 64;

// NVTX range over a host-side phase (header-only NVTX v3: free unless a
// profiler is attached).  Phases mirror the reference's perf_counter splits
// (engine.py:221,269; node_based.py:21-29,75-78; workload.py:96-110):
// upload, setup overhead, traversal loop, distances back, and per BSP
// iteration of a sharded run the local relaxation and the peer exchange.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- errors ---
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};

#define GLB_CUDA_TRY(expr)                                                       \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      throw ::glb::Error{_e == cudaErrorMemoryAllocation ? GLB_ENOMEM : GLB_ECUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(_e)};    \
    }                                                                            \
  } while (0)

// Every kernel launch site ends with GLB_CHECK_LAUNCH(): it surfaces launch
// errors and counts the launch (glb_kernel_launches()).
void count_launch();
void count_launches(unsigned long long n);  // kernels executed inside a CUDA graph
#define GLB_CHECK_LAUNCH()             \
  do {                                 \
    ::glb::count_launch();             \
    GLB_CUDA_TRY(cudaGetLastError());  \
  } while (0)

// ------------------------------------------------------- distance traits ---
template <typename D>
struct DistTraits;
template <>
struct DistTraits<uint32_t> {
  static constexpr uint32_t kInf = 0xFFFFFFFFu;
};
template <>
struct DistTraits<unsigned long long> {
  static constexpr unsigned long long kInf = 0x7FFFFFFFFFFFFFFFull;
};
// 24-bit distances: a distinct 32-bit unsigned type tags the tier whose cell
// is a single u32 (below).
typedef char32_t dist24_t;
template <>
struct DistTraits<dist24_t> {
  static constexpr dist24_t kInf = 0xFFFFFFu;
};

// Distance cells.  With 32-bit distances a cell packs (dist << 32 | gen):
// one 64-bit atomicMin both lowers the distance (engine.py:120-139) and
// reports, through the old generation, whether this node was already pushed
// to this iteration's out-list -- the dedup flag of worklist.py:107-130
// folded into the relaxation atomic.  Equal distances keep the older
// generation, so only a strict improvement can claim the push.  64-bit
// distances (the overflow re-run) keep a separate stamp array instead.
//
// Three tiers, tried in order (an overflow re-runs in the next):
//   dist24_t            u32 cell  = dist << 8 | tag            (16.8 MB at C2)
//   uint32_t            u64 cell  = dist << 32 | gen           (33.5 MB)
//   unsigned long long  u64 dist  + a separate stamp array
// The 24-bit tier halves the randomly gathered array, so more of it stays in
// L2.  Its tag is (gen mod 128) + 1 and 0 means "pushed long ago"; before
// every generation that is a multiple of 128 the control inserts a
// renormalisation step (k_renorm) that resets all tags to 0.  Within such an
// epoch tags grow with the generation like the 32-bit tier's, so an equal
// distance never replaces an older tag and only a strict improvement can
// claim the push.  S is the storage type, tag() the generation as stored,
// make_tag() a cell with a raw tag (0 = no generation).
template <typename D>
struct Cell;
template <>
struct Cell<dist24_t> {
  using S = uint32_t;
  static constexpr bool kPacked = true;
  static constexpr int kGenBits = 8;
  static constexpr int kDistBits = 24;
  __host__ __device__ static constexpr uint32_t tag(uint32_t gen) { return (gen & 127u) + 1u; }
  __host__ __device__ static constexpr uint32_t make_tag(uint32_t d, uint32_t t) {
    return (d << 8) | t;
  }
  __host__ __device__ static constexpr uint32_t make(uint32_t d, uint32_t gen) {
    return make_tag(d, tag(gen));
  }
  __device__ static dist24_t dist(uint32_t c) { return (dist24_t)(c >> 8); }
  __device__ static uint32_t gen(uint32_t c) { return c & 0xFFu; }
};
template <>
struct Cell<uint32_t> {
  using S = unsigned long long;
  static constexpr bool kPacked = true;
  static constexpr int kGenBits = 32;
  static constexpr int kDistBits = 32;
  __host__ __device__ static constexpr unsigned long long make_tag(uint32_t d, uint32_t t) {
    return ((unsigned long long)d << 32) | t;
  }
  __host__ __device__ static constexpr unsigned long long make(uint32_t d, uint32_t gen) {
    return make_tag(d, gen);
  }
  __host__ __device__ static constexpr uint32_t tag(uint32_t gen) { return gen; }
  __device__ static uint32_t dist(unsigned long long c) { return (uint32_t)(c >> 32); }
  __device__ static uint32_t gen(unsigned long long c) { return (uint32_t)c; }
};
template <>
struct Cell<unsigned long long> {
  using S = unsigned long long;
  static constexpr bool kPacked = false;
  static constexpr int kGenBits = 0;
  static constexpr int kDistBits = 64;
  __host__ __device__ static constexpr unsigned long long make(unsigned long long d, uint32_t) {
    return d;
  }
  __host__ __device__ static constexpr unsigned long long make_tag(unsigned long long d, uint32_t) {
    return d;
  }
  __host__ __device__ static constexpr uint32_t tag(uint32_t) { return 0; }
  __device__ static unsigned long long dist(unsigned long long c) { return c; }
  __device__ static uint32_t gen(unsigned long long) { return 0; }
};
template <typename D>
using CellS = typename Cell<D>::S;

// ---------------------------------------------------- per-launch counters ---
// One LaunchStats per kernel invocation; kStatSlots copies spread the atomics
// (summed on the host).  Mirrors MetricsRecord (engine.py:142-174).
struct StatSlot {
  unsigned long long relax;
  unsigned long long push;
  unsigned long long work;
  unsigned long long work_sq;
  unsigned long long work_max;
  unsigned long long pad[3];
};
struct LaunchStats {
  StatSlot slot[kStatSlots];
};

// Step modes of the device-side strategy state machine (k_control).
// kModeSmall is the CTA-resident loop of glb_small.cuh running the strategy's
// own step (the underlying mode stays in DevCtrl::mode, `use_small` selects it).
// kModeWDF is a WD step whose item list the previous step already appended
// (fused pushes): relax only, no scan.
// kModeRenorm retags the 24-bit tier's cells (see Cell<dist24_t>).
enum StepMode : int {
  kModeDone = 0, kModeRelax = 1, kModeWD = 2, kModeHP = 3, kModeSmall = 4, kModeWDF = 5,
  kModeRenorm = 6
};
constexpr int kNumModes = 7;

// One long HP window [lo, hi) of node u at distance dn, relaxed in 2048-edge
// pieces claimed by any CTA (hierarchical processing's CTA granularity).
struct HpBig {
  unsigned long long dn;
  long long lo, hi;
  unsigned int qbase;        // first piece of this window in the step's piece space
  unsigned int pad;
};

struct StepTimer {  // %globaltimer ns, min over CTA starts / max over CTA ends
  unsigned long long start;
  unsigned long long end;
};

// One kernel invocation as recorded on the device by k_control
// (MetricsRecord, engine.py:142-174).
struct DevRecord {
  int iteration, sub, tag, pad;
  long long active, threads, work, relax, push, work_max;
  double work_sumsq;
  unsigned long long k0, k1, o0, o1;  // relax kernel / scan kernel timers
  long long ptw_off;                  // first per-thread work slot, -1 = not recorded
  long long pad2;
};

// Device control block: worklist cursors, the current step's frame (which
// lists it reads and writes, stamp generation, HP window) and the strategy
// state machine.  Written by k_control_init / k_control, read by every step
// kernel at launch, so the same kernels run under the host loop and inside
// the device-driven CUDA graph.
struct DevCtrl {
  unsigned int qcount[8];       // worklist cursors
  unsigned int overflow;        // a u32 candidate reached INF -> re-run in u64
  unsigned int bad_input;       // upload validation failure
  long long wd_total;           // WD: active edges of this invocation
  long long wd_items;           // WD: worklist items with remaining edges
  long long aux[4];
  uint32_t* qptr[4];            // worklist buffers
  // ---- current step
  int in, out, next, mode;      // lists read / pushed / carried (HP), StepMode
  unsigned int gen;             // dedup stamp generation of the out list
  int iteration, sub, tag;      // record fields
  long long window, mdt;        // HP window start s*mdt (also WD-fallback base)
  unsigned int scan_epoch;      // look-back epoch of the next WD scan
  int done;
  unsigned long long scan_ticket, relax_ticket;  // dynamic tile tickets of the WD step
  int shard_mode;   // sharded run: pause at every iteration boundary for the exchange
  int paused;
  int small_ok;     // small-frontier iterations may run in k_small_loop
  int use_small;    // the next step runs in k_small_loop
  int small_exit;   // k_small_loop ran (and already recorded / advanced) this step
  unsigned long long kernels;  // kernels the device loop has executed (graph mode launch count)
  // ---- WD with fused pushes: relax kernels append WdItems (pre, base, node)
  // for the next step directly, reserving (items, edges) with one 64-bit
  // atomic per warp batch, so no scan runs between WD steps
  void* wd_items_buf[2];        // WdItem lists (the step's input is [wd_cur])
  unsigned int* wd_tf_buf[2];   // tile_first of each list
  int wd_fused;                 // WD strategy outside sharded runs
  int wd_fused_small;           // fused pushes inside the cluster loop only
  int wd_cur;
  unsigned long long wd_next;   // (items << 32) | edges appended to list [wd_cur ^ 1]
  unsigned int wd_zero_next;    // zero-degree nodes pushed (counted for the record only)
  int wd_dense;                 // the WD scan reads the frontier from the cells, not the queue
  int dense_ok;                 // WD id-order scans from frontiers of >= n_nodes / dense_ok (0: off)
  int tag_bits;                 // generation bits stored in a cell (8: 24-bit tier)
  int saved_mode;               // the step a renormalisation step interrupted
  unsigned int renorm_gen;      // generation of the last renormalisation
  long long n_nodes;            // nodes of the traversed graph
  // ---- HP: windows >= kHpCtaThreshold edges form a grid-wide CTA bin
  struct HpBig* hp_big;         // bin entries of the current window step
  unsigned int* hp_owner;       // CTA-bin piece -> entry
  unsigned long long hp_big_ctr;  // (entries << 32) | pieces reserved, in one atomic
  unsigned int hp_piece_next;   // next piece ticket
  int bins_two;                 // HP / NS steps launch k_bigbin after the window kernel
  // ---- HP super-iteration state (hierarchical.py:54-136)
  int sup_in, sup_out, cur, spare;
  long long s;
  long long hp_threshold;       // KernelConfig.block_size
  int hp_fallback, strategy;
  long long relax_threads, hp_threads;  // launched threads (record field)
  StepTimer t_relax, t_scan;
  unsigned int nrec, rec_cap;
  DevRecord* recs;
  struct LaunchStats* ls;
  unsigned int tail_done;       // CTAs of the step's last kernel that finished (ctl_tail)
  unsigned int tail_pad;
  // ---- per-thread work lists (MetricsRecord.per_thread_work, engine.py:142-174):
  // thread t of the launch recorded next adds its work to ptw[ptw_off + t]
  uint32_t* ptw;                // null: summed counters only
  unsigned long long ptw_off, ptw_cap;
  // ---- BS id-ordered frontiers: bm[i] holds one bit per node of list i's
  // members; a relax step over >= bm_thr nodes first rebuilds its list in id
  // order from the bitmap (k_bm_compact), so the row / column / weight /
  // cell accesses of neighbouring lanes fall on shared sectors
  uint32_t* bm[2];
  unsigned int bm_thr;          // 0: off
  unsigned int bm_ctr;          // compaction cursor (zeroed by the relax step after it)
  unsigned int bm_err;          // a compaction produced a list of another length
  unsigned int bm_pad;
  int bm_valid[2];              // bm[i] holds exactly list i's members (else it is all zero)
  int hp_dense;                 // HP: this window step's list is rebuilt in id order from the cell tags
  unsigned int tag_ctr;         // k_tag_compact cursor
  // EP on unweighted graphs inside the cluster loop: the level of each listed
  // edge's source, written at push time next to the edge (lists 0 / 1)
  uint32_t* ep_dn[2];
};

// --------------------------------------------------------- device graph ---
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Workspace {
  DevBuf dist, stamp, q[4];
  DevBuf wd_items[2], wd_tiles[2];           // WD item lists + tile_first (double-buffered)
  DevBuf scan_flags, scan_vals;              // decoupled look-back state
  DevBuf stats;                              // LaunchStats[kMaxLaunchSlots]
  DevBuf ctrl;                               // DevCtrl
  DevBuf ns_row, ns_col, ns_w, ns_parent, ns_cs, ns_tmp;  // NS split graph
  DevBuf ep_src, eq[2];                      // EP COO src + edge worklists
  DevBuf out64;                              // widened distances
  DevBuf recs;                               // DevRecord[kMaxRecords]
  DevBuf misc;
  DevBuf hist;                               // histogram counts
  DevBuf tile_node;                          // first node of every edge tile
  DevBuf misc_small, shard_tmp;              // sharded-run counters / local split
  DevBuf hp_big;                             // HP CTA-bin entries
  DevBuf ptw;                                // per-thread work lists (instrumented runs)
  DevBuf bm;                                 // BS frontier bitmaps (two lists)
  DevBuf ep_dn[2];                           // EP carried source levels (unweighted cluster loop)
  // every buffer above (glb_graph_destroy frees them all)
  template <class F>
  void each(F f) {
    for (DevBuf* b : {&dist, &stamp, &q[0], &q[1], &q[2], &q[3], &wd_items[0], &wd_items[1],
                      &wd_tiles[0], &wd_tiles[1], &scan_flags, &scan_vals, &stats, &ctrl, &ns_row,
                      &ns_col, &ns_w, &ns_parent, &ns_cs, &ns_tmp, &ep_src, &eq[0], &eq[1], &out64,
                      &recs, &misc, &hist, &tile_node, &misc_small, &shard_tmp, &hp_big, &ptw, &bm,
                      &ep_dn[0], &ep_dn[1]})
      f(*b);
  }
};
static_assert(sizeof(Workspace) == 35 * sizeof(DevBuf), "Workspace::each must list every buffer");

}  // namespace glb

namespace glb {
// One rank's part of a sharded run (glb_shard_* C-ABI, glb_driver.cu).
struct ShardSessionBase {
  virtual ~ShardSessionBase() {}
  virtual void local(int64_t* send_counts, unsigned long long* send, long long cap,
                     int64_t* local_next) = 0;
  virtual void apply(const unsigned long long* recv, long long n) = 0;
  virtual long long advance() = 0;
  virtual void finish(int64_t* dist_owned, glb_run_stats* st) = 0;
};
}  // namespace glb

namespace glb {
struct PeerTable;
}

// One rank of a peer-memory sharded run (glb_peer_* C-ABI, glb_driver.cu):
// the exchange region in this rank's HBM and every peer's region as mapped
// in this process.
struct glb_peer {
  glb_graph* g = nullptr;        // this rank's shard (not owned)
  int parts = 0, rank = 0;
  long long bounds[65] = {};
  char* region = nullptr;        // own exchange region (cudaMalloc: IPC-exportable)
  size_t region_bytes = 0;
  char* base[64] = {};           // every rank's region in this process's address space
  bool ipc_opened[64] = {};      // base[r] came from cudaIpcOpenMemHandle
  glb::PeerTable* table = nullptr;  // device table of the exchange kernels
  unsigned long long seq = 0;    // iterations exchanged so far (lockstep on every rank)
  int transport = 0;             // GLB_PEER_IPC / GLB_PEER_LOCAL once connected
  bool connected = false;
  bool poisoned = false;         // a timed-out exchange: the ranks are out of lockstep
  bool narrow_overflow[2] = {false, false};
};

struct glb_graph {
  int device = 0;
  int64_t n = 0, m = 0;
  bool weighted = false;
  int64_t max_degree = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int l2_bytes = 0;            // cudaDevAttrL2CacheSize
  int l2_persist_max = 0;      // cudaDevAttrMaxPersistingL2CacheSize (0: unsupported)
  int l2_window_max = 0;       // cudaDevAttrMaxAccessPolicyWindowSize
  long long* row = nullptr;
  uint32_t* col = nullptr;
  uint32_t* wt = nullptr;
  glb::Workspace ws;
  uint32_t stamp_epoch = 0;   // last stamp generation handed out
  uint32_t scan_epoch = 0;    // last look-back epoch handed out
  bool narrow_overflow[2] = {false, false};  // a 24-bit run overflowed (BFS, SSSP)
  void* host_ctrl = nullptr;  // pinned DevCtrl + stats mirror
  cudaEvent_t ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> ev_pool;
  std::vector<glb_record> last_records;  // records of the most recent glb_run
  long long ptw_len = 0;                 // per-thread work slots of the most recent glb_run
  long long ptw_dirty = -1;              // slots of the list buffer that may be nonzero (-1: all)
  glb::ShardSessionBase* shard = nullptr;                       // sharded run in progress
  std::mutex mu;              // drivers are not re-entrant (common.py:5-6)
};

namespace glb {

// -------------------------------------------------------- host helpers ---
// Device memory goes through the process-wide cache of glb_memory.cu; dfree
// requires that no queued work still uses the block.
void* dmalloc(size_t bytes);
void dfree(void* p);
size_t release_cached(int device);  // device < 0: every device
void* ensure(DevBuf& b, size_t bytes);  // grow-only device allocation (contents undefined)
void* ensure_zero(DevBuf& b, size_t bytes, cudaStream_t s);  // ... zeroed when (re)acquired
void free_buf(DevBuf& b);
constexpr size_t kPinnedSmallBytes = size_t(1) << 16;
void* pinned_small_get();  // pooled pinned block of kPinnedSmallBytes
void pinned_small_put(void* p);
unsigned host_workers();
// staged transfers (glb_memory.cu)
void upload_rows(glb_graph* g, const int64_t* row, long long n, long long m, long long* d_row,
                 long long* max_degree);
void upload_narrow(glb_graph* g, const int64_t* src, long long count, uint32_t* d_dst,
                   unsigned long long limit, bool allow_u8, void* d_scratch, const char* what);
void download_dist_u32(cudaStream_t s, const uint32_t* d_src, long long count, int64_t* out);
constexpr size_t kUploadScratchBytes = size_t(32) << 20;  // u8 weight chunks on the device
int max_resident_blocks(const void* kernel, int block, size_t smem, int num_sms);

inline unsigned int grid_for(long long items, int per_block, int cap) {
  long long b = (items + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned int)b;
}

// ------------------------------------------------------ device helpers ---
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: a step's first kernel lets the second one
// launch early (its CTAs wait in griddepcontrol.wait until the first grid has
// finished and its writes are visible), hiding the second launch's latency.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifndef GLB_STREAM_POLICY
#define GLB_STREAM_POLICY 1  // evict-first L2 policy on the col / weight streams
#endif
// Single-use streams (col / weights): an L2 evict-first access policy, made
// once per thread, so a pass over the 537 MB edge arrays does not push the
// randomly re-read distance cells out of L2 (ncu: with plain or .cs loads
// every sector of the stream is allocated evict_normal).
__device__ __forceinline__ unsigned long long l2_evict_first() {
#if GLB_STREAM_POLICY
  unsigned long long p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
#else
  return 0;
#endif
}
__device__ __forceinline__ uint32_t ld_stream_pol(const uint32_t* p, unsigned long long pol) {
#if GLB_STREAM_POLICY
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
#else
  (void)pol;
  return __ldg(p);
#endif
}

// Warp-aggregated append (one atomicAdd per converged group) -- the device
// form of wl_push_node's cursor bump (worklist.py:107-130).
__device__ __forceinline__ void q_append(uint32_t* q, unsigned int* cursor,
                                         uint32_t item) {
  unsigned mask = __activemask();
  unsigned leader = __ffs(mask) - 1;
  unsigned rank = __popc(mask & ((1u << lane_id()) - 1u));
  unsigned base = 0;
  if (lane_id() == leader) base = atomicAdd(cursor, (unsigned)__popc(mask));
  base = __shfl_sync(mask, base, leader);
  q[base + rank] = item;
}

// Dedup test-and-set: the first thread to stamp `v` with generation `gen`
// wins (replaces Worklist.flags + clear(), worklist.py:68-75,107-130).
__device__ __forceinline__ bool claim(uint32_t* stamp, uint32_t v, uint32_t gen) {
  if (stamp[v] == gen) return false;
  return atomicExch(stamp + v, gen) != gen;
}

// atomic_relax_min (engine.py:120-139) on a cell: plain-load pre-check
// (sound because cells only decrease), then atomicMin.  Returns true iff the
// distance strictly decreased; *first tells whether this is the first such
// decrease in generation `gen` (packed cells) -- the caller pushes then.
template <typename D>
__device__ __forceinline__ bool relax_cell(CellS<D>* cells, uint32_t v, D cand, uint32_t gen,
                                           bool* first) {
  const CellS<D> cur = cells[v];
  if (cand >= Cell<D>::dist(cur)) return false;
  const CellS<D> old = atomicMin(cells + v, Cell<D>::make(cand, gen));
  if (cand >= Cell<D>::dist(old)) return false;
  *first = Cell<D>::gen(old) != Cell<D>::tag(gen);
  return true;
}

// Candidate distance with overflow detection for the u32 path.
template <typename D>
__device__ __forceinline__ bool make_cand(D dn, uint32_t w, D& cand, unsigned int* ovf) {
  unsigned long long c = (unsigned long long)dn + (unsigned long long)w;
  if (c >= (unsigned long long)DistTraits<D>::kInf) {
    atomicOr(ovf, 1u);
    return false;
  }
  cand = (D)c;
  return true;
}

// Per-thread counters reduced per warp then spread across kStatSlots.
struct ThreadCounters {
  unsigned long long work = 0;
  unsigned long long relax = 0;
  unsigned long long push = 0;
};

__device__ __forceinline__ void flush_counters(LaunchStats* ls, const ThreadCounters& c);

// Per-thread work into the instrumented run's list (atomic: HP's window and
// CTA-bin kernels are one launch of the record), then the summed counters.
__device__ __forceinline__ void flush_counters(DevCtrl* ctrl, const ThreadCounters& c) {
  uint32_t* ptw = ctrl->ptw;
  if (ptw && c.work) {
    const unsigned long long i =
        ctrl->ptw_off + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ctrl->ptw_cap)
      atomicAdd(ptw + i, c.work > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c.work);
  }
  flush_counters(ctrl->ls, c);
}

__device__ __forceinline__ void flush_counters(LaunchStats* ls, const ThreadCounters& c) {
  unsigned long long w = c.work, r = c.relax, p = c.push, sq = c.work * c.work, mx = c.work;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    w += __shfl_xor_sync(0xffffffffu, w, off);
    r += __shfl_xor_sync(0xffffffffu, r, off);
    p += __shfl_xor_sync(0xffffffffu, p, off);
    sq += __shfl_xor_sync(0xffffffffu, sq, off);
    unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = o > mx ? o : mx;
  }
  // sums in 64-bit shared atomics (native adds); the per-thread maximum in a
  // 32-bit one (a 64-bit shared atomicMax is a CAS loop)
  __shared__ unsigned long long s_acc[4];
  __shared__ unsigned int s_max;
  if (threadIdx.x < 4) s_acc[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  if (lane_id() == 0) {
    atomicAdd(&s_acc[0], w);
    atomicAdd(&s_acc[1], r);
    atomicAdd(&s_acc[2], p);
    atomicAdd(&s_acc[3], sq);
    atomicMax(&s_max, mx > 0xFFFFFFFFull ? 0xFFFFFFFFu : (unsigned)mx);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    StatSlot& s = ls->slot[blockIdx.x % kStatSlots];
    if (s_acc[0]) atomicAdd(&s.work, s_acc[0]);
    if (s_acc[1]) atomicAdd(&s.relax, s_acc[1]);
    if (s_acc[2]) atomicAdd(&s.push, s_acc[2]);
    if (s_acc[3]) atomicAdd(&s.work_sq, s_acc[3]);
    if (s_max) atomicMax(&s.work_max, (unsigned long long)s_max);
  }
}

}  // namespace glb
