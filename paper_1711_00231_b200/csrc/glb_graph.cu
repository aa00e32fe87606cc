// glb_graph.cu -- graph upload (CsrGraph, csr.py:42-118), degree analysis
// (degrees.py:27-76), COO expansion (csr.py:155-170), node splitting
// (splitting.py:58-99) and the device primitives behind inclusive_scan
// (scan.py:19-65) and find_offsets (workload.py:45-72).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "glb_internal.cuh"
#include "glb_scan.cuh"
#include "glb_tiles.cuh"

namespace glb {

// ======================================================== error plumbing ===
static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

void* ensure(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return b.p;
  if (b.p) {  // queued work may still read the old block: drain before recycling it
    GLB_CUDA_TRY(cudaDeviceSynchronize());
    dfree(b.p);
  }
  b.p = nullptr;
  b.bytes = 0;
  b.p = dmalloc(bytes);
  b.bytes = bytes;
  return b.p;
}

// A recycled block holds another graph's data: buffers whose protocol needs
// zeros (look-back flags, stamps, counters) are cleared whenever they are
// (re)acquired.
void* ensure_zero(DevBuf& b, size_t bytes, cudaStream_t s) {
  const bool grow = b.bytes < (bytes ? bytes : 16);
  void* p = ensure(b, bytes);
  if (grow) GLB_CUDA_TRY(cudaMemsetAsync(p, 0, b.bytes, s));
  return p;
}

void free_buf(DevBuf& b) {
  if (b.p) dfree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

int max_resident_blocks(const void* kernel, int block, size_t smem, int num_sms) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return per_sm * num_sms;
}

// ========================================================== graph upload ===
// Narrow int64 -> uint32 with 128-bit loads (two int64 per ld.v2.s64) and a
// range check [0, limit); any violation sets *bad.
__global__ void k_narrow_u32(const long long* __restrict__ src, uint32_t* __restrict__ dst,
                             long long count, unsigned long long limit, unsigned int* bad,
                             unsigned int bad_code) {
  long long pairs = count >> 1;
  const longlong2* s2 = reinterpret_cast<const longlong2*>(src);
  uint2* d2 = reinterpret_cast<uint2*>(dst);
  bool err = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < pairs;
       i += (long long)gridDim.x * blockDim.x) {
    longlong2 v = __ldcs(s2 + i);
    err |= (unsigned long long)v.x >= limit || (unsigned long long)v.y >= limit;
    d2[i] = make_uint2((uint32_t)v.x, (uint32_t)v.y);
  }
  if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    long long v = src[count - 1];
    err |= (unsigned long long)v >= limit;
    dst[count - 1] = (uint32_t)v;
  }
  if (err) atomicOr(bad, bad_code);
}

// Row-offset invariants (csr.py:74-79) + max outdegree.
__global__ void k_check_rows(const long long* __restrict__ row, long long n, long long m,
                             unsigned int* bad, unsigned long long* max_deg) {
  unsigned long long mx = 0;
  bool err = false;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    long long d = row[v + 1] - row[v];
    err |= d < 0;
    if (d > 0 && (unsigned long long)d > mx) mx = (unsigned long long)d;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) err |= (row[0] != 0) || (row[n] != m);
  for (int off = 16; off > 0; off >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, off);
    mx = o > mx ? o : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_deg, mx);
  if (err) atomicOr(bad, 1u);
}

void rmat_device(glb_graph* g, int scale, long long edge_factor, double t_a, double t_ab,
                 double t_abc, const unsigned long long state[2], const unsigned long long inc[2],
                 bool weighted, long long max_weight);

void measure_gather(glb_graph* g, double out[4]);

void graph_upload(glb_graph* g, const int64_t* row, const int64_t* col, const int64_t* w) {
  g->row = (long long*)dmalloc((size_t)(g->n + 1) * 8);
  g->col = (uint32_t*)dmalloc((size_t)std::max<long long>(g->m, 1) * 4 + kEdgePad);
  if (w) g->wt = (uint32_t*)dmalloc((size_t)std::max<long long>(g->m, 1) * 4 + kEdgePad);
  long long mx = 0;
  upload_rows(g, row, g->n, g->m, g->row, &mx);
  upload_narrow(g, col, g->m, g->col, (unsigned long long)g->n, false, nullptr,
                "col_indices contains a node id out of range");
  if (w) {
    void* scratch = ensure(g->ws.misc, kUploadScratchBytes);
    upload_narrow(g, w, g->m, g->wt, 0x100000000ull, true, scratch,
                  "edge weights must be nonnegative and below 2^32 on the device");
  }
  g->max_degree = mx;
}

// ======================================================= degree analysis ===
__global__ void k_degree_sq(const long long* __restrict__ row, long long n,
                            unsigned long long* sumsq_hi, double* dummy) {
  // sum of squared outdegrees, exact in 64 bits for degree < 2^32
  unsigned long long acc = 0;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    unsigned long long d = (unsigned long long)(row[v + 1] - row[v]);
    acc += d * d;
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(sumsq_hi, acc);
}

// degree d > 0 -> bin ceil(d*B/max) (1-based), degree 0 -> bin 1 (degrees.py:55-60).
// Lanes holding the same bin are merged with __match_any before the shared
// atomic, so a 10-bin histogram does not serialise 32 lanes on one word.
__global__ void k_histogram(const long long* __restrict__ row, long long n, int bins,
                            unsigned long long max_deg, unsigned long long* counts) {
  extern __shared__ unsigned long long s_cnt[];
  const bool smem = bins <= 4096;
  const bool narrow = max_deg <= (0x7FFFFFFFFFFFFFFFull / ((unsigned long long)bins + 1));
  if (smem)
    for (int b = threadIdx.x; b < bins; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = blockIdx.x * (long long)blockDim.x; base < n; base += stride) {
    const long long v = base + threadIdx.x;
    unsigned long long bin = 0;  // 0 = no node
    if (v < n) {
      const unsigned long long d = (unsigned long long)(row[v + 1] - row[v]);
      bin = 1;
      if (max_deg > 0 && d > 0) {
        if (narrow)
          bin = (d * (unsigned)bins + (max_deg - 1)) / max_deg;
        else
          bin = (unsigned long long)(((unsigned __int128)d * (unsigned)bins + (max_deg - 1)) /
                                     max_deg);
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin != 0 && (int)lane_id() == __ffs(peers) - 1) {
      const unsigned long long c = (unsigned long long)__popc(peers);
      if (smem)
        atomicAdd(&s_cnt[bin - 1], c);
      else
        atomicAdd(&counts[bin - 1], c);
    }
  }
  __syncthreads();
  if (smem)
    for (int b = threadIdx.x; b < bins; b += blockDim.x)
      if (s_cnt[b]) atomicAdd(&counts[b], s_cnt[b]);
}

void degree_stats(glb_graph* g, int64_t* max_degree, int64_t* sum_degree, double* sum_sq) {
  DevCtrl* ctrl = (DevCtrl*)ensure(g->ws.ctrl, sizeof(DevCtrl));
  GLB_CUDA_TRY(cudaMemsetAsync(&ctrl->aux[1], 0, 8, g->stream));
  if (g->n > 0) {
    unsigned grid = grid_for(g->n, kBlock, g->num_sms * 8);
    k_degree_sq<<<grid, kBlock, 0, g->stream>>>(g->row, g->n,
                                                (unsigned long long*)&ctrl->aux[1], nullptr);
    GLB_CHECK_LAUNCH();
  }
  unsigned long long sq = 0;
  GLB_CUDA_TRY(cudaMemcpyAsync(&sq, &ctrl->aux[1], 8, cudaMemcpyDeviceToHost, g->stream));
  GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  *max_degree = g->max_degree;
  *sum_degree = g->m;
  *sum_sq = (double)sq;
}

void histogram(glb_graph* g, const long long* row, long long n, unsigned long long max_deg,
               int bins, int64_t* counts_out, int32_t* arg_max_bin, int64_t* mdt) {
  unsigned long long* d_counts = (unsigned long long*)ensure(g->ws.hist, (size_t)bins * 8);
  {
    GLB_CUDA_TRY(cudaMemsetAsync(d_counts, 0, (size_t)bins * 8, g->stream));
    if (n > 0) {
      unsigned grid = grid_for(n, kBlock, g->num_sms * 8);
      size_t smem = bins <= 4096 ? (size_t)bins * 8 : 0;
      k_histogram<<<grid, kBlock, smem, g->stream>>>(row, n, bins, max_deg, d_counts);
      GLB_CHECK_LAUNCH();
    }
    std::vector<unsigned long long> h(bins);
    GLB_CUDA_TRY(cudaMemcpyAsync(h.data(), d_counts, (size_t)bins * 8, cudaMemcpyDeviceToHost,
                                 g->stream));
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
    // first argmax (degrees.py:62) and mdt = max(1, bin*max // B) (degrees.py:72-76)
    int arg = 0;
    for (int b = 0; b < bins; ++b) {
      if (counts_out) counts_out[b] = (int64_t)h[b];
      if (h[b] > h[arg]) arg = b;
    }
    if (arg_max_bin) *arg_max_bin = arg + 1;
    if (mdt) {
      unsigned __int128 num = (unsigned __int128)(arg + 1) * max_deg;
      unsigned long long v = (unsigned long long)(num / (unsigned)bins);
      *mdt = (int64_t)std::max<unsigned long long>(1, v);
    }
  }
}

// ========================================================= COO expansion ===
// src[e] = v for e in [row[v], row[v+1]) -- np.repeat(arange(n), outdeg),
// csr.py:168.  Edge tiles: coalesced writes, no per-node serial loops.
__global__ void __launch_bounds__(kBlock) k_coo_src(const long long* __restrict__ row, long long n,
                                                    long long m,
                                                    const unsigned int* __restrict__ tile_node,
                                                    uint32_t* __restrict__ src) {
  __shared__ __align__(16) int s_head[kEdgeTile];
  __shared__ uint32_t s_v[kEdgeTile];
  __shared__ typename cub::BlockScan<int, kBlock>::TempStorage ts;
  const long long ntiles = (m + kEdgeTile - 1) / kEdgeTile;
  for (long long b = blockIdx.x; b < ntiles; b += gridDim.x) {
    const long long e0 = b * kEdgeTile, e1 = e0 + kEdgeTile < m ? e0 + kEdgeTile : m;
    const long long v0 = tile_node[b];
    const long long v1 = b + 1 < ntiles ? (long long)tile_node[b + 1] : n - 1;
    tile_heads(row, v0, v1, e0, e1, s_head, ts, [&](long long v, int h) { s_v[h] = (uint32_t)v; });
#pragma unroll
    for (int k = 0; k < kEdgeEPT; ++k) {
      const int local = k * kBlock + threadIdx.x;
      if (e0 + local < e1) src[e0 + local] = s_v[s_head[local]];
    }
    __syncthreads();
  }
}

void coo_src(glb_graph* g, uint32_t* d_src) {
  if (g->n == 0 || g->m == 0) return;
  const long long ntiles = (g->m + kEdgeTile - 1) / kEdgeTile;
  unsigned* tile_node = (unsigned*)ensure(g->ws.ns_tmp, (size_t)(ntiles + 1) * 4);
  k_tile_nodes<<<grid_for(g->n, kBlock, g->num_sms * 8), kBlock, 0, g->stream>>>(g->row, g->n,
                                                                                 tile_node);
  GLB_CHECK_LAUNCH();
  k_coo_src<<<grid_for(ntiles, 1, g->num_sms * 4), kBlock, 0, g->stream>>>(g->row, g->n, g->m,
                                                                           tile_node, d_src);
  GLB_CHECK_LAUNCH();
}

__global__ void k_widen_u32_to_i64(const uint32_t* __restrict__ s, long long* __restrict__ d,
                                   long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = (long long)s[i];
}

// ========================================================= node splitting ===
// Per-node scan vector: {children, parent edges, excess edges, split nodes}.
constexpr int kSplitIPT = 4;
constexpr int kSplitTile = kBlock * kSplitIPT;

__global__ void __launch_bounds__(kBlock) k_split_scan(const long long* __restrict__ row, long long n,
                                                       long long mdt, LookbackState<4> lb,
                                                       unsigned epoch, long long* __restrict__ cs,
                                                       long long* __restrict__ new_row,
                                                       long long* __restrict__ excess_pre,
                                                       long long* totals) {
  using TS = TileScan<4, kBlock>;
  __shared__ typename TS::Storage st;
  long long ntiles = (n + kSplitTile - 1) / kSplitTile;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    Vec<4> item[kSplitIPT];
    Vec<4> sum;
    long long first = t * kSplitTile + (long long)threadIdx.x * kSplitIPT;
#pragma unroll
    for (int k = 0; k < kSplitIPT; ++k) {
      long long v = first + k;
      if (v < n) {
        long long d = row[v + 1] - row[v];
        long long pieces = d > 0 ? (d + mdt - 1) / mdt : 1;  // max(1, ceil(d/mdt))
        long long keep = d < mdt ? d : mdt;
        item[k].w[0] = pieces - 1;
        item[k].w[1] = keep;
        item[k].w[2] = d - keep;
        item[k].w[3] = d > mdt ? 1 : 0;
      }
      sum = sum + item[k];
    }
    Vec<4> incl;
    Vec<4> ex = TS::run(st, lb, epoch, t, sum, incl);
#pragma unroll
    for (int k = 0; k < kSplitIPT; ++k) {
      long long v = first + k;
      if (v < n) {
        cs[v] = ex.w[0];
        new_row[v] = ex.w[1];
        excess_pre[v] = ex.w[2];
      }
      ex = ex + item[k];
    }
    if (t == ntiles - 1 && threadIdx.x == 0) {
      cs[n] = incl.w[0];
      totals[0] = incl.w[0];
      totals[1] = incl.w[1];
      totals[2] = incl.w[2];
      totals[3] = incl.w[3];
    }
  }
}

// Parent keeps its first mdt edges; children take the following mdt-chunks,
// laid out after all parents' chunks (splitting.py:72-99).  Edge e of node v
// at local offset j moves to new_row[v] + j (j < mdt) or to
// ptotal + excess_pre[v] + (j - mdt): one coalesced pass over the edge tiles.
template <bool W>
__global__ void __launch_bounds__(kBlock) k_split_scatter(
    const long long* __restrict__ row, const uint32_t* __restrict__ col,
    const uint32_t* __restrict__ wt, long long n, long long m, long long mdt,
    const unsigned int* __restrict__ tile_node, const long long* __restrict__ new_row,
    const long long* __restrict__ excess_pre, const long long* __restrict__ totals,
    uint32_t* __restrict__ new_col, uint32_t* __restrict__ new_w) {
  __shared__ __align__(16) int s_head[kEdgeTile];
  __shared__ uint32_t s_v[kEdgeTile];
  __shared__ typename cub::BlockScan<int, kBlock>::TempStorage ts;
  const long long ptotal = totals[1];
  const long long ntiles = (m + kEdgeTile - 1) / kEdgeTile;
  for (long long b = blockIdx.x; b < ntiles; b += gridDim.x) {
    const long long e0 = b * kEdgeTile, e1 = e0 + kEdgeTile < m ? e0 + kEdgeTile : m;
    const long long v0 = tile_node[b];
    const long long v1 = b + 1 < ntiles ? (long long)tile_node[b + 1] : n - 1;
    tile_heads(row, v0, v1, e0, e1, s_head, ts, [&](long long v, int h) { s_v[h] = (uint32_t)v; });
#pragma unroll
    for (int k = 0; k < kEdgeEPT; ++k) {
      const int local = k * kBlock + threadIdx.x;
      const long long e = e0 + local;
      if (e < e1) {
        const uint32_t v = s_v[s_head[local]];
        const long long j = e - __ldg(row + v);
        const long long dst =
            j < mdt ? __ldg(new_row + v) + j : ptotal + __ldg(excess_pre + v) + (j - mdt);
        new_col[dst] = __ldcs(col + e);
        if (W) new_w[dst] = __ldcs(wt + e);
      }
    }
    __syncthreads();
  }
}

// Child row offsets and parent_of for every split node.
__global__ void k_split_children(const long long* __restrict__ row, long long n, long long m,
                                 long long mdt, const long long* __restrict__ cs,
                                 const long long* __restrict__ excess_pre,
                                 const long long* __restrict__ totals, long long* __restrict__ new_row,
                                 long long* __restrict__ parent_of) {
  const long long ptotal = totals[1];
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const long long c0 = cs[v], c1 = cs[v + 1];
    const long long base = ptotal + excess_pre[v];
    for (long long k = 0; k < c1 - c0; ++k) {
      new_row[n + c0 + k] = base + k * mdt;
      parent_of[c0 + k] = v;
    }
    if (v == 0) new_row[n + totals[0]] = m;
  }
}

// Split graph on the device; returns totals {children, parent edges, excess, split nodes}.
void split_device(glb_graph* g, long long mdt, long long totals_out[4]) {
  Workspace& ws = g->ws;
  long long n = g->n, m = g->m;
  long long* cs = (long long*)ensure(ws.ns_cs, (size_t)(n + 1) * 8);
  long long* exc = (long long*)ensure(ws.ns_tmp, (size_t)(n + 1) * 8 + 64);
  long long* totals = exc + (n + 1);
  // scan look-back state
  long long ntiles = (n + kSplitTile - 1) / kSplitTile;
  unsigned* flags =
      (unsigned*)ensure_zero(ws.scan_flags, (size_t)std::max<long long>(ntiles, 1) * 4 + 4096, g->stream);
  size_t vbytes = (size_t)std::max<long long>(ntiles, 1) * sizeof(Vec<4>);
  char* vals = (char*)ensure(ws.scan_vals, 2 * vbytes + 4096);
  LookbackState<4> lb{flags, (Vec<4>*)vals, (Vec<4>*)(vals + vbytes)};
  // parents' row offsets live in the first n entries of new_row; sized after the scan
  long long* tmp_row = (long long*)ensure(ws.ns_row, (size_t)(n + 1) * 8);
  GLB_CUDA_TRY(cudaMemsetAsync(totals, 0, 64, g->stream));
  if (n > 0) {
    unsigned epoch = ++g->scan_epoch;
    int cap = max_resident_blocks((const void*)k_split_scan, kBlock, 0, g->num_sms);
    unsigned grid = grid_for(ntiles, 1, cap);
    k_split_scan<<<grid, kBlock, 0, g->stream>>>(g->row, n, mdt, lb, epoch, cs, tmp_row, exc,
                                                 totals);
    GLB_CHECK_LAUNCH();
  } else {
    GLB_CUDA_TRY(cudaMemsetAsync(cs, 0, 8, g->stream));
  }
  GLB_CUDA_TRY(cudaMemcpyAsync(totals_out, totals, 32, cudaMemcpyDeviceToHost, g->stream));
  GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  long long nchild = totals_out[0];
  long long new_n = n + nchild;
  // grow new_row preserving the parent prefix already written
  if (ws.ns_row.bytes < (size_t)(new_n + 1) * 8) {
    DevBuf nb;
    ensure(nb, (size_t)(new_n + 1) * 8);
    GLB_CUDA_TRY(cudaMemcpyAsync(nb.p, ws.ns_row.p, (size_t)n * 8, cudaMemcpyDeviceToDevice,
                                 g->stream));
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
    free_buf(ws.ns_row);
    ws.ns_row = nb;
  }
  long long* new_row = (long long*)ws.ns_row.p;
  uint32_t* new_col = (uint32_t*)ensure(ws.ns_col, (size_t)std::max<long long>(m, 1) * 4 + kEdgePad);
  uint32_t* new_w = g->wt ? (uint32_t*)ensure(ws.ns_w, (size_t)std::max<long long>(m, 1) * 4 + kEdgePad) : nullptr;
  long long* parent_of = (long long*)ensure(ws.ns_parent, (size_t)std::max<long long>(nchild, 1) * 8);
  if (n > 0) {
    const long long etiles = (m + kEdgeTile - 1) / kEdgeTile;
    if (m > 0) {
      unsigned* tile_node = (unsigned*)ensure(ws.tile_node, (size_t)(etiles + 1) * 4);
      k_tile_nodes<<<grid_for(n, kBlock, g->num_sms * 8), kBlock, 0, g->stream>>>(g->row, n,
                                                                                 tile_node);
      GLB_CHECK_LAUNCH();
      const unsigned egrid = grid_for(etiles, 1, g->num_sms * 4);
      if (g->wt)
        k_split_scatter<true><<<egrid, kBlock, 0, g->stream>>>(g->row, g->col, g->wt, n, m, mdt,
                                                               tile_node, new_row, exc, totals,
                                                               new_col, new_w);
      else
        k_split_scatter<false><<<egrid, kBlock, 0, g->stream>>>(g->row, g->col, g->wt, n, m, mdt,
                                                                tile_node, new_row, exc, totals,
                                                                new_col, new_w);
      GLB_CHECK_LAUNCH();
    }
    k_split_children<<<grid_for(n, kBlock, g->num_sms * 8), kBlock, 0, g->stream>>>(
        g->row, n, m, mdt, cs, exc, totals, new_row, parent_of);
    GLB_CHECK_LAUNCH();
  } else {
    long long mm = m;
    GLB_CUDA_TRY(cudaMemcpyAsync(new_row, &mm, 8, cudaMemcpyHostToDevice, g->stream));
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  }
}

// =================================================== scan / find_offsets ===
constexpr int kScanIPT = 8;
constexpr int kScanTile = kBlock * kScanIPT;

// Inclusive int64 scan with first-overflow detection (scan.py:19-65).
__global__ void __launch_bounds__(kBlock) k_inclusive_scan(const long long* __restrict__ in,
                                                           long long n, long long* __restrict__ out,
                                                           LookbackState<1> lb, unsigned epoch,
                                                           unsigned int* ovf) {
  using TS = TileScan<1, kBlock>;
  __shared__ typename TS::Storage st;
  long long ntiles = (n + kScanTile - 1) / kScanTile;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    long long x[kScanIPT];
    Vec<1> sum;
    long long first = t * kScanTile + (long long)threadIdx.x * kScanIPT;
#pragma unroll
    for (int k = 0; k < kScanIPT; ++k) {
      x[k] = first + k < n ? in[first + k] : 0;
      sum.w[0] = (long long)((unsigned long long)sum.w[0] + (unsigned long long)x[k]);
    }
    Vec<1> incl;
    Vec<1> ex = TS::run(st, lb, epoch, t, sum, incl);
    long long run = ex.w[0];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < kScanIPT; ++k) {
      long long nxt = (long long)((unsigned long long)run + (unsigned long long)x[k]);
      // the first signed overflow is visible locally: operands agree in sign, result differs
      bad |= ((run ^ nxt) & (x[k] ^ nxt)) < 0;
      if (first + k < n) out[first + k] = nxt;
      run = nxt;
    }
    if (bad) atomicOr(ovf, 1u);
  }
}

// bisect_right(prefix, t*ept) per thread (workload.py:45-72)
__global__ void k_find_offsets(const long long* __restrict__ prefix, long long size, long long ept,
                               long long threads, long long* node_off, long long* edge_off) {
  long long total = size > 0 ? prefix[size - 1] : 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < threads;
       t += (long long)gridDim.x * blockDim.x) {
    long long start = t * ept;
    if (start >= total || (ept > 0 && start / ept != t)) {
      node_off[t] = -1;
      edge_off[t] = 0;
      continue;
    }
    long long lo = 0, hi = size;  // first j with prefix[j] > start
    while (lo < hi) {
      long long mid = (lo + hi) >> 1;
      if (prefix[mid] <= start)
        lo = mid + 1;
      else
        hi = mid;
    }
    node_off[t] = lo;
    edge_off[t] = start - (lo ? prefix[lo - 1] : 0);
  }
}


// ------------------------------------------------ distance certificate ---
// glb_validate: proves a BFS/SSSP distance array correct without an oracle
// (the check run_benchmark(verify=True) needs, bench.py:186-196 /
// oracles.py:58-82).  With w(e) = 1 for BFS and unweighted SSSP:
//   (1) d[src] == 0;
//   (2) every edge u->v out of a reached u has d[v] <= d[u] + w  (so d is at
//       most the true distance and every truly reachable node is reached);
//   (3) every reached node is reachable from src over tight edges
//       (d[u] + w == d[v]), so d[v] is the length of a real path, i.e. at
//       least the true distance.  Zero-weight edges are fine: tightness is
//       followed from the source, not from the node.
// A node violating any rule gets a flag; the call returns their count and
// the smallest flagged id.
constexpr long long kInf64 = 0x7FFFFFFFFFFFFFFFll;

__device__ __forceinline__ unsigned long long val_w(const uint32_t* wt, long long e) {
  return wt ? (unsigned long long)__ldg(wt + e) : 1ull;
}

// (2) and (1): warp per node, lanes over its out-edges
__global__ void k_val_edges(const long long* __restrict__ row, const uint32_t* __restrict__ col,
                            const uint32_t* __restrict__ wt, long long n,
                            const long long* __restrict__ d, long long src,
                            unsigned char* __restrict__ bad) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  for (long long u = warp; u < n; u += nwarps) {
    const long long du = d[u];
    if (lane == 0 && (du < 0 || (u == src && du != 0))) bad[u] = 1;
    if (du < 0 || du == kInf64) continue;
    const long long lo = row[u], hi = row[u + 1];
    for (long long e = lo + lane; e < hi; e += 32) {
      const uint32_t v = __ldg(col + e);
      const long long dv = d[v];
      if (dv == kInf64 || (unsigned long long)dv > (unsigned long long)du + val_w(wt, e)) bad[v] = 1;
    }
  }
}

// (3): one level of the tight-edge BFS from the source, warp per node
__global__ void k_val_tight(const long long* __restrict__ row, const uint32_t* __restrict__ col,
                            const uint32_t* __restrict__ wt, const long long* __restrict__ d,
                            const uint32_t* __restrict__ qin, const unsigned* nin,
                            uint32_t* __restrict__ qout, unsigned* nout,
                            unsigned* __restrict__ seen) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31u;
  const long long cnt = *nin;
  for (long long i = warp; i < cnt; i += nwarps) {
    const uint32_t u = qin[i];
    const unsigned long long du = (unsigned long long)d[u];
    const long long lo = row[u], hi = row[u + 1];
    for (long long e = lo + lane; e < hi; e += 32) {
      const uint32_t v = __ldg(col + e);
      if ((unsigned long long)d[v] == du + val_w(wt, e) && atomicExch(seen + v, 1u) == 0u)
        qout[atomicAdd(nout, 1u)] = v;
    }
  }
}

// reached but not tight-reachable -> flagged; then count + smallest flagged id
__global__ void k_val_finish(const long long* __restrict__ d, const unsigned* __restrict__ seen,
                             unsigned char* __restrict__ bad, long long n,
                             unsigned long long* __restrict__ out /* [count, min id] */) {
  unsigned long long c = 0, first = ~0ull;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const long long dv = d[v];
    bool b = bad[v] != 0 || (dv >= 0 && dv != kInf64 && !seen[v]);
    if (b) {
      ++c;
      if ((unsigned long long)v < first) first = (unsigned long long)v;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, off);
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, first, off);
    first = o < first ? o : first;
  }
  if ((threadIdx.x & 31u) == 0 && c) {
    atomicAdd(out, c);
    atomicMin(out + 1, first);
  }
}

__global__ void k_val_seed(const long long* d, long long src, uint32_t* q, unsigned* nq,
                           unsigned* seen) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const bool ok = d[src] == 0;
    *nq = ok ? 1u : 0u;
    if (ok) {
      q[0] = (uint32_t)src;
      seen[src] = 1u;
    }
  }
}

void validate(glb_graph* g, bool weights, long long src, const int64_t* dist, long long* n_bad,
              long long* first_bad) {
  Workspace& ws = g->ws;
  const long long n = g->n;
  const size_t nb = (size_t)std::max<long long>(n, 1);
  cudaStream_t s = g->stream;
  long long* d = (long long*)ensure(ws.out64, nb * 8);
  uint32_t* q[2] = {(uint32_t*)ensure(ws.q[0], nb * 4), (uint32_t*)ensure(ws.q[1], nb * 4)};
  char* flags = (char*)ensure(ws.misc, nb * 5 + 64);
  unsigned* seen = (unsigned*)flags;
  unsigned char* bad = (unsigned char*)(flags + nb * 4);
  unsigned* counts = (unsigned*)ensure(ws.misc_small, 64);  // nq[2], out[2] (u64) at +16
  unsigned long long* out = (unsigned long long*)(counts + 4);
  GLB_CUDA_TRY(cudaMemcpyAsync(d, dist, (size_t)n * 8, cudaMemcpyHostToDevice, s));
  GLB_CUDA_TRY(cudaMemsetAsync(flags, 0, nb * 5, s));
  const unsigned long long init[2] = {0ull, ~0ull};
  GLB_CUDA_TRY(cudaMemcpyAsync(out, init, 16, cudaMemcpyHostToDevice, s));
  const uint32_t* wt = weights ? g->wt : nullptr;
  const unsigned grid = grid_for(n * 32, kBlock, g->num_sms * 8);
  k_val_edges<<<grid, kBlock, 0, s>>>(g->row, g->col, wt, n, d, src, bad);
  GLB_CHECK_LAUNCH();
  k_val_seed<<<1, 32, 0, s>>>(d, src, q[0], counts, seen);
  GLB_CHECK_LAUNCH();
  unsigned h_n = 1;
  for (int lvl = 0; h_n; ++lvl) {  // tight-edge BFS, one launch per level
    const int a = lvl & 1;
    GLB_CUDA_TRY(cudaMemsetAsync(counts + (a ^ 1), 0, 4, s));
    k_val_tight<<<grid, kBlock, 0, s>>>(g->row, g->col, wt, d, q[a], counts + a, q[a ^ 1],
                                         counts + (a ^ 1), seen);
    GLB_CHECK_LAUNCH();
    GLB_CUDA_TRY(cudaMemcpyAsync(&h_n, counts + (a ^ 1), 4, cudaMemcpyDeviceToHost, s));
    GLB_CUDA_TRY(cudaStreamSynchronize(s));
  }
  k_val_finish<<<grid_for(n, kBlock, g->num_sms * 8), kBlock, 0, s>>>(d, seen, bad, n, out);
  GLB_CHECK_LAUNCH();
  unsigned long long h[2];
  GLB_CUDA_TRY(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s));
  GLB_CUDA_TRY(cudaStreamSynchronize(s));
  *n_bad = (long long)h[0];
  *first_bad = h[0] ? (long long)h[1] : -1;
}

}  // namespace glb

// ================================================================ C-ABI ===
using glb::Error;
using namespace glb;

namespace {
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    GLB_CUDA_TRY(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return GLB_OK;
  } catch (const Error& e) {
    glb::set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    glb::set_error("host allocation failed");
    return GLB_ENOMEM;
  } catch (const std::exception& e) {
    glb::set_error(e.what());
    return GLB_ECUDA;
  }
}

void require_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    throw Error{GLB_ENODEV, "no CUDA device is visible"};
  if (device < 0 || device >= count)
    throw Error{GLB_EINVAL, "device ordinal " + std::to_string(device) + " out of range"};
}
}  // namespace

extern "C" {

const char* glb_last_error(void) { return glb::last_error(); }
const char* glb_version(void) { return "graphlb_b200 0.1.0 (sm_100a)"; }

uint64_t glb_kernel_launches(void) { return glb::g_launches.load(); }

int glb_device_count(int* count) {
  return guarded([&] {
    if (!count) throw Error{GLB_EINVAL, "count is NULL"};
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

int glb_graph_create(const int64_t* row_offsets, const int64_t* col, const int64_t* weights_or_null,
                     int64_t n, int64_t m, int device, glb_graph** out) {
  glb::NvtxRange nvtx_range("glb_graph_create (validate, narrow, upload)");
  return guarded([&] {
    if (!out) throw Error{GLB_EINVAL, "out is NULL"};
    *out = nullptr;
    if (n < 0 || m < 0) throw Error{GLB_EINVAL, "node and edge counts must be nonnegative"};
    if (!row_offsets || (m > 0 && !col)) throw Error{GLB_EINVAL, "row_offsets/col_indices is NULL"};
    if (n >= (int64_t)0xFFFFFFFFll) throw Error{GLB_EINVAL, "num_nodes must be below 2^32-1 on the device"};
    if (m >= (int64_t)0xFFFFFFFFll) throw Error{GLB_EINVAL, "num_edges must be below 2^32-1 on the device"};
    require_device(device);
    DeviceGuard dg(device);
    glb_graph* g = new glb_graph();
    try {
      g->device = device;
      g->n = n;
      g->m = m;
      g->weighted = weights_or_null != nullptr;
      GLB_CUDA_TRY(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
      GLB_CUDA_TRY(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
      GLB_CUDA_TRY(cudaDeviceGetAttribute(&g->l2_bytes, cudaDevAttrL2CacheSize, device));
      // Opt-in L2 persistence for the distance cells (GLB_L2_PERSIST=1).  It
      // carves the persisting set out of the 126 MB L2 for every kernel, and
      // measured slower on C2 than plain evict-first streaming, so it is off
      // by default.
      if (getenv("GLB_L2_PERSIST") &&
          (cudaDeviceGetAttribute(&g->l2_persist_max, cudaDevAttrMaxPersistingL2CacheSize,
                                  device) != cudaSuccess ||
           cudaDeviceGetAttribute(&g->l2_window_max, cudaDevAttrMaxAccessPolicyWindowSize,
                                  device) != cudaSuccess ||
           cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)g->l2_persist_max) !=
               cudaSuccess)) {
        cudaGetLastError();
        g->l2_persist_max = g->l2_window_max = 0;
      }
      GLB_CUDA_TRY(cudaEventCreate(&g->ev[0]));
      GLB_CUDA_TRY(cudaEventCreate(&g->ev[1]));
      g->host_ctrl = glb::pinned_small_get();
      glb::graph_upload(g, row_offsets, col, weights_or_null);
    } catch (...) {
      glb_graph_destroy(g);
      throw;
    }
    *out = g;
  });
}

int glb_graph_create_rmat(int scale, int64_t edge_factor, double t_a, double t_ab, double t_abc,
                          const uint64_t* state_hi_lo, const uint64_t* inc_hi_lo, int weighted,
                          int64_t max_weight, int device, glb_graph** out) {
  glb::NvtxRange nvtx_range("glb_graph_create_rmat (generate + CSR build in HBM)");
  return guarded([&] {
    if (!out || !state_hi_lo || !inc_hi_lo) throw Error{GLB_EINVAL, "NULL argument"};
    *out = nullptr;
    if (scale < 1 || scale > 31) throw Error{GLB_EINVAL, "scale must be in [1, 31]"};
    if (edge_factor < 0) throw Error{GLB_EINVAL, "edge_factor must be nonnegative"};
    if (((unsigned long long)edge_factor << scale) >= 0xFFFFFFFFull)
      throw Error{GLB_EINVAL, "the device generator needs fewer than 2^32 edges"};
    if (weighted && (max_weight < 1 || max_weight >= 0xFFFFFFFFll))
      throw Error{GLB_EINVAL, "max_weight must be in [1, 2^32-1)"};
    require_device(device);
    DeviceGuard dg(device);
    glb_graph* g = new glb_graph();
    try {
      g->device = device;
      g->n = 1ll << scale;
      g->m = edge_factor << scale;
      g->weighted = weighted != 0;
      GLB_CUDA_TRY(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
      GLB_CUDA_TRY(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
      GLB_CUDA_TRY(cudaDeviceGetAttribute(&g->l2_bytes, cudaDevAttrL2CacheSize, device));
      GLB_CUDA_TRY(cudaEventCreate(&g->ev[0]));
      GLB_CUDA_TRY(cudaEventCreate(&g->ev[1]));
      g->host_ctrl = glb::pinned_small_get();
      const unsigned long long st[2] = {state_hi_lo[0], state_hi_lo[1]};
      const unsigned long long ic[2] = {inc_hi_lo[0], inc_hi_lo[1]};
      glb::rmat_device(g, scale, edge_factor, t_a, t_ab, t_abc, st, ic, weighted != 0, max_weight);
      glb::DevCtrl* ctrl = (glb::DevCtrl*)glb::ensure(g->ws.ctrl, sizeof(glb::DevCtrl));
      GLB_CUDA_TRY(cudaMemsetAsync(ctrl, 0, sizeof(glb::DevCtrl), g->stream));
      glb::k_check_rows<<<glb::grid_for(g->n, glb::kBlock, g->num_sms * 8), glb::kBlock, 0,
                          g->stream>>>(g->row, g->n, g->m, &ctrl->bad_input,
                                       (unsigned long long*)&ctrl->aux[0]);
      GLB_CHECK_LAUNCH();
      long long mx = 0;
      GLB_CUDA_TRY(cudaMemcpyAsync(&mx, &ctrl->aux[0], 8, cudaMemcpyDeviceToHost, g->stream));
      GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
      g->max_degree = mx;
    } catch (...) {
      glb_graph_destroy(g);
      throw;
    }
    *out = g;
  });
}

int glb_graph_download(glb_graph* g, int64_t* row_offsets, int64_t* col, int64_t* weights) {
  return guarded([&] {
    if (!g) throw Error{GLB_EINVAL, "graph is NULL"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    if (row_offsets)
      GLB_CUDA_TRY(cudaMemcpyAsync(row_offsets, g->row, (size_t)(g->n + 1) * 8,
                                   cudaMemcpyDeviceToHost, g->stream));
    auto widen = [&](const uint32_t* src, int64_t* dst) {
      if (g->m == 0 || !dst) return;
      const long long chunk = 1ll << 26;
      long long* d = (long long*)glb::ensure(g->ws.out64, (size_t)std::min<long long>(g->m, chunk) * 8);
      for (long long off = 0; off < g->m; off += chunk) {
        const long long len = std::min<long long>(chunk, g->m - off);
        glb::k_widen_u32_to_i64<<<glb::grid_for(len, glb::kBlock, g->num_sms * 8), glb::kBlock, 0,
                                  g->stream>>>(src + off, d, len);
        GLB_CHECK_LAUNCH();
        GLB_CUDA_TRY(cudaMemcpyAsync(dst + off, d, (size_t)len * 8, cudaMemcpyDeviceToHost,
                                     g->stream));
        GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
      }
    };
    widen(g->col, col);
    if (g->wt) widen(g->wt, weights);
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  });
}

int glb_graph_download_u32(glb_graph* g, int64_t* row_offsets, uint32_t* col, uint32_t* weights) {
  return guarded([&] {
    if (!g) throw Error{GLB_EINVAL, "graph is NULL"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    if (row_offsets)
      GLB_CUDA_TRY(cudaMemcpyAsync(row_offsets, g->row, (size_t)(g->n + 1) * 8,
                                   cudaMemcpyDeviceToHost, g->stream));
    if (col && g->m)
      GLB_CUDA_TRY(cudaMemcpyAsync(col, g->col, (size_t)g->m * 4, cudaMemcpyDeviceToHost, g->stream));
    if (weights && g->m) {
      if (!g->wt) throw Error{GLB_EINVAL, "graph is unweighted"};
      GLB_CUDA_TRY(cudaMemcpyAsync(weights, g->wt, (size_t)g->m * 4, cudaMemcpyDeviceToHost,
                                   g->stream));
    }
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  });
}

int glb_graph_partition(glb_graph* g, int parts, int64_t* bounds) {
  return guarded([&] {
    if (!g || !bounds) throw Error{GLB_EINVAL, "NULL argument"};
    if (parts < 1 || parts > 64) throw Error{GLB_EINVAL, "parts must be in [1, 64]"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    // edge-balanced contiguous ranges: bounds[r] = first v with row[v] >= r*m/parts
    std::vector<long long> h((size_t)g->n + 1);
    GLB_CUDA_TRY(cudaMemcpy(h.data(), g->row, ((size_t)g->n + 1) * 8, cudaMemcpyDeviceToHost));
    bounds[0] = 0;
    for (int r = 1; r < parts; ++r) {
      const long long target = (long long)((__int128)g->m * r / parts);
      bounds[r] = std::lower_bound(h.begin(), h.end() - 1, target) - h.begin();
      if (bounds[r] < bounds[r - 1]) bounds[r] = bounds[r - 1];
    }
    bounds[parts] = g->n;
  });
}

__global__ void k_restrict_rows(const long long* __restrict__ row, long long n, long long lo,
                                long long hi, long long e_lo, long long e_hi,
                                long long* __restrict__ out) {
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v <= n;
       v += (long long)gridDim.x * blockDim.x) {
    long long r = row[v];
    r = r < e_lo ? e_lo : (r > e_hi ? e_hi : r);
    out[v] = (v <= lo ? e_lo : (v >= hi ? e_hi : r)) - e_lo;
  }
}

int glb_graph_restrict(glb_graph* g, int64_t v_lo, int64_t v_hi) {
  return guarded([&] {
    if (!g) throw Error{GLB_EINVAL, "graph is NULL"};
    if (v_lo < 0 || v_hi < v_lo || v_hi > g->n) throw Error{GLB_EINVAL, "bad vertex range"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    long long e[2];
    GLB_CUDA_TRY(cudaMemcpy(&e[0], g->row + v_lo, 8, cudaMemcpyDeviceToHost));
    GLB_CUDA_TRY(cudaMemcpy(&e[1], g->row + v_hi, 8, cudaMemcpyDeviceToHost));
    const long long m2 = e[1] - e[0];
    long long* row2 = nullptr;
    uint32_t *col2 = nullptr, *w2 = nullptr;
    row2 = (long long*)dmalloc((size_t)(g->n + 1) * 8);
    col2 = (uint32_t*)dmalloc((size_t)std::max<long long>(m2, 1) * 4 + kEdgePad);
    if (g->wt) w2 = (uint32_t*)dmalloc((size_t)std::max<long long>(m2, 1) * 4 + kEdgePad);
    k_restrict_rows<<<grid_for(g->n + 1, kBlock, g->num_sms * 8), kBlock, 0, g->stream>>>(
        g->row, g->n, v_lo, v_hi, e[0], e[1], row2);
    GLB_CHECK_LAUNCH();
    if (m2) {
      GLB_CUDA_TRY(cudaMemcpyAsync(col2, g->col + e[0], (size_t)m2 * 4, cudaMemcpyDeviceToDevice,
                                   g->stream));
      if (g->wt)
        GLB_CUDA_TRY(cudaMemcpyAsync(w2, g->wt + e[0], (size_t)m2 * 4, cudaMemcpyDeviceToDevice,
                                     g->stream));
    }
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
    dfree(g->row);
    dfree(g->col);
    dfree(g->wt);
    g->row = row2;
    g->col = col2;
    g->wt = w2;
    g->m = m2;
    DevCtrl* ctrl = (DevCtrl*)ensure(g->ws.ctrl, sizeof(DevCtrl));
    GLB_CUDA_TRY(cudaMemsetAsync(ctrl, 0, sizeof(DevCtrl), g->stream));
    k_check_rows<<<grid_for(g->n, kBlock, g->num_sms * 8), kBlock, 0, g->stream>>>(
        g->row, g->n, g->m, &ctrl->bad_input, (unsigned long long*)&ctrl->aux[0]);
    GLB_CHECK_LAUNCH();
    long long mx = 0;
    GLB_CUDA_TRY(cudaMemcpyAsync(&mx, &ctrl->aux[0], 8, cudaMemcpyDeviceToHost, g->stream));
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
    g->max_degree = mx;
  });
}

int glb_graph_destroy(glb_graph* g) {
  if (!g) return GLB_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  glb::dfree(g->row);
  glb::dfree(g->col);
  glb::dfree(g->wt);
  glb::Workspace& ws = g->ws;
  delete g->shard;
  g->shard = nullptr;
  ws.each([](glb::DevBuf& b) { glb::free_buf(b); });
  for (auto e : g->ev_pool) cudaEventDestroy(e);
  if (g->ev[0]) cudaEventDestroy(g->ev[0]);
  if (g->ev[1]) cudaEventDestroy(g->ev[1]);
  glb::pinned_small_put(g->host_ctrl);
  if (g->stream) cudaStreamDestroy(g->stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete g;
  return GLB_OK;
}

int glb_measure_gather(glb_graph* g, double* out4) {
  return guarded([&] {
    if (!g || !out4) throw Error{GLB_EINVAL, "NULL argument"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    glb::measure_gather(g, out4);
  });
}

int glb_graph_info(const glb_graph* g, int64_t* n, int64_t* m, int* weighted, int* device) {
  return guarded([&] {
    if (!g) throw Error{GLB_EINVAL, "graph is NULL"};
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (weighted) *weighted = g->weighted ? 1 : 0;
    if (device) *device = g->device;
  });
}

int glb_graph_stream(const glb_graph* g, void** stream) {
  return guarded([&] {
    if (!g || !stream) throw Error{GLB_EINVAL, "graph/stream is NULL"};
    *stream = (void*)g->stream;
  });
}

int glb_degree_stats(glb_graph* g, int64_t* max_degree, int64_t* sum_degree, double* sum_sq) {
  return guarded([&] {
    if (!g || !max_degree || !sum_degree || !sum_sq) throw Error{GLB_EINVAL, "NULL argument"};
    if (g->n < 1) throw Error{GLB_EINVAL, "degree statistics need at least one node"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    glb::degree_stats(g, max_degree, sum_degree, sum_sq);
  });
}

int glb_histogram(glb_graph* g, int bins, int64_t* counts, int64_t* max_degree,
                  int32_t* arg_max_bin, int64_t* mdt) {
  return guarded([&] {
    if (!g) throw Error{GLB_EINVAL, "graph is NULL"};
    if (bins < 1) throw Error{GLB_EINVAL, "bins must be >= 1"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    if (max_degree) *max_degree = g->max_degree;
    glb::histogram(g, g->row, g->n, (unsigned long long)g->max_degree, bins, counts, arg_max_bin,
                   mdt);
  });
}

int glb_split_graph(glb_graph* g, int64_t mdt, int64_t* new_n, int64_t* num_children,
                    int64_t* new_row_offsets, int64_t* new_col, int64_t* new_weights,
                    int64_t* parent_of, int64_t* children_start) {
  return guarded([&] {
    if (!g) throw Error{GLB_EINVAL, "graph is NULL"};
    if (mdt < 1) throw Error{GLB_EINVAL, "mdt must be >= 1"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    long long tot[4];
    glb::split_device(g, mdt, tot);
    long long nn = g->n + tot[0];
    if (new_n) *new_n = nn;
    if (num_children) *num_children = tot[0];
    if (!new_row_offsets) return;
    glb::Workspace& ws = g->ws;
    GLB_CUDA_TRY(cudaMemcpyAsync(new_row_offsets, ws.ns_row.p, (size_t)(nn + 1) * 8,
                                 cudaMemcpyDeviceToHost, g->stream));
    if (children_start)
      GLB_CUDA_TRY(cudaMemcpyAsync(children_start, ws.ns_cs.p, (size_t)(g->n + 1) * 8,
                                   cudaMemcpyDeviceToHost, g->stream));
    if (parent_of && tot[0] > 0)
      GLB_CUDA_TRY(cudaMemcpyAsync(parent_of, ws.ns_parent.p, (size_t)tot[0] * 8,
                                   cudaMemcpyDeviceToHost, g->stream));
    auto widen = [&](const uint32_t* src, int64_t* dst) {
      if (g->m == 0) return;
      long long* d = (long long*)glb::ensure(ws.out64, (size_t)g->m * 8);
      unsigned grid = glb::grid_for(g->m, glb::kBlock, g->num_sms * 8);
      glb::k_widen_u32_to_i64<<<grid, glb::kBlock, 0, g->stream>>>(src, d, g->m);
      GLB_CHECK_LAUNCH();
      GLB_CUDA_TRY(cudaMemcpyAsync(dst, d, (size_t)g->m * 8, cudaMemcpyDeviceToHost, g->stream));
      GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
    };
    if (new_col) widen((const uint32_t*)ws.ns_col.p, new_col);
    if (new_weights && g->wt) widen((const uint32_t*)ws.ns_w.p, new_weights);
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  });
}

int glb_csr_to_coo(glb_graph* g, int64_t max_cells, int64_t* src_out) {
  return guarded([&] {
    if (!g) throw Error{GLB_EINVAL, "graph is NULL"};
    long long required = (g->weighted ? 3 : 2) * g->m;
    if (required > max_cells)
      throw Error{GLB_ECOO_CAPACITY, "coordinate layout needs " + std::to_string(required) +
                                         " cells but the budget allows " +
                                         std::to_string(max_cells)};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    if (g->m == 0) return;
    uint32_t* src = (uint32_t*)glb::ensure(g->ws.ep_src, (size_t)g->m * 4);
    glb::coo_src(g, src);
    if (src_out) {
      long long* d = (long long*)glb::ensure(g->ws.out64, (size_t)g->m * 8);
      unsigned grid = glb::grid_for(g->m, glb::kBlock, g->num_sms * 8);
      glb::k_widen_u32_to_i64<<<grid, glb::kBlock, 0, g->stream>>>(src, d, g->m);
      GLB_CHECK_LAUNCH();
      GLB_CUDA_TRY(cudaMemcpyAsync(src_out, d, (size_t)g->m * 8, cudaMemcpyDeviceToHost, g->stream));
    }
    GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  });
}

int glb_inclusive_scan(const int64_t* values, int64_t n, int64_t* out, int device) {
  return guarded([&] {
    if (n < 0) throw Error{GLB_EINVAL, "n must be nonnegative"};
    if (n == 0) return;
    if (!values || !out) throw Error{GLB_EINVAL, "NULL argument"};
    require_device(device);
    DeviceGuard dg(device);
    cudaStream_t s;
    GLB_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    long long ntiles = (n + glb::kScanTile - 1) / glb::kScanTile;
    size_t bytes = (size_t)n * 8 * 2 + (size_t)ntiles * (4 + 2 * sizeof(glb::Vec<1>)) + 256;
    char* base = nullptr;
    cudaError_t e = cudaMalloc(&base, bytes);
    if (e != cudaSuccess) {
      cudaStreamDestroy(s);
      throw Error{GLB_ENOMEM, "device allocation for inclusive_scan failed"};
    }
    long long* d_in = (long long*)base;
    long long* d_out = d_in + n;
    unsigned* ovf = (unsigned*)(d_out + n);
    unsigned* flags = ovf + 16;
    glb::Vec<1>* aggs = (glb::Vec<1>*)(((uintptr_t)(flags + ntiles) + 63) & ~uintptr_t(63));
    glb::Vec<1>* incls = aggs + ntiles;
    unsigned hovf = 0;
    try {
      GLB_CUDA_TRY(cudaMemsetAsync(ovf, 0, (size_t)(16 + ntiles) * 4, s));
      GLB_CUDA_TRY(cudaMemcpyAsync(d_in, values, (size_t)n * 8, cudaMemcpyHostToDevice, s));
      int cap = glb::max_resident_blocks((const void*)glb::k_inclusive_scan, glb::kBlock, 0, 148);
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      cap = glb::max_resident_blocks((const void*)glb::k_inclusive_scan, glb::kBlock, 0, sms);
      unsigned grid = glb::grid_for(ntiles, 1, cap);
      glb::k_inclusive_scan<<<grid, glb::kBlock, 0, s>>>(
          d_in, n, d_out, glb::LookbackState<1>{flags, aggs, incls}, 1u, ovf);
      GLB_CHECK_LAUNCH();
      GLB_CUDA_TRY(cudaMemcpyAsync(out, d_out, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
      GLB_CUDA_TRY(cudaMemcpyAsync(&hovf, ovf, 4, cudaMemcpyDeviceToHost, s));
      GLB_CUDA_TRY(cudaStreamSynchronize(s));
    } catch (...) {
      cudaFree(base);
      cudaStreamDestroy(s);
      throw;
    }
    cudaFree(base);
    cudaStreamDestroy(s);
    if (hovf) throw Error{GLB_EOVERFLOW, "prefix sum exceeds the 64-bit counter range"};
  });
}

int glb_find_offsets(const int64_t* prefix, int64_t size, int64_t edges_per_thread, int64_t threads,
                     int64_t* node_off, int64_t* edge_off, int device) {
  return guarded([&] {
    if (size < 0 || threads < 0) throw Error{GLB_EINVAL, "size/threads must be nonnegative"};
    if (edges_per_thread < 1) throw Error{GLB_EINVAL, "edges_per_thread must be >= 1"};
    if (threads == 0) return;
    if ((size > 0 && !prefix) || !node_off || !edge_off) throw Error{GLB_EINVAL, "NULL argument"};
    require_device(device);
    DeviceGuard dg(device);
    cudaStream_t s;
    GLB_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    size_t bytes = (size_t)(size + 2 * threads + 1) * 8;
    long long* base = nullptr;
    if (cudaMalloc(&base, bytes) != cudaSuccess) {
      cudaStreamDestroy(s);
      throw Error{GLB_ENOMEM, "device allocation for find_offsets failed"};
    }
    long long* d_pre = base;
    long long* d_node = base + size;
    long long* d_edge = d_node + threads;
    try {
      if (size > 0)
        GLB_CUDA_TRY(cudaMemcpyAsync(d_pre, prefix, (size_t)size * 8, cudaMemcpyHostToDevice, s));
      unsigned grid = glb::grid_for(threads, glb::kBlock, 148 * 8);
      glb::k_find_offsets<<<grid, glb::kBlock, 0, s>>>(d_pre, size, edges_per_thread, threads,
                                                       d_node, d_edge);
      GLB_CHECK_LAUNCH();
      GLB_CUDA_TRY(cudaMemcpyAsync(node_off, d_node, (size_t)threads * 8, cudaMemcpyDeviceToHost, s));
      GLB_CUDA_TRY(cudaMemcpyAsync(edge_off, d_edge, (size_t)threads * 8, cudaMemcpyDeviceToHost, s));
      GLB_CUDA_TRY(cudaStreamSynchronize(s));
    } catch (...) {
      cudaFree(base);
      cudaStreamDestroy(s);
      throw;
    }
    cudaFree(base);
    cudaStreamDestroy(s);
  });
}

int glb_validate(glb_graph* g, int32_t algo, int64_t source, const int64_t* dist,
                 int64_t* n_bad, int64_t* first_bad) {
  return guarded([&] {
    if (!g || !dist || !n_bad || !first_bad) throw Error{GLB_EINVAL, "NULL argument"};
    if (algo != GLB_BFS && algo != GLB_SSSP) throw Error{GLB_EINVAL, "unknown relaxation kind"};
    if (source < 0 || source >= g->n)
      throw Error{GLB_EINVAL, "source " + std::to_string(source) + " out of range for " +
                                  std::to_string(g->n) + " nodes"};
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    long long nb = 0, fb = -1;
    glb::validate(g, algo == GLB_SSSP && g->wt != nullptr, source, dist, &nb, &fb);
    *n_bad = nb;
    *first_bad = fb;
  });
}

}  // extern "C"
