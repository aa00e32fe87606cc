// glb_memory.cu -- host-side runtime of libgraphlb_b200.so: the device memory
// cache, the pinned host pools, the host worker pool and the staged
// host <-> HBM transfers of graph arrays and distances.
//
// Upload (the `.tolist()` / CsrGraph validation of the reference,
// strategies/common.py:73-82 and csr.py:66-85, done once per graph):
//   * host int64 arrays are narrowed ON THE HOST by a pool of worker threads
//     straight into pinned staging buffers -- col to u32 (range-checked
//     against n), weights to u8 when a chunk's maximum is <= 255 (else u32,
//     range-checked against 2^32), row offsets verbatim with the CSR
//     invariants and the maximum outdegree computed on the way -- so the PCIe
//     stream carries 4 B (1 B) per edge instead of 8 B;
//   * a ring of kStages pinned buffers keeps the next chunk's narrowing on the
//     CPU overlapped with the previous chunk's DMA;
//   * u8 weight chunks are widened into the device's u32 weight array by a
//     tiny kernel on the graph's stream.
// Distances go back as u32 (half the bytes of int64) into pinned staging and
// are widened to the reference's int64 with INF = 2^63-1 (engine.py:27) by the
// same workers.
#include <cuda_runtime.h>

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "glb_internal.cuh"

extern "C" {  // glb_host_simd.cpp (AVX2, non-temporal stores)
int glb_cpu_has_avx2(void);
int glb_narrow_u32_avx2(const int64_t* src, uint32_t* dst, long long count, uint64_t limit);
uint64_t glb_narrow_u8_avx2(const int64_t* src, uint8_t* dst, long long count);
}

namespace glb {
namespace {
bool has_avx2() {
  static const bool v = glb_cpu_has_avx2() != 0;
  return v;
}
}  // namespace

// ==================================================== device memory cache ===
// Grow-only workspaces and graph arrays are recycled across graph handles
// instead of going back to the driver: cudaMalloc/cudaFree of hundreds of MB
// cost milliseconds each (and cudaFree synchronises the device), which would
// dominate a create -> run -> destroy cycle.  Callers of dfree guarantee that
// no queued work still uses the block (they synchronise the owning stream or
// the device first), so a cached block can be handed to any stream.
namespace {
constexpr int kMaxDev = 64;
struct DevCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks[kMaxDev];
  std::unordered_map<void*, std::pair<int, size_t>> live;
  size_t cached[kMaxDev] = {};
  size_t limit[kMaxDev] = {};
};
DevCache& dcache() {
  static DevCache* c = new DevCache();  // leaked: outlives static destructors
  return *c;
}
size_t size_class(size_t b) {
  if (b < 512) return 512;
  if (b <= (size_t(1) << 20)) {
    size_t p = 512;
    while (p < b) p <<= 1;
    return p;
  }
  const size_t g = size_t(2) << 20;
  return (b + g - 1) / g * g;
}
void release_locked(DevCache& c, int dev, size_t keep) {
  auto& fb = c.free_blocks[dev];
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != dev) cudaSetDevice(dev);
  while (c.cached[dev] > keep && !fb.empty()) {
    auto it = std::prev(fb.end());  // largest first
    cudaFree(it->second);
    c.cached[dev] -= it->first;
    fb.erase(it);
  }
  if (prev >= 0 && prev != dev) cudaSetDevice(prev);
}
}  // namespace

void* dmalloc(size_t bytes) {
  int dev = 0;
  GLB_CUDA_TRY(cudaGetDevice(&dev));
  const size_t cap = size_class(bytes ? bytes : 1);
  DevCache& c = dcache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto& fb = c.free_blocks[dev];
    auto it = fb.lower_bound(cap);
    // reuse a cached block of the same class, or one at most 25 % larger
    if (it != fb.end() && it->first <= cap + cap / 4) {
      void* p = it->second;
      c.cached[dev] -= it->first;
      c.live[p] = {dev, it->first};
      fb.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, cap) != cudaSuccess) {
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> lk(c.mu);
      release_locked(c, dev, 0);
    }
    if (cudaMalloc(&p, cap) != cudaSuccess) {
      cudaGetLastError();
      throw Error{GLB_ENOMEM, "cudaMalloc of " + std::to_string(cap) + " bytes failed"};
    }
  }
  std::lock_guard<std::mutex> lk(c.mu);
  c.live[p] = {dev, cap};
  return p;
}

void dfree(void* p) {
  if (!p) return;
  DevCache& c = dcache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) {  // not ours (should not happen): hand it back to the driver
    cudaFree(p);
    return;
  }
  const int dev = it->second.first;
  const size_t cap = it->second.second;
  c.live.erase(it);
  c.free_blocks[dev].emplace(cap, p);
  c.cached[dev] += cap;
  if (!c.limit[dev]) {
    size_t fr = 0, tot = 0;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
    c.limit[dev] = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? tot / 4 : (size_t(16) << 30);
    cudaGetLastError();
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
  if (c.cached[dev] > c.limit[dev]) release_locked(c, dev, c.limit[dev] / 2);
}

size_t release_cached(int dev) {
  DevCache& c = dcache();
  std::lock_guard<std::mutex> lk(c.mu);
  size_t freed = 0;
  for (int d = 0; d < kMaxDev; ++d) {
    if (dev >= 0 && d != dev) continue;
    freed += c.cached[d];
    release_locked(c, d, 0);
  }
  return freed;
}

// ===================================================== pinned host blocks ===
// Small pinned blocks (the per-graph control mirror) are pooled: cudaHostAlloc
// pins pages and costs far more than the block is worth per graph.
namespace {
struct PinnedSmall {
  std::mutex mu;
  std::vector<void*> free_list;
};
PinnedSmall& pinned_small() {
  static PinnedSmall* p = new PinnedSmall();
  return *p;
}
}  // namespace

void* pinned_small_get() {
  PinnedSmall& ps = pinned_small();
  {
    std::lock_guard<std::mutex> lk(ps.mu);
    if (!ps.free_list.empty()) {
      void* p = ps.free_list.back();
      ps.free_list.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  GLB_CUDA_TRY(cudaHostAlloc(&p, kPinnedSmallBytes, cudaHostAllocPortable));
  return p;
}

void pinned_small_put(void* p) {
  if (!p) return;
  PinnedSmall& ps = pinned_small();
  std::lock_guard<std::mutex> lk(ps.mu);
  ps.free_list.push_back(p);
}

// ======================================================= host worker pool ===
namespace {
class Workers {
 public:
  static Workers& get() {
    static Workers* w = new Workers();  // leaked: threads never joined at exit
    return *w;
  }
  unsigned size() const { return nt_; }
  // f(worker, nworkers) on every worker, the caller being worker 0.  Workers
  // spin briefly between jobs (an upload issues one job per 32 MB chunk, back
  // to back), then sleep on a condition variable.
  void run(const std::function<void(unsigned, unsigned)>& f) {
    std::lock_guard<std::mutex> serial(run_mu_);
    if (nt_ == 1) {
      f(0, 1);
      return;
    }
    job_.store(&f, std::memory_order_relaxed);
    pending_.store(nt_ - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    f(0, nt_);
    while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
  }

 private:
  Workers() {
    unsigned hw = std::thread::hardware_concurrency();
    nt_ = std::max(1u, std::min(hw ? hw : 1u, 32u));
    for (unsigned t = 1; t < nt_; ++t) std::thread([this, t] { loop(t); }).detach();
  }
  void loop(unsigned t) {
    unsigned seen = 0;
    while (true) {
      unsigned g = gen_.load(std::memory_order_acquire);
      for (int spin = 0; g == seen && spin < (1 << 16); ++spin) {
        _mm_pause();
        g = gen_.load(std::memory_order_acquire);
      }
      if (g == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        g = gen_.load(std::memory_order_acquire);
      }
      seen = g;
      (*job_.load(std::memory_order_relaxed))(t, nt_);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  unsigned nt_ = 1;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_;
  std::atomic<const std::function<void(unsigned, unsigned)>*> job_{nullptr};
  std::atomic<unsigned> gen_{0}, pending_{0};
};

// [begin, end) slice of `count` items for worker t of nt (64-item aligned)
inline void slice(long long count, unsigned t, unsigned nt, long long& b, long long& e) {
  long long per = (count + nt - 1) / nt;
  per = (per + 63) & ~63ll;
  b = std::min<long long>(count, per * t);
  e = std::min<long long>(count, b + per);
}

// ------------------------------------------------------ pinned staging ring
constexpr int kStages = 4;
constexpr size_t kStageBytes = size_t(32) << 20;
struct Staging {
  std::mutex mu;
  void* buf[kStages] = {};
  bool ok = false;
  void init() {
    if (ok) return;
    for (int i = 0; i < kStages; ++i)
      GLB_CUDA_TRY(cudaHostAlloc(&buf[i], kStageBytes, cudaHostAllocPortable));
    ok = true;
  }
};
Staging& staging() {
  static Staging* s = new Staging();
  return *s;
}

// Per-transfer ring state on one stream.
struct Ring {
  cudaStream_t s;
  cudaEvent_t ev[kStages];
  bool used[kStages] = {};
  int next = 0;
  explicit Ring(cudaStream_t st) : s(st) {
    for (int i = 0; i < kStages; ++i)
      GLB_CUDA_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  }
  ~Ring() {
    for (int i = 0; i < kStages; ++i) cudaEventDestroy(ev[i]);
  }
  int acquire() {  // a staging slot whose previous DMA has completed
    const int b = next;
    next = (next + 1) % kStages;
    if (used[b]) GLB_CUDA_TRY(cudaEventSynchronize(ev[b]));
    return b;
  }
  void release(int b) {
    GLB_CUDA_TRY(cudaEventRecord(ev[b], s));
    used[b] = true;
  }
};

__global__ void k_widen_u8(const uint8_t* __restrict__ src, uint32_t* __restrict__ dst,
                           long long count) {
  const long long quads = count >> 2;
  const uchar4* s4 = reinterpret_cast<const uchar4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < quads;
       i += (long long)gridDim.x * blockDim.x) {
    const uchar4 v = s4[i];
    d4[i] = make_uint4(v.x, v.y, v.z, v.w);
  }
  if (blockIdx.x == 0 && threadIdx.x < (count & 3)) {
    const long long i = (quads << 2) + threadIdx.x;
    dst[i] = src[i];
  }
}
}  // namespace

unsigned host_workers() { return Workers::get().size(); }

// Row offsets: int64 copied verbatim; CsrGraph invariants (csr.py:74-79) and
// the maximum outdegree computed by the workers on the way.
void upload_rows(glb_graph* g, const int64_t* row, long long n, long long m, long long* d_row,
                 long long* max_degree) {
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.mu);
  st.init();
  Ring ring(g->stream);
  Workers& W = Workers::get();
  const long long count = n + 1;
  const long long chunk = (long long)(kStageBytes / 8);
  std::vector<long long> mx(W.size(), 0);
  std::vector<char> bad(W.size(), 0);
  for (long long off = 0; off < count; off += chunk) {
    const long long len = std::min(chunk, count - off);
    const int b = ring.acquire();
    long long* dst = (long long*)st.buf[b];
    W.run([&](unsigned t, unsigned nt) {
      long long lo, hi;
      slice(len, t, nt, lo, hi);
      long long prev = off + lo > 0 ? row[off + lo - 1] : 0;
      long long mxt = mx[t];
      bool badt = false;
      for (long long i = lo; i < hi; ++i) {
        const long long r = row[off + i];
        dst[i] = r;
        const long long d = r - prev;
        badt |= d < 0;
        mxt = d > mxt ? d : mxt;
        prev = r;
      }
      mx[t] = mxt;
      if (badt) bad[t] = 1;
    });
    GLB_CUDA_TRY(cudaMemcpyAsync(d_row + off, dst, (size_t)len * 8, cudaMemcpyHostToDevice, g->stream));
    ring.release(b);
  }
  GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  bool any_bad = row[0] != 0 || row[n] != m;
  long long mxd = 0;
  for (size_t t = 0; t < mx.size(); ++t) {
    any_bad |= bad[t] != 0;
    mxd = std::max(mxd, mx[t]);
  }
  if (any_bad)
    throw Error{GLB_EINVAL, "row_offsets must start at 0, end at num_edges and be nondecreasing"};
  *max_degree = mxd;
}

// int64 -> u32 with a range check v < limit (col: limit n; weights: 2^32).
// allow_u8: a chunk whose values all fit in a byte travels as u8 and is
// widened on the device (d_scratch: >= kStageBytes bytes of device memory).
void upload_narrow(glb_graph* g, const int64_t* src, long long count, uint32_t* d_dst,
                   unsigned long long limit, bool allow_u8, void* d_scratch, const char* what) {
  if (count <= 0) return;
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.mu);
  st.init();
  Ring ring(g->stream);
  Workers& W = Workers::get();
  const long long chunk = (long long)(kStageBytes / 4);
  std::vector<char> bad(W.size(), 0), wide(W.size(), 0);
  uint8_t* d_u8[kStages];
  for (int i = 0; i < kStages; ++i)
    d_u8[i] = allow_u8 ? (uint8_t*)d_scratch + (size_t)i * (size_t)chunk : nullptr;
  for (long long off = 0; off < count; off += chunk) {
    const long long len = std::min(chunk, count - off);
    const int b = ring.acquire();
    bool as_u8 = allow_u8;
    if (as_u8) {  // optimistic byte pass; any value > 255 falls back to u32
      uint8_t* dst = (uint8_t*)st.buf[b];
      std::fill(wide.begin(), wide.end(), 0);
      W.run([&](unsigned t, unsigned nt) {
        long long lo, hi;
        slice(len, t, nt, lo, hi);
        unsigned long long orv = 0;
        if (has_avx2()) {
          orv = glb_narrow_u8_avx2(src + off + lo, dst + lo, hi - lo);
        } else {
          for (long long i = lo; i < hi; ++i) {
            const unsigned long long v = (unsigned long long)src[off + i];
            orv |= v;
            dst[i] = (uint8_t)v;
          }
        }
        if (orv > 255) wide[t] = 1;
      });
      for (char w : wide) as_u8 &= !w;
    }
    if (as_u8) {
      GLB_CUDA_TRY(cudaMemcpyAsync(d_u8[b], st.buf[b], (size_t)len, cudaMemcpyHostToDevice,
                                   g->stream));
      k_widen_u8<<<grid_for((len + 3) / 4, kBlock, g->num_sms * 4), kBlock, 0, g->stream>>>(
          d_u8[b], d_dst + off, len);
      GLB_CHECK_LAUNCH();
    } else {
      uint32_t* dst = (uint32_t*)st.buf[b];
      W.run([&](unsigned t, unsigned nt) {
        long long lo, hi;
        slice(len, t, nt, lo, hi);
        bool badt = false;
        if (has_avx2()) {
          badt = glb_narrow_u32_avx2(src + off + lo, dst + lo, hi - lo, limit) != 0;
        } else {
          for (long long i = lo; i < hi; ++i) {
            const unsigned long long v = (unsigned long long)src[off + i];
            badt |= v >= limit;
            dst[i] = (uint32_t)v;
          }
        }
        if (badt) bad[t] = 1;
      });
      GLB_CUDA_TRY(cudaMemcpyAsync(d_dst + off, dst, (size_t)len * 4, cudaMemcpyHostToDevice,
                                   g->stream));
    }
    ring.release(b);
  }
  GLB_CUDA_TRY(cudaStreamSynchronize(g->stream));
  for (char x : bad)
    if (x) throw Error{GLB_EINVAL, what};
}

// Device u32 distances (INF = 0xFFFFFFFF) -> host int64 (INF = 2^63-1).
void download_dist_u32(cudaStream_t s, const uint32_t* d_src, long long count, int64_t* out) {
  if (count <= 0) return;
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.mu);
  st.init();
  Ring ring(s);
  Workers& W = Workers::get();
  const long long chunk = (long long)(kStageBytes / 4);
  // all chunks in flight first, then widen each as its copy lands
  struct Pending {
    int b;
    long long off, len;
  };
  std::vector<Pending> q;
  auto drain = [&](const Pending& p) {
    GLB_CUDA_TRY(cudaEventSynchronize(ring.ev[p.b]));
    const uint32_t* srcb = (const uint32_t*)st.buf[p.b];
    W.run([&](unsigned t, unsigned nt) {
      long long lo, hi;
      slice(p.len, t, nt, lo, hi);
      for (long long i = lo; i < hi; ++i) {
        const uint32_t v = srcb[i];
        out[p.off + i] = v == 0xFFFFFFFFu ? (int64_t)0x7FFFFFFFFFFFFFFFll : (int64_t)v;
      }
    });
  };
  for (long long off = 0; off < count; off += chunk) {
    const long long len = std::min(chunk, count - off);
    if ((int)q.size() == kStages) {
      drain(q.front());
      q.erase(q.begin());
    }
    const int b = ring.next;
    ring.next = (ring.next + 1) % kStages;
    GLB_CUDA_TRY(cudaMemcpyAsync(st.buf[b], d_src + off, (size_t)len * 4, cudaMemcpyDeviceToHost, s));
    GLB_CUDA_TRY(cudaEventRecord(ring.ev[b], s));
    q.push_back({b, off, len});
  }
  for (auto& p : q) drain(p);
}

}  // namespace glb

extern "C" int glb_release_cached_memory(int device, int64_t* bytes_released) {
  const size_t r = glb::release_cached(device);
  if (bytes_released) *bytes_released = (int64_t)r;
  return GLB_OK;
}
