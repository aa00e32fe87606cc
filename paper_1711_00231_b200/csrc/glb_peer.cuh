// glb_peer.cuh -- the sharded BSP iteration's exchange over peer memory.
//
// Every rank owns an exchange region in its own HBM:
//
//   [0, kPeerHdrBytes)   mailbox: slot[parity][sender] = {seq, count, work, ovf}
//   [kPeerHdrBytes, ..)  inbox:   entry[parity][sender][0 .. seg) of the
//                        (dist, v) updates `sender` produced for vertices this
//                        rank owns; seg = the rank's owned-range length (a
//                        sender pushes each vertex at most once per iteration:
//                        the push claim is per generation)
//
// Ranks write each other's regions directly: P2P stores over NVLink /
// NVSwitch, with the regions of other processes mapped through CUDA IPC and
// those of ranks in the same process used as plain device pointers.  After
// the local relaxation of iteration t (the reference's host loop body,
// node_based.py:33-80 / workload.py:175-189 / hierarchical.py:54-136, run to
// the iteration boundary) one iteration's exchange is four kernels:
//
//   k_peer_scatter  the out list split by owner: owned vertices into the
//                   local list, remote ones as (shadow-cell distance, v)
//                   straight into the owner's inbox segment (warp-aggregated
//                   cursor per owner, system-scope fence after the stores)
//   k_peer_publish  mailbox of every peer: count, this rank's pending work and
//                   overflow flag, then seq with st.release.sys; the local
//                   list becomes the out list (buffer swap, no copy)
//   k_peer_wait     one thread polls its own mailbox (ld.acquire.sys) until
//                   every peer's seq for iteration t arrived; prefix of the
//                   received counts, global pending work, global overflow
//   k_peer_apply    received entries relaxed with this iteration's generation
//                   (atomic_relax_min, engine.py:120-139), so local and remote
//                   improvements of a vertex deduplicate into one push
//
// Inbox and mailbox are double-buffered by iteration parity: a sender that has
// passed iteration t's wait knows every peer finished applying t-1, so writing
// t+1 (parity of t-1) cannot overwrite unread entries.  Global termination is
// the sum of the pending work every rank published, so all ranks stop after
// the same iteration; relaxation is confluent (engine.py:7-9), so the result
// is the single-GPU fixpoint bit for bit.
#pragma once

#include "glb_internal.cuh"
#include "glb_relax.cuh"

namespace glb {

constexpr int kPeerMaxParts = 64;
constexpr size_t kPeerHdrBytes = 8192;
constexpr size_t kPeerEntryMax = 16;          // bytes per inbox entry (64-bit tier)
constexpr unsigned kPeerTimeoutFlag = 0x7EE70000u;  // DevCtrl::bad_input | sender

struct __align__(32) PeerSlot {
  unsigned long long seq;    // iteration sequence number (written last, release)
  unsigned long long count;  // entries in the sender's inbox segment
  unsigned long long work;   // sender's pending work: owned next-frontier + sent
  unsigned int ovf;          // sender hit a distance overflow
  unsigned int pad;
};
static_assert(sizeof(PeerSlot) * 2 * kPeerMaxParts <= kPeerHdrBytes, "mailbox fits the header");

// Per-rank device table (own device memory).
struct PeerTable {
  char* base[kPeerMaxParts];          // every rank's region as mapped in this process
  long long seg[kPeerMaxParts];       // every rank's owned-range length
  long long bounds[kPeerMaxParts + 1];
  unsigned long long recv_off[kPeerMaxParts + 1];  // k_peer_wait: prefix of received counts
  unsigned long long cursor[kPeerMaxParts];        // k_peer_scatter: per-owner append cursors
  unsigned long long my_work;          // k_peer_publish: this rank's pending work
  unsigned long long sent;             // entries sent (whole run)
  unsigned long long recv;             // entries received (whole run)
  unsigned long long wait_ns;          // time spent polling the mailbox (whole run)
  uint32_t* tmp;                       // the list the next scatter fills with owned vertices
  int parts, me;
  unsigned long long timeout_ns;
};

// inbox entries: (dist << 32 | v) for distances of <= 32 bits, {dist, v} for 64
template <typename D>
struct PeerEntry {
  static constexpr size_t kBytes = 8;
  __device__ static void put(char* p, D d, uint32_t v) {
    *reinterpret_cast<unsigned long long*>(p) = ((unsigned long long)(uint32_t)d << 32) | v;
  }
  __device__ static void get(const char* p, D& d, uint32_t& v) {
    const unsigned long long e = *reinterpret_cast<const unsigned long long*>(p);
    d = (D)(uint32_t)(e >> 32);
    v = (uint32_t)e;
  }
};
template <>
struct PeerEntry<unsigned long long> {
  static constexpr size_t kBytes = 16;
  __device__ static void put(char* p, unsigned long long d, uint32_t v) {
    *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(d, (unsigned long long)v);
  }
  __device__ static void get(const char* p, unsigned long long& d, uint32_t& v) {
    const ulonglong2 e = *reinterpret_cast<const ulonglong2*>(p);
    d = e.x;
    v = (uint32_t)e.y;
  }
};

__device__ __forceinline__ PeerSlot* peer_slot(char* region, int parity, int sender) {
  return reinterpret_cast<PeerSlot*>(region) + parity * kPeerMaxParts + sender;
}
__device__ __forceinline__ size_t peer_entry_off(int parity, int parts, int sender, long long seg,
                                                 unsigned long long slot, size_t ebytes) {
  return kPeerHdrBytes + (((size_t)parity * parts + sender) * (size_t)seg + slot) * ebytes;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int peer_owner(const long long* b, int parts, uint32_t v) {
  int lo = 0, hi = parts;  // b[0] = 0 <= v < b[parts]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((long long)v >= b[mid])
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int peer_out_list(const DevCtrl* c) {
  return c->strategy == GLB_HP ? c->sup_out : c->out;
}

// ------------------------------------------------------------ scatter ---
template <typename D>
__global__ void __launch_bounds__(kBlock) k_peer_scatter(const DevCtrl* __restrict__ c,
                                                         PeerTable* t,
                                                         const CellS<D>* __restrict__ cells,
                                                         int parity) {
  __shared__ long long s_b[kPeerMaxParts + 1];
  __shared__ char* s_base[kPeerMaxParts];
  __shared__ long long s_seg[kPeerMaxParts];
  const int parts = t->parts, me = t->me;
  for (int i = threadIdx.x; i <= parts; i += blockDim.x) s_b[i] = t->bounds[i];
  for (int i = threadIdx.x; i < parts; i += blockDim.x) {
    s_base[i] = t->base[i];
    s_seg[i] = t->seg[i];
  }
  __syncthreads();
  const int ol = peer_out_list(c);
  const uint32_t* __restrict__ q = c->qptr[ol];
  const unsigned n = c->qcount[ol];
  uint32_t* tmp = t->tmp;
  bool remote = false;
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned b0 = blockIdx.x * blockDim.x; b0 < n; b0 += stride) {  // warp-uniform bound
    const unsigned i = b0 + threadIdx.x;
    const bool ok = i < n;
    const uint32_t v = ok ? q[i] : 0u;
    const int o = ok ? peer_owner(s_b, parts, v) : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, o);
    const int leader = __ffs(grp) - 1;
    unsigned long long base = 0;
    if (o >= 0 && (int)lane_id() == leader) base = atomicAdd(&t->cursor[o], (unsigned long long)__popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (!ok) continue;
    const unsigned long long slot = base + __popc(grp & ((1u << lane_id()) - 1u));
    if (o == me) {
      tmp[slot] = v;
    } else {
      char* p = s_base[o] + peer_entry_off(parity, parts, me, s_seg[o], slot, PeerEntry<D>::kBytes);
      PeerEntry<D>::put(p, Cell<D>::dist(cells[v]), v);
      remote = true;
    }
  }
  if (remote) __threadfence_system();
}

// ------------------------------------------------------------ publish ---
__global__ void k_peer_publish(DevCtrl* c, PeerTable* t, unsigned long long seq, int parity) {
  const int parts = t->parts, me = t->me;
  __shared__ unsigned long long s_work;
  if (threadIdx.x == 0) {
    unsigned long long w = 0;
    for (int o = 0; o < parts; ++o) w += t->cursor[o];  // owned next frontier + sent
    s_work = w;
    t->my_work = w;
    t->sent += w - t->cursor[me];
    // the owned vertices become the out list (swap with the scatter target)
    const int ol = peer_out_list(c);
    uint32_t* old = c->qptr[ol];
    c->qptr[ol] = t->tmp;
    t->tmp = old;
    c->qcount[ol] = (unsigned)t->cursor[me];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < parts; o += blockDim.x) {
    if (o == me) continue;
    PeerSlot* s = peer_slot(t->base[o], parity, me);
    s->count = t->cursor[o];
    s->work = s_work;
    s->ovf = c->overflow;
    __threadfence_system();
    st_release_sys(&s->seq, seq);
  }
}

// --------------------------------------------------------------- wait ---
__global__ void k_peer_wait(DevCtrl* c, PeerTable* t, unsigned long long seq, int parity) {
  if (threadIdx.x != 0) return;
  const int parts = t->parts, me = t->me;
  char* own = t->base[me];
  const unsigned long long t0 = gtime();
  unsigned long long off = 0, work = t->my_work;
  unsigned ovf = 0;
  for (int s = 0; s < parts; ++s) {
    t->recv_off[s] = off;
    if (s == me) continue;
    PeerSlot* sl = peer_slot(own, parity, s);
    while (ld_acquire_sys(&sl->seq) != seq) {
      if (gtime() - t0 > t->timeout_ns) {  // a peer never arrived: fail loudly, do not hang
        c->bad_input = kPeerTimeoutFlag | (unsigned)s;
        c->overflow = 0;
        t->recv_off[parts] = 0;
        c->aux[0] = 0;
        c->aux[1] = 0;
        return;
      }
      __nanosleep(200);
    }
    const unsigned long long cnt = *(volatile unsigned long long*)&sl->count;
    off += cnt;
    work += *(volatile unsigned long long*)&sl->work;
    ovf |= *(volatile unsigned*)&sl->ovf;
  }
  t->recv_off[parts] = off;
  t->recv += off;
  t->wait_ns += gtime() - t0;
  c->aux[0] = (long long)off;   // entries received
  c->aux[1] = (long long)work;  // global pending work (0: every rank is done)
  c->overflow |= ovf;
}

// -------------------------------------------------------------- apply ---
template <typename D>
__global__ void __launch_bounds__(kBlock) k_peer_apply(DevCtrl* c, const PeerTable* __restrict__ t,
                                                       CellS<D>* cells, uint32_t* stamp,
                                                       int parity) {
  __shared__ unsigned long long s_off[kPeerMaxParts + 1];
  const int parts = t->parts, me = t->me;
  for (int i = threadIdx.x; i <= parts; i += blockDim.x) s_off[i] = t->recv_off[i];
  __syncthreads();
  const unsigned long long total = s_off[parts];
  if (total == 0) return;
  const char* own = t->base[me];
  const long long seg = t->seg[me];
  const int ol = peer_out_list(c);
  uint32_t* q = c->qptr[ol];
  unsigned int* nq = &c->qcount[ol];
  const uint32_t gen = c->gen;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = parts;  // sender: last s with s_off[s] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= i)
        lo = mid;
      else
        hi = mid;
    }
    D d;
    uint32_t v;
    PeerEntry<D>::get(own + peer_entry_off(parity, parts, lo, seg, i - s_off[lo], PeerEntry<D>::kBytes),
                      d, v);
    bool first = false;
    if (!relax_cell<D>(cells, v, d, gen, &first)) continue;
    if (Cell<D>::kPacked ? first : claim(stamp, v, gen)) q_append(q, nq, v);
  }
}

}  // namespace glb
