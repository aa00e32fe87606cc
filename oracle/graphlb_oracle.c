/*
 * graphlb_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference `graphlb` algorithms on the BFS/SSSP hot
 * path, used as the parity checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.  The product
 * (paper_1711_00231_b200 + libgraphlb_b200.so) never links or calls this.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py).
 *
 * All paths below are under /root/reference/pkg/src/graphlb/.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define ORACLE_INF INT64_MAX /* engine.py:27 INF = (1 << 63) - 1 */

/* ------------------------------------------------------------------------
 * sequential_bfs (oracles.py:13-30): FIFO queue, levels, weights ignored.
 * Returns 0, or -1 when the source is out of range.
 */
int oracle_bfs(int64_t n, const int64_t* row, const int64_t* col, int64_t source,
               int64_t* dist) {
  if (source < 0 || source >= n) return -1;
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_INF;
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (!queue) return -2;
  int64_t head = 0, tail = 0;
  dist[source] = 0;
  queue[tail++] = source;
  while (head < tail) {
    int64_t u = queue[head++];
    int64_t du = dist[u];
    for (int64_t e = row[u]; e < row[u + 1]; ++e) {
      int64_t v = col[e];
      if (dist[v] == ORACLE_INF) {
        dist[v] = du + 1;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
  return 0;
}

/* ------------------------------------------------------------------------
 * dijkstra (oracles.py:33-55): binary min-heap of (dist, node) pairs with
 * lazy deletion; missing weights count as 1; negative weights rejected.
 * Returns 0, -1 bad source, -3 negative weight.
 */
typedef struct {
  int64_t d, v;
} heap_item;

static int item_less(heap_item a, heap_item b) {
  return a.d < b.d || (a.d == b.d && a.v < b.v); /* heapq tuple order */
}

int oracle_dijkstra(int64_t n, int64_t m, const int64_t* row, const int64_t* col,
                    const int64_t* w, int64_t source, int64_t* dist) {
  if (source < 0 || source >= n) return -1;
  if (w)
    for (int64_t e = 0; e < m; ++e)
      if (w[e] < 0) return -3;
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_INF;
  size_t cap = 1024, size = 0;
  heap_item* h = (heap_item*)malloc(sizeof(heap_item) * cap);
  if (!h) return -2;
  dist[source] = 0;
  h[size++] = (heap_item){0, source};
  while (size > 0) {
    heap_item top = h[0];
    heap_item last = h[--size];
    if (size > 0) { /* sift down */
      size_t i = 0;
      for (;;) {
        size_t l = 2 * i + 1, r = l + 1, s = i;
        heap_item best = last;
        if (l < size && item_less(h[l], best)) { s = l; best = h[l]; }
        if (r < size && item_less(h[r], best)) { s = r; best = h[r]; }
        if (s == i) break;
        h[i] = h[s];
        i = s;
      }
      h[i] = last;
    }
    int64_t du = top.d, u = top.v;
    if (du > dist[u]) continue;
    for (int64_t e = row[u]; e < row[u + 1]; ++e) {
      int64_t v = col[e];
      int64_t alt = du + (w ? w[e] : 1);
      if (alt < dist[v]) {
        dist[v] = alt;
        if (size == cap) {
          cap *= 2;
          heap_item* nh = (heap_item*)realloc(h, sizeof(heap_item) * cap);
          if (!nh) { free(h); return -2; }
          h = nh;
        }
        size_t i = size++; /* sift up */
        heap_item it = {alt, v};
        while (i > 0) {
          size_t p = (i - 1) / 2;
          if (!item_less(it, h[p])) break;
          h[i] = h[p];
          i = p;
        }
        h[i] = it;
      }
    }
  }
  free(h);
  return 0;
}

/* ------------------------------------------------------------------------
 * build_histogram + compute_mdt (degrees.py:45-76).
 * counts[b-1] for 1-based bin b; degree d>0 -> ceil(d*B/max), 0 -> bin 1;
 * arg_max_bin = first maximum; mdt = max(1, arg*max // B).
 */
int oracle_histogram(int64_t n, const int64_t* row, int32_t bins, int64_t* counts,
                     int64_t* max_degree, int32_t* arg_max_bin, int64_t* mdt) {
  if (bins < 1) return -1;
  int64_t mx = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t d = row[v + 1] - row[v];
    if (d > mx) mx = d;
  }
  for (int32_t b = 0; b < bins; ++b) counts[b] = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t d = row[v + 1] - row[v];
    int64_t bin = 1;
    if (mx > 0 && d > 0) bin = (int64_t)(((__int128)d * bins + mx - 1) / mx);
    counts[bin - 1]++;
  }
  int32_t arg = 0;
  for (int32_t b = 1; b < bins; ++b)
    if (counts[b] > counts[arg]) arg = b;
  *max_degree = mx;
  *arg_max_bin = arg + 1;
  int64_t t = (int64_t)(((__int128)(arg + 1) * mx) / bins);
  *mdt = t < 1 ? 1 : t;
  return 0;
}

/* ------------------------------------------------------------------------
 * split_graph (splitting.py:58-99).  Size query with new_row == NULL.
 * pieces = max(1, ceil(d/mdt)); children_start = prefix of (pieces-1);
 * parent keeps its first min(d,mdt) edges; children take the following
 * mdt-chunks in adjacency order, child ids appended after n in node order.
 */
int oracle_split_graph(int64_t n, int64_t m, const int64_t* row, const int64_t* col,
                       const int64_t* w, int64_t mdt, int64_t* new_n, int64_t* num_children,
                       int64_t* new_row, int64_t* new_col, int64_t* new_w,
                       int64_t* parent_of, int64_t* children_start) {
  if (mdt < 1) return -1;
  int64_t kids = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t d = row[v + 1] - row[v];
    int64_t pieces = d > 0 ? (d + mdt - 1) / mdt : 1;
    kids += pieces - 1;
  }
  *new_n = n + kids;
  *num_children = kids;
  if (!new_row) return 0;
  (void)m;
  int64_t pos = 0, child = 0;
  children_start[0] = 0;
  /* parents' first chunks in node order */
  for (int64_t v = 0; v < n; ++v) {
    int64_t d = row[v + 1] - row[v];
    int64_t keep = d < mdt ? d : mdt;
    new_row[v] = pos;
    for (int64_t k = 0; k < keep; ++k) {
      new_col[pos] = col[row[v] + k];
      if (w && new_w) new_w[pos] = w[row[v] + k];
      ++pos;
    }
    int64_t pieces = d > 0 ? (d + mdt - 1) / mdt : 1;
    children_start[v + 1] = children_start[v] + pieces - 1;
  }
  /* then every child chunk, grouped by parent in node order */
  for (int64_t v = 0; v < n; ++v) {
    for (int64_t s = row[v] + mdt; s < row[v + 1]; s += mdt) {
      int64_t e = s + mdt < row[v + 1] ? s + mdt : row[v + 1];
      new_row[n + child] = pos;
      parent_of[child] = v;
      ++child;
      for (int64_t k = s; k < e; ++k) {
        new_col[pos] = col[k];
        if (w && new_w) new_w[pos] = w[k];
        ++pos;
      }
    }
  }
  new_row[n + kids] = pos;
  return 0;
}

/* ------------------------------------------------------------------------
 * find_offsets (workload.py:45-72): bisect_right per thread; idle = -1.
 */
void oracle_find_offsets(const int64_t* prefix, int64_t size, int64_t ept, int64_t threads,
                         int64_t* node_off, int64_t* edge_off) {
  int64_t total = size > 0 ? prefix[size - 1] : 0;
  for (int64_t t = 0; t < threads; ++t) {
    node_off[t] = -1;
    edge_off[t] = 0;
  }
  for (int64_t t = 0; t < threads; ++t) {
    int64_t start = t * ept;
    if (start >= total) break;
    int64_t lo = 0, hi = size;
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (start < prefix[mid]) hi = mid; else lo = mid + 1;
    }
    node_off[t] = lo;
    edge_off[t] = start - (lo ? prefix[lo - 1] : 0);
  }
}

/* ------------------------------------------------------------------------
 * inclusive_scan (scan.py:19-65).  Returns 1 when a 4096-block carry leaves
 * the int64 range (the reference's OverflowError), else 0.
 */
int oracle_inclusive_scan(const int64_t* values, int64_t n, int64_t* out) {
  __int128 acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    acc += values[i];
    out[i] = (int64_t)acc;
    if (((i + 1) % 4096 == 0 || i == n - 1) && (acc > INT64_MAX || acc < INT64_MIN)) return 1;
  }
  return 0;
}

/* csr_to_coo source ids (csr.py:168): np.repeat(arange(n), outdegrees) */
void oracle_coo_src(int64_t n, const int64_t* row, int64_t* src) {
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = row[v]; e < row[v + 1]; ++e) src[e] = v;
}

/* ------------------------------------------------------------------------
 * Node-based data-driven BFS/SSSP (run_bs, node_based.py:19-82) as a
 * multithreaded CPU port: the CPU baseline timed by bench.py.  Worklist
 * dedup by test-and-set flags cleared on swap (worklist.py:107-130,68-75),
 * relaxation by CAS-min (engine.py:120-139), INF sources skipped.  A pthread
 * pool claims 64-node chunks of the worklist (dynamic schedule) and meets at
 * a barrier per iteration.  `w` NULL applies unit weights (BFS, or SSSP on an
 * unweighted graph).  Returns 0; *iterations / *relax_ops report the work.
 */
static int relax_cas(int64_t* cell, int64_t cand) {
  int64_t cur = __atomic_load_n(cell, __ATOMIC_RELAXED);
  while (cand < cur) {
    if (__atomic_compare_exchange_n(cell, &cur, cand, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED))
      return 1;
  }
  return 0;
}

typedef struct {
  const int64_t *row, *col, *w;
  int64_t* dist;
  int64_t *in, *out;
  unsigned char* flag;
  int64_t n_in, n_out, next, ops, iterations;
  int nthreads;
  pthread_barrier_t bar;
} bs_state;

static void* bs_worker(void* arg) {
  bs_state* st = (bs_state*)arg;
  int64_t ops = 0;
  for (;;) {
    pthread_barrier_wait(&st->bar); /* iteration start */
    int64_t n_in = st->n_in;
    if (n_in == 0) break;
    for (;;) {
      int64_t lo = __atomic_fetch_add(&st->next, 64, __ATOMIC_RELAXED);
      if (lo >= n_in) break;
      int64_t hi = lo + 64 < n_in ? lo + 64 : n_in;
      for (int64_t i = lo; i < hi; ++i) {
        int64_t u = st->in[i];
        int64_t du = __atomic_load_n(&st->dist[u], __ATOMIC_RELAXED);
        if (du == ORACLE_INF) continue;
        for (int64_t e = st->row[u]; e < st->row[u + 1]; ++e) {
          int64_t v = st->col[e];
          ++ops;
          if (relax_cas(&st->dist[v], du + (st->w ? st->w[e] : 1)) &&
              !__atomic_exchange_n(&st->flag[v], 1, __ATOMIC_RELAXED)) {
            int64_t slot = __atomic_fetch_add(&st->n_out, 1, __ATOMIC_RELAXED);
            st->out[slot] = v;
          }
        }
      }
    }
    if (pthread_barrier_wait(&st->bar) == PTHREAD_BARRIER_SERIAL_THREAD) {
      for (int64_t i = 0; i < st->n_out; ++i) st->flag[st->out[i]] = 0; /* clear() on swap */
      int64_t* t = st->in; st->in = st->out; st->out = t;
      st->n_in = st->n_out;
      st->n_out = 0;
      st->next = 0;
      st->iterations++;
    }
  }
  __atomic_fetch_add(&st->ops, ops, __ATOMIC_RELAXED);
  return NULL;
}

int oracle_bs_run(int64_t n, const int64_t* row, const int64_t* col, const int64_t* w,
                  int64_t source, int threads, int64_t* dist, int64_t* iterations,
                  int64_t* relax_ops) {
  if (source < 0 || source >= n) return -1;
  if (threads < 1) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (threads < 1) threads = 1;
  bs_state st;
  memset(&st, 0, sizeof(st));
  st.row = row; st.col = col; st.w = w; st.dist = dist;
  st.in = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  st.out = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  st.flag = (unsigned char*)calloc((size_t)n, 1);
  if (!st.in || !st.out || !st.flag) { free(st.in); free(st.out); free(st.flag); return -2; }
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_INF;
  dist[source] = 0;
  st.in[0] = source;
  st.n_in = 1;
  st.nthreads = threads;
  pthread_barrier_init(&st.bar, NULL, (unsigned)threads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, bs_worker, &st);
  bs_worker(&st);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  pthread_barrier_destroy(&st.bar);
  free(th); free(st.in); free(st.out); free(st.flag);
  if (iterations) *iterations = st.iterations;
  if (relax_ops) *relax_ops = st.ops;
  return 0;
}

int oracle_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
