/*
 * graphlb_oracle_big.c -- TEST INFRASTRUCTURE ONLY (see graphlb_oracle.c).
 *
 * The oracle restated for BASELINE.json's largest configurations (C3 grid
 * k=4096, C5 RMAT scale 27 = 2^31 edges), where the int64 arrays of the
 * reference layout no longer fit comfortably in host memory and a serial
 * pass takes minutes:
 *
 *   oracle_rmat_u32       generate_rmat + CsrGraph.from_edges
 *                         (generators.py:23-58, csr.py:97-118) under numpy's
 *                         PCG64 stream, multithreaded, into the narrow layout
 *                         (int64 row offsets, u32 columns, u32 weights);
 *   oracle_bfs_u32        sequential_bfs (oracles.py:13-30), FIFO queue;
 *   oracle_bfs_levels_u32 the same levels, level-synchronous on all cores:
 *                         a FIFO BFS dequeues level L entirely before level
 *                         L+1, so the level sets (and every dist) coincide;
 *   oracle_bs_run_u32     run_bs (node_based.py:19-82), the pthread port of
 *                         graphlb_oracle.c over the narrow layout, with an
 *                         optional time bound (a bounded CPU-baseline sample).
 *
 * tests/test_oracle_golden.py pins each against the reference's golden
 * vectors / digests and against the int64 restatements.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#define ORACLE_INF INT64_MAX

typedef unsigned __int128 u128;

static int nthreads_or_all(int t) {
  if (t < 1) t = (int)sysconf(_SC_NPROCESSORS_ONLN);
  return t < 1 ? 1 : t;
}

typedef struct {
  void* (*fn)(void*, int, int);
  void* arg;
  int tid, nth;
} job_t;

static void* job_tramp(void* p) {
  job_t* j = (job_t*)p;
  j->fn(j->arg, j->tid, j->nth);
  return NULL;
}

/* run fn(arg, tid, nth) on nth threads and join */
static void parallel(void* (*fn)(void*, int, int), void* arg, int nth) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nth);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)nth);
  for (int t = 0; t < nth; ++t) {
    jobs[t].fn = fn;
    jobs[t].arg = arg;
    jobs[t].tid = t;
    jobs[t].nth = nth;
    if (t) pthread_create(&th[t], NULL, job_tramp, &jobs[t]);
  }
  fn(arg, 0, nth);
  for (int t = 1; t < nth; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

/* ==================================================================== R-MAT
 * numpy Generator(PCG64): 128-bit LCG, XSL-RR output; random() is
 * (raw >> 11) * 2^-53; integers(1, W+1, dtype=int64) for W-1 < 2^32 draws
 * buffered 32-bit halves (low first) through Lemire's bounded method with
 * rejection of (u32 * W) mod 2^32 < (2^32 - W) mod W.
 */
static const u128 PCG_MULT = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

static u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = inc;
  while (delta) {
    if (delta & 1u) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

static inline uint64_t pcg_out(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  unsigned rot = (unsigned)(hi >> 58);
  uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

typedef struct {
  int scale;
  uint64_t m, n;
  double t_a, t_ab, t_abc;
  u128 s0, inc;
  uint32_t *src, *dst;
  /* weights */
  uint64_t ndraw;
  uint32_t W, threshold;
  uint32_t* wval;     /* [ndraw] */
  uint8_t* wok;       /* [ndraw] */
  uint64_t* tcount;   /* per-thread accepted counts / bucket counts */
  uint32_t* wout;     /* [m] accepted draws in order */
  /* sort */
  int nb, shift;      /* buckets by src >> shift */
  uint64_t* bcount;   /* [nth * nb] */
  uint32_t *tsrc, *tdst, *tw;
  uint64_t* bstart;   /* [nb + 1] */
  int64_t* row;
  uint32_t *col, *w;
  int next_bucket;
} rmat_t;

static void* rmat_edges_job(void* p, int tid, int nth) {
  rmat_t* r = (rmat_t*)p;
  const uint64_t chunk = 4096;
  uint32_t s[4096], d[4096];
  for (uint64_t c0 = (uint64_t)tid * chunk; c0 < r->m; c0 += (uint64_t)nth * chunk) {
    uint64_t cnt = r->m - c0 < chunk ? r->m - c0 : chunk;
    memset(s, 0, sizeof(uint32_t) * cnt);
    memset(d, 0, sizeof(uint32_t) * cnt);
    for (int l = 0; l < r->scale; ++l) { /* level l, edge i: raw draw l*m + i */
      u128 st = pcg_advance(r->s0, r->inc, (uint64_t)l * r->m + c0);
      for (uint64_t j = 0; j < cnt; ++j) {
        st = st * PCG_MULT + r->inc;
        double u = (double)(pcg_out(st) >> 11) * (1.0 / 9007199254740992.0);
        uint32_t row_bit = u >= r->t_ab;
        uint32_t col_bit = (u >= r->t_a && u < r->t_ab) || u >= r->t_abc;
        s[j] = (s[j] << 1) | row_bit;
        d[j] = (d[j] << 1) | col_bit;
      }
    }
    memcpy(r->src + c0, s, sizeof(uint32_t) * cnt);
    memcpy(r->dst + c0, d, sizeof(uint32_t) * cnt);
  }
  return NULL;
}

/* draws [lo, hi) of this thread: raw index scale*m + d/2, low half first */
static void wrange(const rmat_t* r, int tid, int nth, uint64_t* lo, uint64_t* hi) {
  uint64_t per = ((r->ndraw + (uint64_t)nth - 1) / (uint64_t)nth + 1) & ~1ull;
  *lo = per * (uint64_t)tid;
  *hi = *lo + per;
  if (*lo > r->ndraw) *lo = r->ndraw;
  if (*hi > r->ndraw) *hi = r->ndraw;
}

static void* rmat_wdraw_job(void* p, int tid, int nth) {
  rmat_t* r = (rmat_t*)p;
  uint64_t lo, hi, acc = 0;
  wrange(r, tid, nth, &lo, &hi);
  if (lo < hi) {
    u128 st = pcg_advance(r->s0, r->inc, (uint64_t)r->scale * r->m + lo / 2);
    for (uint64_t d = lo; d < hi; d += 2) {
      st = st * PCG_MULT + r->inc;
      uint64_t raw = pcg_out(st);
      for (int h = 0; h < 2 && d + (uint64_t)h < hi; ++h) {
        uint32_t x = h ? (uint32_t)(raw >> 32) : (uint32_t)raw;
        uint64_t mm = (uint64_t)x * r->W;
        int ok = (uint32_t)mm >= r->threshold;
        r->wval[d + h] = 1u + (uint32_t)(mm >> 32);
        r->wok[d + h] = (uint8_t)ok;
        acc += (uint64_t)ok;
      }
    }
  }
  r->tcount[tid] = acc;
  return NULL;
}

static void* rmat_wcompact_job(void* p, int tid, int nth) {
  rmat_t* r = (rmat_t*)p;
  uint64_t lo, hi, k = 0;
  wrange(r, tid, nth, &lo, &hi);
  for (int t = 0; t < tid; ++t) k += r->tcount[t];
  for (uint64_t d = lo; d < hi && k < r->m; ++d)
    if (r->wok[d]) r->wout[k++] = r->wval[d];
  return NULL;
}

/* stable MSD pass: bucket b = src >> shift, per-thread contiguous edge chunks */
static void* rmat_bcount_job(void* p, int tid, int nth) {
  rmat_t* r = (rmat_t*)p;
  uint64_t per = (r->m + (uint64_t)nth - 1) / (uint64_t)nth;
  uint64_t lo = per * (uint64_t)tid, hi = lo + per < r->m ? lo + per : r->m;
  uint64_t* c = r->bcount + (size_t)tid * (size_t)r->nb;
  memset(c, 0, sizeof(uint64_t) * (size_t)r->nb);
  for (uint64_t e = lo; e < hi; ++e) c[r->src[e] >> r->shift]++;
  return NULL;
}

static void* rmat_bscatter_job(void* p, int tid, int nth) {
  rmat_t* r = (rmat_t*)p;
  uint64_t per = (r->m + (uint64_t)nth - 1) / (uint64_t)nth;
  uint64_t lo = per * (uint64_t)tid, hi = lo + per < r->m ? lo + per : r->m;
  uint64_t* c = r->bcount + (size_t)tid * (size_t)r->nb; /* exclusive offsets */
  for (uint64_t e = lo; e < hi; ++e) {
    uint64_t pos = c[r->src[e] >> r->shift]++;
    r->tsrc[pos] = r->src[e];
    r->tdst[pos] = r->dst[e];
    if (r->tw) r->tw[pos] = r->wout[e];
  }
  return NULL;
}

/* every bucket: stable counting sort of its edges by src into the CSR */
static void* rmat_bsort_job(void* p, int tid, int nth) {
  rmat_t* r = (rmat_t*)p;
  (void)tid;
  (void)nth;
  const uint64_t span = 1ull << r->shift;
  uint64_t* cnt = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(span + 1));
  for (;;) {
    int b = __atomic_fetch_add(&r->next_bucket, 1, __ATOMIC_RELAXED);
    if (b >= r->nb) break;
    uint64_t e0 = r->bstart[b], e1 = r->bstart[b + 1];
    uint64_t v0 = (uint64_t)b << r->shift;
    memset(cnt, 0, sizeof(uint64_t) * (size_t)(span + 1));
    for (uint64_t e = e0; e < e1; ++e) cnt[r->tsrc[e] - v0 + 1]++;
    for (uint64_t v = 0; v < span; ++v) {
      cnt[v + 1] += cnt[v];
      r->row[v0 + v] = (int64_t)(e0 + cnt[v]);
    }
    for (uint64_t e = e0; e < e1; ++e) {
      uint64_t pos = e0 + cnt[r->tsrc[e] - v0]++;
      r->col[pos] = r->tdst[e];
      if (r->w) r->w[pos] = r->tw[e];
    }
  }
  free(cnt);
  return NULL;
}

/* Returns 0, -2 on allocation failure.  row: int64[2^scale + 1], col/w:
 * u32[edge_factor * 2^scale] (w NULL or weighted == 0: unweighted). */
int oracle_rmat_u32(int scale, int64_t edge_factor, double t_a, double t_ab, double t_abc,
                    const uint64_t* state_hi_lo, const uint64_t* inc_hi_lo, int weighted,
                    int64_t max_weight, int threads, int64_t* row, uint32_t* col, uint32_t* w) {
  int nth = nthreads_or_all(threads);
  rmat_t r;
  memset(&r, 0, sizeof(r));
  r.scale = scale;
  r.n = 1ull << scale;
  r.m = (uint64_t)edge_factor * r.n;
  r.t_a = t_a;
  r.t_ab = t_ab;
  r.t_abc = t_abc;
  r.s0 = ((u128)state_hi_lo[0] << 64) | state_hi_lo[1];
  r.inc = ((u128)inc_hi_lo[0] << 64) | inc_hi_lo[1];
  size_t mb = (size_t)(r.m ? r.m : 1);
  r.src = (uint32_t*)malloc(mb * 4);
  r.dst = (uint32_t*)malloc(mb * 4);
  r.tcount = (uint64_t*)calloc((size_t)nth, 8);
  if (!r.src || !r.dst || !r.tcount) goto oom;
  parallel(rmat_edges_job, &r, nth);
  if (weighted && w && max_weight == 1) { /* rng == 0: numpy draws nothing */
    r.wout = (uint32_t*)malloc(mb * 4);
    if (!r.wout) goto oom;
    for (uint64_t e = 0; e < r.m; ++e) r.wout[e] = 1;
  } else if (weighted && w) {
    r.W = (uint32_t)max_weight; /* rng.integers(1, W + 1): range W values */
    r.threshold = (uint32_t)((0x100000000ull - r.W) % r.W);
    r.wout = (uint32_t*)malloc(mb * 4);
    if (!r.wout) goto oom;
    for (uint64_t slack = 64;; slack *= 16) {
      r.ndraw = r.m + slack;
      free(r.wval);
      free(r.wok);
      r.wval = (uint32_t*)malloc((size_t)r.ndraw * 4);
      r.wok = (uint8_t*)malloc((size_t)r.ndraw);
      if (!r.wval || !r.wok) goto oom;
      parallel(rmat_wdraw_job, &r, nth);
      uint64_t acc = 0;
      for (int t = 0; t < nth; ++t) acc += r.tcount[t];
      if (acc >= r.m) break;
    }
    parallel(rmat_wcompact_job, &r, nth);
    free(r.wval);
    free(r.wok);
    r.wval = NULL;
    r.wok = NULL;
  }
  /* CsrGraph.from_edges: stable grouping by source (argsort kind="stable") */
  r.shift = scale > 8 ? scale - 8 : 0;
  r.nb = (int)(r.n >> r.shift);
  r.bcount = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)nth * (size_t)r.nb);
  r.bstart = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(r.nb + 1));
  r.tsrc = (uint32_t*)malloc(mb * 4);
  r.tdst = (uint32_t*)malloc(mb * 4);
  r.tw = r.wout ? (uint32_t*)malloc(mb * 4) : NULL;
  if (!r.bcount || !r.bstart || !r.tsrc || !r.tdst || (r.wout && !r.tw)) goto oom;
  parallel(rmat_bcount_job, &r, nth);
  {
    uint64_t run = 0;
    for (int b = 0; b < r.nb; ++b) {
      r.bstart[b] = run;
      for (int t = 0; t < nth; ++t) {
        uint64_t c = r.bcount[(size_t)t * r.nb + b];
        r.bcount[(size_t)t * r.nb + b] = run;
        run += c;
      }
    }
    r.bstart[r.nb] = run;
  }
  parallel(rmat_bscatter_job, &r, nth);
  free(r.src);
  free(r.dst);
  r.src = r.dst = NULL;
  r.row = row;
  r.col = col;
  r.w = r.wout ? w : NULL;
  parallel(rmat_bsort_job, &r, nth);
  row[r.n] = (int64_t)r.m;
  free(r.tsrc);
  free(r.tdst);
  free(r.tw);
  free(r.wout);
  free(r.bcount);
  free(r.bstart);
  free(r.tcount);
  return 0;
oom:
  free(r.src); free(r.dst); free(r.tcount); free(r.wout); free(r.wval); free(r.wok);
  free(r.bcount); free(r.bstart); free(r.tsrc); free(r.tdst); free(r.tw);
  return -2;
}

/* ==================================================================== BFS */
int oracle_bfs_u32(int64_t n, const int64_t* row, const uint32_t* col, int64_t source,
                   int64_t* dist) {
  if (source < 0 || source >= n) return -1;
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_INF;
  uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  if (!queue) return -2;
  int64_t head = 0, tail = 0;
  dist[source] = 0;
  queue[tail++] = (uint32_t)source;
  while (head < tail) {
    uint32_t u = queue[head++];
    int64_t du = dist[u];
    for (int64_t e = row[u]; e < row[u + 1]; ++e) {
      uint32_t v = col[e];
      if (dist[v] == ORACLE_INF) {
        dist[v] = du + 1;
        queue[tail++] = v;
      }
    }
  }
  free(queue);
  return 0;
}

typedef struct {
  int64_t n;
  const int64_t* row;
  const uint32_t* col;
  int64_t* dist;
  uint32_t *cur, *nxt;
  int64_t ncur, nnext, next, level;
  pthread_barrier_t bar;
} lvl_t;

static void* lvl_job(void* p, int tid, int nth) {
  lvl_t* s = (lvl_t*)p;
  (void)nth;
  uint32_t buf[1024];
  for (;;) {
    pthread_barrier_wait(&s->bar);
    if (s->ncur == 0) break;
    const int64_t lv = s->level + 1;
    int nb = 0;
    for (;;) {
      int64_t lo = __atomic_fetch_add(&s->next, 64, __ATOMIC_RELAXED);
      if (lo >= s->ncur) break;
      int64_t hi = lo + 64 < s->ncur ? lo + 64 : s->ncur;
      for (int64_t i = lo; i < hi; ++i) {
        uint32_t u = s->cur[i];
        for (int64_t e = s->row[u]; e < s->row[u + 1]; ++e) {
          uint32_t v = s->col[e];
          int64_t expect = ORACLE_INF;
          if (__atomic_load_n(&s->dist[v], __ATOMIC_RELAXED) == ORACLE_INF &&
              __atomic_compare_exchange_n(&s->dist[v], &expect, lv, 0, __ATOMIC_RELAXED,
                                          __ATOMIC_RELAXED)) {
            buf[nb++] = v;
            if (nb == 1024) {
              int64_t at = __atomic_fetch_add(&s->nnext, nb, __ATOMIC_RELAXED);
              memcpy(s->nxt + at, buf, sizeof(uint32_t) * 1024);
              nb = 0;
            }
          }
        }
      }
    }
    if (nb) {
      int64_t at = __atomic_fetch_add(&s->nnext, nb, __ATOMIC_RELAXED);
      memcpy(s->nxt + at, buf, sizeof(uint32_t) * (size_t)nb);
    }
    if (pthread_barrier_wait(&s->bar) == PTHREAD_BARRIER_SERIAL_THREAD) {
      uint32_t* t = s->cur;
      s->cur = s->nxt;
      s->nxt = t;
      s->ncur = s->nnext;
      s->nnext = 0;
      s->next = 0;
      s->level = lv;
    }
  }
  (void)tid;
  return NULL;
}

int oracle_bfs_levels_u32(int64_t n, const int64_t* row, const uint32_t* col, int64_t source,
                          int threads, int64_t* dist) {
  if (source < 0 || source >= n) return -1;
  int nth = nthreads_or_all(threads);
  lvl_t s;
  memset(&s, 0, sizeof(s));
  s.n = n;
  s.row = row;
  s.col = col;
  s.dist = dist;
  s.cur = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  s.nxt = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  if (!s.cur || !s.nxt) { free(s.cur); free(s.nxt); return -2; }
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_INF;
  dist[source] = 0;
  s.cur[0] = (uint32_t)source;
  s.ncur = 1;
  pthread_barrier_init(&s.bar, NULL, (unsigned)nth);
  parallel(lvl_job, &s, nth);
  pthread_barrier_destroy(&s.bar);
  free(s.cur);
  free(s.nxt);
  return 0;
}

/* ========================================================== run_bs (port) */
typedef struct {
  const int64_t* row;
  const uint32_t *col, *w;
  int64_t* dist;
  uint32_t *in, *out;
  unsigned char* flag;
  int64_t n_in, n_out, next, ops, iterations;
  double deadline;  /* CLOCK_MONOTONIC seconds; 0 = none */
  int stopped;
  pthread_barrier_t bar;
} bs32_t;

static double mono_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

static int relax_cas(int64_t* cell, int64_t cand) {
  int64_t cur = __atomic_load_n(cell, __ATOMIC_RELAXED);
  while (cand < cur)
    if (__atomic_compare_exchange_n(cell, &cur, cand, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED))
      return 1;
  return 0;
}

static void* bs32_job(void* p, int tid, int nth) {
  bs32_t* st = (bs32_t*)p;
  (void)tid;
  (void)nth;
  int64_t ops = 0;
  for (;;) {
    pthread_barrier_wait(&st->bar);
    const int64_t n_in = st->n_in;
    if (n_in == 0 || st->stopped) break;
    for (;;) {
      int64_t lo = __atomic_fetch_add(&st->next, 64, __ATOMIC_RELAXED);
      if (lo >= n_in) break;
      int64_t hi = lo + 64 < n_in ? lo + 64 : n_in;
      for (int64_t i = lo; i < hi; ++i) {
        uint32_t u = st->in[i];
        int64_t du = __atomic_load_n(&st->dist[u], __ATOMIC_RELAXED);
        if (du == ORACLE_INF) continue;
        for (int64_t e = st->row[u]; e < st->row[u + 1]; ++e) {
          uint32_t v = st->col[e];
          ++ops;
          if (relax_cas(&st->dist[v], du + (st->w ? (int64_t)st->w[e] : 1)) &&
              !__atomic_exchange_n(&st->flag[v], 1, __ATOMIC_RELAXED)) {
            int64_t slot = __atomic_fetch_add(&st->n_out, 1, __ATOMIC_RELAXED);
            st->out[slot] = v;
          }
        }
      }
    }
    if (pthread_barrier_wait(&st->bar) == PTHREAD_BARRIER_SERIAL_THREAD) {
      for (int64_t i = 0; i < st->n_out; ++i) st->flag[st->out[i]] = 0; /* clear() on swap */
      uint32_t* t = st->in;
      st->in = st->out;
      st->out = t;
      st->n_in = st->n_out;
      st->n_out = 0;
      st->next = 0;
      st->iterations++;
      if (st->deadline > 0 && st->n_in && mono_s() > st->deadline) st->stopped = 1;
    }
  }
  __atomic_fetch_add(&st->ops, ops, __ATOMIC_RELAXED);
  return NULL;
}

/* run_bs over the narrow layout.  max_seconds > 0 stops after the first
 * iteration that ends past the bound (*completed = 0; dist is then partial
 * and *relax_ops counts the edges examined so far). */
int oracle_bs_run_u32(int64_t n, const int64_t* row, const uint32_t* col, const uint32_t* w,
                      int64_t source, int threads, double max_seconds, int64_t* dist,
                      int64_t* iterations, int64_t* relax_ops, int* completed) {
  if (source < 0 || source >= n) return -1;
  int nth = nthreads_or_all(threads);
  bs32_t st;
  memset(&st, 0, sizeof(st));
  st.row = row;
  st.col = col;
  st.w = w;
  st.dist = dist;
  st.in = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  st.out = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  st.flag = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!st.in || !st.out || !st.flag) { free(st.in); free(st.out); free(st.flag); return -2; }
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_INF;
  dist[source] = 0;
  st.in[0] = (uint32_t)source;
  st.n_in = 1;
  st.deadline = max_seconds > 0 ? mono_s() + max_seconds : 0;
  pthread_barrier_init(&st.bar, NULL, (unsigned)nth);
  parallel(bs32_job, &st, nth);
  pthread_barrier_destroy(&st.bar);
  free(st.in);
  free(st.out);
  free(st.flag);
  if (iterations) *iterations = st.iterations;
  if (relax_ops) *relax_ops = st.ops;
  if (completed) *completed = !st.stopped;
  return 0;
}

/* ========================================================== run_wd (port) */
/* Workload decomposition (strategies/workload.py:75-159, run_wd loop
 * workload.py:162-189) over the narrow layout: per iteration the frontier's
 * out-degrees are prefix-summed (inclusive_scan, scan.py:19-65), every host
 * thread takes an equal slice of ept = ceil(total / threads) edges, finds its
 * first item by binary search over the prefix (find_offsets,
 * workload.py:45-72) and walks the slice, reading the item's distance when it
 * enters a node (workload.py:131,140).  Test / baseline infrastructure only. */
typedef struct {
  const int64_t* row;
  const uint32_t *col, *w;
  int64_t* dist;
  uint32_t *in, *out;
  int64_t* prefix;      /* inclusive prefix of the frontier's out-degrees */
  int64_t* part;        /* per-thread partial sums of the scan */
  unsigned char* flag;
  int64_t n_in, n_out, ops, iterations, total;
  double deadline;
  int stopped, nth;
  pthread_barrier_t bar;
} wd32_t;

static void* wd32_job(void* p, int tid, int nth) {
  wd32_t* st = (wd32_t*)p;
  int64_t ops = 0;
  for (;;) {
    pthread_barrier_wait(&st->bar);
    const int64_t n_in = st->n_in;
    if (n_in == 0 || st->stopped) break;
    /* scan pass 1: this thread's chunk of the frontier */
    const int64_t c0 = n_in * tid / nth, c1 = n_in * (tid + 1) / nth;
    int64_t s = 0;
    for (int64_t i = c0; i < c1; ++i) {
      const uint32_t u = st->in[i];
      s += st->row[u + 1] - st->row[u];
    }
    st->part[tid] = s;
    if (pthread_barrier_wait(&st->bar) == PTHREAD_BARRIER_SERIAL_THREAD) {
      int64_t run = 0;
      for (int t = 0; t < nth; ++t) {
        const int64_t x = st->part[t];
        st->part[t] = run;
        run += x;
      }
      st->total = run;
    }
    pthread_barrier_wait(&st->bar);
    s = st->part[tid];
    for (int64_t i = c0; i < c1; ++i) {
      const uint32_t u = st->in[i];
      s += st->row[u + 1] - st->row[u];
      st->prefix[i] = s;
    }
    pthread_barrier_wait(&st->bar);
    /* relax: an equal slice of edges per thread */
    const int64_t total = st->total;
    const int64_t ept = (total + nth - 1) / nth;
    int64_t start = (int64_t)tid * ept, end = start + ept < total ? start + ept : total;
    if (start < end) {
      int64_t lo = 0, hi = n_in - 1; /* first item whose inclusive prefix > start */
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (st->prefix[mid] > start)
          hi = mid;
        else
          lo = mid + 1;
      }
      int64_t wi = lo;
      int64_t f = start;
      while (f < end) {
        const uint32_t u = st->in[wi];
        const int64_t pre0 = st->prefix[wi] - (st->row[u + 1] - st->row[u]);
        const int64_t stop = st->prefix[wi] < end ? st->prefix[wi] : end;
        const int64_t du = __atomic_load_n(&st->dist[u], __ATOMIC_RELAXED); /* dn at node entry */
        for (; f < stop; ++f) {
          const int64_t e = st->row[u] + (f - pre0);
          const uint32_t v = st->col[e];
          ++ops;
          if (du != ORACLE_INF &&
              relax_cas(&st->dist[v], du + (st->w ? (int64_t)st->w[e] : 1)) &&
              !__atomic_exchange_n(&st->flag[v], 1, __ATOMIC_RELAXED)) {
            const int64_t slot = __atomic_fetch_add(&st->n_out, 1, __ATOMIC_RELAXED);
            st->out[slot] = v;
          }
        }
        ++wi;
      }
    }
    if (pthread_barrier_wait(&st->bar) == PTHREAD_BARRIER_SERIAL_THREAD) {
      for (int64_t i = 0; i < st->n_out; ++i) st->flag[st->out[i]] = 0; /* clear() on swap */
      uint32_t* t = st->in;
      st->in = st->out;
      st->out = t;
      st->n_in = st->total ? st->n_out : 0; /* no edges left: done (workload.py:181-183) */
      st->n_out = 0;
      st->iterations++;
      if (st->deadline > 0 && st->n_in && mono_s() > st->deadline) st->stopped = 1;
    }
  }
  __atomic_fetch_add(&st->ops, ops, __ATOMIC_RELAXED);
  return NULL;
}

/* run_wd over the narrow layout; arguments and results as oracle_bs_run_u32. */
int oracle_wd_run_u32(int64_t n, const int64_t* row, const uint32_t* col, const uint32_t* w,
                      int64_t source, int threads, double max_seconds, int64_t* dist,
                      int64_t* iterations, int64_t* relax_ops, int* completed) {
  if (source < 0 || source >= n) return -1;
  int nth = nthreads_or_all(threads);
  wd32_t st;
  memset(&st, 0, sizeof(st));
  st.row = row;
  st.col = col;
  st.w = w;
  st.dist = dist;
  st.nth = nth;
  const size_t nb = (size_t)(n > 0 ? n : 1);
  st.in = (uint32_t*)malloc(sizeof(uint32_t) * nb);
  st.out = (uint32_t*)malloc(sizeof(uint32_t) * nb);
  st.prefix = (int64_t*)malloc(sizeof(int64_t) * nb);
  st.part = (int64_t*)malloc(sizeof(int64_t) * (size_t)nth);
  st.flag = (unsigned char*)calloc(nb, 1);
  if (!st.in || !st.out || !st.prefix || !st.part || !st.flag) {
    free(st.in); free(st.out); free(st.prefix); free(st.part); free(st.flag);
    return -2;
  }
  for (int64_t i = 0; i < n; ++i) dist[i] = ORACLE_INF;
  dist[source] = 0;
  st.in[0] = (uint32_t)source;
  st.n_in = 1;
  st.deadline = max_seconds > 0 ? mono_s() + max_seconds : 0;
  pthread_barrier_init(&st.bar, NULL, (unsigned)nth);
  parallel(wd32_job, &st, nth);
  pthread_barrier_destroy(&st.bar);
  free(st.in); free(st.out); free(st.prefix); free(st.part); free(st.flag);
  if (iterations) *iterations = st.iterations;
  if (relax_ops) *relax_ops = st.ops;
  if (completed) *completed = !st.stopped;
  return 0;
}
