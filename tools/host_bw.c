/* host_bw.c -- host memory bandwidth of the upload's narrowing pass on the
 * GPU box: T threads read an int64 array and write u32 (plain vs
 * non-temporal stores).   gcc -O3 -march=native -pthread -o host_bw tools/host_bw.c */
#define _GNU_SOURCE
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static int64_t* src;
static uint32_t* dst;
static long long n;
static int nt, mode;

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

static void* work(void* arg) {
  long t = (long)arg;
  long long per = (n + nt - 1) / nt, lo = t * per, hi = lo + per < n ? lo + per : n;
  if (mode == 0) {
    for (long long i = lo; i < hi; ++i) dst[i] = (uint32_t)src[i];
  } else if (mode == 1) {
    lo &= ~7ll;
    for (long long i = lo; i + 8 <= hi; i += 8) {
      __m256i a = _mm256_loadu_si256((const __m256i*)(src + i));
      __m256i b = _mm256_loadu_si256((const __m256i*)(src + i + 4));
      __m256i pa = _mm256_permutevar8x32_epi32(a, _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7));
      __m256i pb = _mm256_permutevar8x32_epi32(b, _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7));
      __m256i r = _mm256_permute2x128_si256(pa, pb, 0x20);
      _mm256_stream_si256((__m256i*)(dst + i), r);
    }
  } else {
    volatile int64_t s = 0;
    int64_t acc = 0;
    for (long long i = lo; i < hi; ++i) acc += src[i];
    s = acc;
    (void)s;
  }
  return NULL;
}

int main(int argc, char** argv) {
  n = 1ll << 27;  /* 1 GiB of int64 */
  src = aligned_alloc(64, n * 8);
  dst = aligned_alloc(64, n * 4);
  for (long long i = 0; i < n; ++i) src[i] = i;
  memset(dst, 0, n * 4);
  int threads[] = {1, 4, 8, 16, 32};
  for (mode = 0; mode < 3; ++mode)
    for (int k = 0; k < 5; ++k) {
      nt = threads[k];
      pthread_t th[64];
      double best = 1e9;
      for (int r = 0; r < 3; ++r) {
        double t0 = now();
        for (long i = 0; i < nt; ++i) pthread_create(&th[i], NULL, work, (void*)i);
        for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
        double dt = now() - t0;
        if (dt < best) best = dt;
      }
      printf("%s threads %2d: %.1f GB/s of int64 input\n",
             mode == 0 ? "narrow(plain)" : mode == 1 ? "narrow(avx2+nt)" : "read-only", nt,
             n * 8 / best / 1e9);
    }
  return 0;
}
