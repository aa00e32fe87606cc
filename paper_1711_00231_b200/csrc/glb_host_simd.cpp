// glb_host_simd.cpp -- AVX2 inner loops of the host-side upload pass
// (glb_memory.cu): int64 -> u32 / u8 narrowing of one worker's slice with the
// range checks of CsrGraph._validate (csr.py:66-85), written to the pinned
// staging ring with non-temporal stores (the ring is DMA'd, never re-read by
// the CPU, so streaming stores skip the read-for-ownership and keep the
// input's cache lines).  Compiled with -mavx2 by build.py; glb_memory.cu only
// calls it when the CPU reports AVX2.
#include <immintrin.h>
#include <stdint.h>

extern "C" {

int glb_cpu_has_avx2(void) { return __builtin_cpu_supports("avx2") ? 1 : 0; }

// dst[i] = (uint32_t)src[i]; returns nonzero when some src[i] >= limit
// (unsigned compare: negative values fail too).  dst must be 32-byte aligned.
int glb_narrow_u32_avx2(const int64_t* src, uint32_t* dst, long long count, uint64_t limit) {
  const __m256i sign = _mm256_set1_epi64x((long long)0x8000000000000000ull);
  const __m256i lim = _mm256_xor_si256(_mm256_set1_epi64x((long long)(limit - 1)), sign);
  const __m256i idx = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  __m256i bad = _mm256_setzero_si256();
  long long i = 0;
  for (; i + 8 <= count; i += 8) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 4));
    bad = _mm256_or_si256(bad, _mm256_cmpgt_epi64(_mm256_xor_si256(a, sign), lim));
    bad = _mm256_or_si256(bad, _mm256_cmpgt_epi64(_mm256_xor_si256(b, sign), lim));
    const __m256i pa = _mm256_permutevar8x32_epi32(a, idx);
    const __m256i pb = _mm256_permutevar8x32_epi32(b, idx);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), _mm256_permute2x128_si256(pa, pb, 0x20));
  }
  int any = !_mm256_testz_si256(bad, bad);
  for (; i < count; ++i) {
    any |= (uint64_t)src[i] >= limit;
    dst[i] = (uint32_t)src[i];
  }
  _mm_sfence();
  return any;
}

// dst[i] = (uint8_t)src[i]; returns the OR of all src values (the caller
// rejects the byte form when it exceeds 255).  dst must be 8-byte aligned.
uint64_t glb_narrow_u8_avx2(const int64_t* src, uint8_t* dst, long long count) {
  const __m256i idx = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
  // byte 0 of every dword, per 128-bit lane
  const __m256i sh = _mm256_setr_epi8(0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                                      0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1);
  __m256i orv = _mm256_setzero_si256();
  long long i = 0;
  for (; i + 8 <= count; i += 8) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 4));
    orv = _mm256_or_si256(orv, _mm256_or_si256(a, b));
    const __m256i pa = _mm256_permutevar8x32_epi32(a, idx);
    const __m256i pb = _mm256_permutevar8x32_epi32(b, idx);
    const __m256i r = _mm256_shuffle_epi8(_mm256_permute2x128_si256(pa, pb, 0x20), sh);
    const uint64_t lo = (uint32_t)_mm256_extract_epi32(r, 0);
    const uint64_t hi = (uint32_t)_mm256_extract_epi32(r, 4);
    _mm_stream_si64(reinterpret_cast<long long*>(dst + i), (long long)(lo | hi << 32));
  }
  uint64_t o = (uint64_t)_mm256_extract_epi64(orv, 0) | (uint64_t)_mm256_extract_epi64(orv, 1) |
               (uint64_t)_mm256_extract_epi64(orv, 2) | (uint64_t)_mm256_extract_epi64(orv, 3);
  for (; i < count; ++i) {
    o |= (uint64_t)src[i];
    dst[i] = (uint8_t)src[i];
  }
  _mm_sfence();
  return o;
}

}  // extern "C"
