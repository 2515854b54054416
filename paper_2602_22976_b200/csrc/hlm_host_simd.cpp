// hlm_host_simd.cpp -- see hlm_host_simd.h.  Plain C++ (host compiler only), no CUDA.
#include "hlm_host_simd.h"

#include <cstdlib>

#if defined(__x86_64__) || defined(_M_X64)
#include <immintrin.h>
#define HLMB_X86 1
#endif

namespace hlmb {

bool host_pack_weights_u8_scalar(const double* w, uint8_t* packed, uint64_t b, uint64_t e) {
  bool bad = false;
  for (uint64_t i = b; i < e; ++i) {
    const double x = w[i];
    const uint32_t q = (x >= 0.0 && x <= 255.0) ? static_cast<uint32_t>(x) : 0u;
    bad |= static_cast<double>(q) != x;  // also true for NaN
    packed[i] = static_cast<uint8_t>(q);
  }
  return bad;
}

bool host_pack_sizes_u16(const uint64_t* off, uint16_t* sizes, uint64_t b, uint64_t e) {
  uint64_t high = 0;
  for (uint64_t i = b; i < e; ++i) {
    const uint64_t d = off[i + 1] - off[i];  // decreasing offsets wrap to a huge value
    high |= d;
    sizes[i] = static_cast<uint16_t>(d);
  }
  return (high >> 16) != 0;
}

bool host_offsets_differ_scalar(const uint64_t* off, uint64_t d, uint64_t b, uint64_t e) {
  uint64_t bad = 0;
  for (uint64_t i = b; i < e; ++i) bad |= (off[i + 1] - off[i]) ^ d;
  return bad != 0;
}

#ifdef HLMB_X86
__attribute__((target("avx2"))) static bool pack_avx2(const double* w, uint8_t* packed, uint64_t b, uint64_t e) {
  __m256d badv = _mm256_setzero_pd();
  const __m256i lim = _mm256_set1_epi32(255), zero = _mm256_setzero_si256();
  uint64_t i = b;
  for (; i + 8 <= e; i += 8) {
    const __m256d x0 = _mm256_loadu_pd(w + i), x1 = _mm256_loadu_pd(w + i + 4);
    // truncating conversion; NaN and anything outside int32 become INT_MIN
    const __m128i q0 = _mm256_cvttpd_epi32(x0), q1 = _mm256_cvttpd_epi32(x1);
    const __m256d r0 = _mm256_cvtepi32_pd(q0), r1 = _mm256_cvtepi32_pd(q1);
    const __m256i q = _mm256_set_m128i(q1, q0);
    // an integer in [0, 255]: the round trip is exact (unordered compares flag NaN) and 0 <= q <= 255
    const __m256d inexact = _mm256_or_pd(_mm256_cmp_pd(r0, x0, _CMP_NEQ_UQ), _mm256_cmp_pd(r1, x1, _CMP_NEQ_UQ));
    const __m256i outside = _mm256_or_si256(_mm256_cmpgt_epi32(q, lim), _mm256_cmpgt_epi32(zero, q));
    badv = _mm256_or_pd(badv, _mm256_or_pd(inexact, _mm256_castsi256_pd(outside)));
    const __m256i s16 = _mm256_packus_epi32(q, q);  // per 128-bit lane: q0 | q1
    const __m256i s8 = _mm256_packus_epi16(s16, s16);
    const uint32_t lo = static_cast<uint32_t>(_mm256_extract_epi32(s8, 0));
    const uint32_t hi = static_cast<uint32_t>(_mm256_extract_epi32(s8, 4));
    __builtin_memcpy(packed + i, &lo, 4);
    __builtin_memcpy(packed + i + 4, &hi, 4);
  }
  const __m256i badi = _mm256_castpd_si256(badv);  // `outside` flags 32-bit lanes: test every bit, not the sign bits
  bool bad = !_mm256_testz_si256(badi, badi);
  if (i < e) bad |= host_pack_weights_u8_scalar(w, packed, i, e);
  return bad;
}

__attribute__((target("avx2"))) static bool differ_avx2(const uint64_t* off, uint64_t d, uint64_t b, uint64_t e) {
  __m256i bad = _mm256_setzero_si256();
  const __m256i dv = _mm256_set1_epi64x(static_cast<long long>(d));
  uint64_t i = b;
  for (; i + 8 <= e; i += 8) {
    const __m256i a0 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i));
    const __m256i a1 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i + 1));
    const __m256i c0 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i + 4));
    const __m256i c1 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i + 5));
    bad = _mm256_or_si256(bad, _mm256_xor_si256(_mm256_sub_epi64(a1, a0), dv));
    bad = _mm256_or_si256(bad, _mm256_xor_si256(_mm256_sub_epi64(c1, c0), dv));
  }
  bool r = !_mm256_testz_si256(bad, bad);
  if (i < e) r |= host_offsets_differ_scalar(off, d, i, e);
  return r;
}

static bool use_avx2() {
  static const bool on = [] {
    const char* env = std::getenv("HLM_B200_HOST_SIMD");  // "0": scalar loops
    if (env && env[0] == '0') return false;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx2") != 0;
  }();
  return on;
}
#else
static bool use_avx2() { return false; }
#endif

bool host_pack_weights_u8(const double* w, uint8_t* packed, uint64_t b, uint64_t e) {
#ifdef HLMB_X86
  if (use_avx2()) return pack_avx2(w, packed, b, e);
#endif
  return host_pack_weights_u8_scalar(w, packed, b, e);
}

bool host_offsets_differ(const uint64_t* off, uint64_t d, uint64_t b, uint64_t e) {
#ifdef HLMB_X86
  if (use_avx2()) return differ_avx2(off, d, b, e);
#endif
  return host_offsets_differ_scalar(off, d, b, e);
}

const char* host_simd_level() { return use_avx2() ? "avx2" : "scalar"; }

}  // namespace hlmb
