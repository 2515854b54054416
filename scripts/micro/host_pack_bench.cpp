// Host-side scan/pack throughput (the loader's critical path): 16 threads over 2 GiB of f64 weights
// and 2 GiB of u64 offsets.  g++ -O2 -pthread host_pack_bench.cpp -o host_pack_bench
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static bool pack_scalar(const double* w, uint8_t* p, uint64_t b, uint64_t e) {
  bool bad = false;
  for (uint64_t i = b; i < e; ++i) {
    const double x = w[i];
    const uint32_t q = (x >= 1.0 && x <= 255.0) ? static_cast<uint32_t>(x) : 0u;
    bad |= static_cast<double>(q) != x;
    p[i] = static_cast<uint8_t>(q);
  }
  return bad;
}

__attribute__((target("avx2"))) static bool pack_avx2(const double* w, uint8_t* p, uint64_t b, uint64_t e) {
  __m256d badv = _mm256_setzero_pd();
  uint64_t i = b;
  for (; i + 8 <= e; i += 8) {
    const __m256d x0 = _mm256_loadu_pd(w + i), x1 = _mm256_loadu_pd(w + i + 4);
    const __m128i q0 = _mm256_cvttpd_epi32(x0), q1 = _mm256_cvttpd_epi32(x1);
    const __m256d r0 = _mm256_cvtepi32_pd(q0), r1 = _mm256_cvtepi32_pd(q1);
    const __m256i q = _mm256_set_m128i(q1, q0);
    // exact integer in [1, 255]: round trip equal and the high 24 bits clear and non-zero
    __m256d ne = _mm256_or_pd(_mm256_cmp_pd(r0, x0, _CMP_NEQ_UQ), _mm256_cmp_pd(r1, x1, _CMP_NEQ_UQ));
    const __m256i out_of_range = _mm256_or_si256(_mm256_cmpgt_epi32(q, _mm256_set1_epi32(255)), _mm256_cmpgt_epi32(_mm256_set1_epi32(1), q));
    badv = _mm256_or_pd(badv, _mm256_or_pd(ne, _mm256_castsi256_pd(out_of_range)));
    const __m256i s16 = _mm256_packus_epi32(q, q);       // per 128-bit lane
    const __m256i s8 = _mm256_packus_epi16(s16, s16);
    const uint32_t lo = static_cast<uint32_t>(_mm256_extract_epi32(s8, 0)), hi = static_cast<uint32_t>(_mm256_extract_epi32(s8, 4));
    *reinterpret_cast<uint32_t*>(p + i) = lo;
    *reinterpret_cast<uint32_t*>(p + i + 4) = hi;
  }
  bool bad = _mm256_movemask_pd(badv) != 0;
  if (i < e) bad |= pack_scalar(w, p, i, e);
  return bad;
}

static uint64_t scan_scalar(const uint64_t* off, uint64_t d0, uint64_t b, uint64_t e) {
  uint64_t bad = 0;
  for (uint64_t i = b; i < e; ++i) bad |= (off[i + 1] - off[i]) ^ d0;
  return bad;
}

__attribute__((target("avx2"))) static uint64_t scan_avx2(const uint64_t* off, uint64_t d0, uint64_t b, uint64_t e) {
  __m256i bad = _mm256_setzero_si256();
  const __m256i d = _mm256_set1_epi64x(static_cast<long long>(d0));
  uint64_t i = b;
  for (; i + 8 <= e; i += 8) {
    const __m256i a0 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i)), a1 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i + 1));
    const __m256i b0 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i + 4)), b1 = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(off + i + 5));
    bad = _mm256_or_si256(bad, _mm256_xor_si256(_mm256_sub_epi64(a1, a0), d));
    bad = _mm256_or_si256(bad, _mm256_xor_si256(_mm256_sub_epi64(b1, b0), d));
  }
  uint64_t r = _mm256_testz_si256(bad, bad) ? 0 : 1;
  if (i < e) r |= scan_scalar(off, d0, i, e);
  return r;
}

int main(int argc, char** argv) {
  const uint64_t m = 1ull << 28;
  const unsigned nt = argc > 1 ? std::atoi(argv[1]) : std::thread::hardware_concurrency();
  double* w = static_cast<double*>(std::aligned_alloc(64, m * 8));
  uint64_t* off = static_cast<uint64_t*>(std::aligned_alloc(64, (m + 8) * 8));
  uint8_t* p = static_cast<uint8_t*>(std::aligned_alloc(64, m));
  auto par = [&](auto&& f) {
    std::atomic<uint64_t> next{0};
    std::vector<std::thread> th;
    const uint64_t chunk = 1ull << 20;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back([&] { for (;;) { const uint64_t c = next.fetch_add(1); if (c * chunk >= m) break; f(c * chunk, std::min(m, (c + 1) * chunk)); } });
    for (auto& t : th) t.join();
  };
  par([&](uint64_t b, uint64_t e) { for (uint64_t i = b; i < e; ++i) { w[i] = 1 + (i * 2654435761u) % 100; off[i] = 2 * i; p[i] = 0; } });
  off[m] = 2 * m;
  std::atomic<uint64_t> sink{0};
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
    par([&](uint64_t b, uint64_t e) { uint64_t s = 0; for (uint64_t i = b; i < e; ++i) s += off[i]; const uint64_t* q = reinterpret_cast<const uint64_t*>(w); for (uint64_t i = b; i < e; ++i) s += q[i]; sink += s; });
    double t1 = now();
    par([&](uint64_t b, uint64_t e) { sink += pack_scalar(w, p, b, e); });
    double t2 = now();
    par([&](uint64_t b, uint64_t e) { sink += scan_scalar(off, 2, b, e); });
    double t3 = now();
    par([&](uint64_t b, uint64_t e) { sink += pack_avx2(w, p, b, e); });
    double t4 = now();
    par([&](uint64_t b, uint64_t e) { sink += scan_avx2(off, 2, b, e); });
    double t5 = now();
    std::printf("threads %u: read 4.3 GB %.1f ms (%.0f GB/s) | pack scalar %.1f ms  scan scalar %.1f ms | pack avx2 %.1f ms  scan avx2 %.1f ms\n", nt,
                (t1 - t0) * 1e3, 2 * m * 8 / (t1 - t0) / 1e9, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t5 - t4) * 1e3);
  }
  std::printf("sink %llu avx2 %d avx512f %d\n", (unsigned long long)sink.load(), __builtin_cpu_supports("avx2"), __builtin_cpu_supports("avx512f"));
  return 0;
}
