// The loader's AVX2 loops (csrc/hlm_host_simd.cpp) against their scalar forms: same verdict for every
// input, same packed bytes whenever the verdict is "packable".
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <vector>

#include "hlm_host_simd.h"

using namespace hlmb;

static int fails = 0;
static void check(bool ok, const char* what) {
  if (!ok) {
    std::printf("FAILED: %s\n", what);
    ++fails;
  }
}

static void weights_case(const std::vector<double>& w, const char* what) {
  for (uint64_t b : {uint64_t(0), uint64_t(1), uint64_t(3)}) {
    if (b > w.size()) continue;
    std::vector<uint8_t> a(w.size() + 8, 0xAA), c(w.size() + 8, 0xAA);
    const bool ba = host_pack_weights_u8(w.data(), a.data(), b, w.size());
    const bool bc = host_pack_weights_u8_scalar(w.data(), c.data(), b, w.size());
    check(ba == bc, what);
    if (!bc) check(std::memcmp(a.data(), c.data(), a.size()) == 0, what);
    else check(std::memcmp(a.data() + w.size(), c.data() + w.size(), 8) == 0 && std::memcmp(a.data(), c.data(), b) == 0, what);  // no stray writes
  }
}

int main() {
  std::mt19937_64 rng(7);
  for (size_t n : {0u, 1u, 7u, 8u, 9u, 63u, 64u, 1000u, 4099u}) {
    std::vector<double> w(n);
    for (auto& x : w) x = 1 + rng() % 255;
    weights_case(w, "integers 1..255");
    for (auto& x : w) x = rng() % 256;
    weights_case(w, "integers 0..255");
    if (n) {
      const double specials[] = {0.5, 255.5, 256.0, -1.0, -0.0, 1e300, -1e300, 2147483648.0, -2147483648.0, 4294967297.0,
                                 std::numeric_limits<double>::quiet_NaN(), std::numeric_limits<double>::infinity(),
                                 -std::numeric_limits<double>::infinity(), 1.0000000000000002, 254.99999999999997,
                                 std::numeric_limits<double>::denorm_min()};
      for (double sp : specials)
        for (size_t pos : {size_t(0), n / 2, n - 1}) {
          std::vector<double> v(w);
          for (auto& x : v) x = 1 + rng() % 255;
          v[pos] = sp;
          weights_case(v, "special value");
        }
    }
  }
  for (size_t n : {1u, 2u, 8u, 9u, 17u, 1000u, 4099u}) {
    for (uint64_t d : {uint64_t(1), uint64_t(2), uint64_t(8), uint64_t(4096)}) {
      std::vector<uint64_t> off(n + 1);
      for (size_t i = 0; i <= n; ++i) off[i] = i * d;
      check(!host_offsets_differ(off.data(), d, 0, n) && !host_offsets_differ_scalar(off.data(), d, 0, n), "uniform offsets");
      for (size_t pos : {size_t(1), n / 2 + 1, n}) {
        std::vector<uint64_t> o(off);
        if (pos > n) continue;
        o[pos] += 1;  // one longer edge, one shorter (or the last one longer)
        for (uint64_t b : {uint64_t(0), uint64_t(1), uint64_t(5)}) {
          if (b >= n) continue;
          check(host_offsets_differ(o.data(), d, b, n) == host_offsets_differ_scalar(o.data(), d, b, n), "perturbed offsets");
        }
        o[pos] = off[pos] + (uint64_t(1) << 40);
        check(host_offsets_differ(o.data(), d, 0, n) && host_offsets_differ_scalar(o.data(), d, 0, n), "high-word difference");
      }
    }
  }
  // 16-bit edge sizes of ragged instances: exact where every size fits, flagged otherwise
  {
    std::mt19937_64 r2(7);
    for (size_t n : {1u, 3u, 64u, 1000u, 70001u}) {
      std::vector<uint64_t> off(n + 1, 0);
      for (size_t i = 0; i < n; ++i) off[i + 1] = off[i] + r2() % 70;  // sizes 0..69
      std::vector<uint16_t> sz(n, 0xABCD);
      check(!host_pack_sizes_u16(off.data(), sz.data(), 0, n), "sizes fit");
      bool same = true;
      for (size_t i = 0; i < n; ++i) same &= sz[i] == off[i + 1] - off[i];
      check(same, "sizes exact");
      if (n >= 3) {  // a sub-range leaves the rest alone
        std::vector<uint16_t> part(n, 0xABCD);
        check(!host_pack_sizes_u16(off.data(), part.data(), 1, n - 1), "sub-range fits");
        check(part[0] == 0xABCD && part[n - 1] == 0xABCD && part[1] == off[2] - off[1], "sub-range only");
      }
      std::vector<uint64_t> big(off);
      for (size_t i = n / 2 + 1; i <= n; ++i) big[i] += 65536;  // one edge of >= 65 536 pins
      check(host_pack_sizes_u16(big.data(), sz.data(), 0, n), "size beyond 16 bits");
      big[n / 2 + 1] = 65535 + big[n / 2];
      if (n >= 2) {
        std::vector<uint64_t> dec(off);
        dec[n / 2 + 1] = dec[n / 2] + 5;
        dec[n / 2] += 9;  // offsets decrease across one edge
        if (dec[n / 2 + 1] < dec[n / 2]) check(host_pack_sizes_u16(dec.data(), sz.data(), 0, n), "decreasing offsets");
      }
    }
  }
  std::printf("host simd (%s): %s\n", host_simd_level(), fails ? "FAILED" : "ok");
  return fails ? 1 : 0;
}
