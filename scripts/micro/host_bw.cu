// Host-side probe for the e2e loader design: multi-threaded read bandwidth of pinned host memory
// (uniformity scan of the offsets, packing of the weights), alone and while a H2D copy is running.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t n = 1ull << 28;  // 2 GiB of u64
  uint64_t* off; double* w; uint8_t* packed; uint32_t* pins; void* d;
  cudaHostAlloc(&off, n * 8, cudaHostAllocDefault);
  cudaHostAlloc(&w, n * 8, cudaHostAllocDefault);
  cudaHostAlloc(&packed, n, cudaHostAllocDefault);
  cudaHostAlloc(&pins, n * 8, cudaHostAllocDefault);
  cudaMalloc(&d, n * 8);
  const unsigned hc = std::thread::hardware_concurrency();
  printf("hardware_concurrency %u\n", hc);
  {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < hc; ++t) th.emplace_back([&, t] { for (size_t i = t * (n / hc); i < (t + 1) * (n / hc); ++i) { off[i] = 2 * i; w[i] = 1 + (i * 2654435761u) % 100; pins[2*i] = i; pins[2*i+1] = i + 1; } });
    for (auto& x : th) x.join();
  }
  cudaStream_t s; cudaStreamCreate(&s);
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now(); cudaMemcpyAsync(d, pins, n * 8, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); double t1 = now();
    printf("H2D alone: %.1f ms  %.1f GB/s\n", (t1 - t0) * 1e3, n * 8 / (t1 - t0) / 1e9);
  }
  for (unsigned T : {1u, 4u, 8u, 16u, 32u}) {
    if (T > hc) break;
    for (int with_copy = 0; with_copy < 2; ++with_copy) {
      std::vector<uint64_t> bad(T, 0);
      double t0 = now();
      if (with_copy) cudaMemcpyAsync(d, pins, n * 8, cudaMemcpyHostToDevice, s);
      std::vector<std::thread> th;
      for (unsigned t = 0; t < T; ++t) th.emplace_back([&, t] {
        const size_t b = t * (n / T), e = (t + 1) * (n / T);
        uint64_t acc = 0;
        for (size_t i = b; i + 1 < e; ++i) acc |= (off[i + 1] - off[i]) ^ 2ull;   // uniformity scan
        for (size_t i = b; i < e; ++i) { const double x = w[i]; const uint32_t q = (uint32_t)x; acc |= (q != x) | (q > 255u); packed[i] = (uint8_t)q; }  // pack
        bad[t] = acc; });
      for (auto& x : th) x.join();
      double t1 = now();
      if (with_copy) cudaStreamSynchronize(s);
      double t2 = now();
      printf("threads %2u %s: scan+pack of 4 GiB in %.1f ms (%.1f GB/s read)%s bad=%llu\n", T, with_copy ? "with H2D" : "alone   ", (t1 - t0) * 1e3,
             2.0 * n * 8 / (t1 - t0) / 1e9, with_copy ? "" : "", (unsigned long long)bad[0]);
      if (with_copy) printf("            H2D of 2 GiB finished %.1f ms after start (%.1f GB/s)\n", (t2 - t0) * 1e3, n * 8 / (t2 - t0) / 1e9);
    }
  }
  return 0;
}
