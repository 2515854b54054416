// Micro-benchmark: how many random 4-byte gathers per second does one B200 sustain from an
// array of a given size (L2-resident or not), as a function of loads in flight per thread?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_bench scripts/micro/gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <int ILP, int MODE>  // MODE 0: ld.ca, 1: ld.cg, 2: indices streamed from memory (ld.cs) + ld.ca gather
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ table, uint32_t mask,
                                                const uint32_t* __restrict__ idx, uint64_t per_thread,
                                                uint32_t* out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t it = 0; it < per_thread; it += ILP) {
    uint32_t a[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      const uint64_t g = (it + k) * nthreads + tid;
      if (MODE == 2) a[k] = __ldcs(idx + g) & mask;
      else a[k] = (uint32_t)mix(g) & mask;
    }
    uint32_t v[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = MODE == 1 ? __ldcg(table + a[k]) : __ldca(table + a[k]);
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc += v[k];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int ILP, int MODE>
void run(const char* name, const uint32_t* table, uint32_t entries, const uint32_t* idx, uint32_t* out, int blocks_per_sm) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * blocks_per_sm;
  const uint64_t total = 1ull << 29;
  const uint64_t per_thread = total / ((uint64_t)grid * 256) / ILP * ILP;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    k_gather<ILP, MODE><<<grid, 256>>>(table, entries - 1, idx, per_thread, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double n = (double)per_thread * grid * 256;
  printf("%-10s table %7u KB  ilp %d  ctas/sm %d : %.3f ms  %.1f G gathers/s  (%.2f sectors/clk/SM at 1.92 GHz)\n", name,
         entries / (1u << 8), ILP, blocks_per_sm, best, n / best / 1e6, n / best / 1e6 / 1.92 / sms);
}

int main() {
  uint32_t *table, *idx, *out;
  const uint32_t max_entries = 1u << 28;  // 1 GB
  cudaMalloc(&table, (size_t)max_entries * 4);
  cudaMemset(table, 1, (size_t)max_entries * 4);
  cudaMalloc(&idx, (size_t)(1ull << 29) * 4 + (1 << 20));
  cudaMemset(idx, 0x5a, (size_t)(1ull << 29) * 4);
  cudaMalloc(&out, 4);
  for (uint32_t lg : {13u, 14u, 15u, 16u, 17u, 19u, 24u, 27u, 28u}) {  // 32 KB .. 512 KB (L1), 2 MB, 64 MB (L2), 512 MB, 1 GB (HBM)
    const uint32_t entries = 1u << lg;
    run<1, 0>("ld.ca", table, entries, idx, out, 8);
    run<4, 0>("ld.ca", table, entries, idx, out, 8);
    run<8, 0>("ld.ca", table, entries, idx, out, 4);
    run<4, 1>("ld.cg", table, entries, idx, out, 8);
    run<8, 1>("ld.cg", table, entries, idx, out, 4);
  }
  printf("cudaGetLastError: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
