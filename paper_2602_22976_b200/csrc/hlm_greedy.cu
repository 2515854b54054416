// hlm_greedy.cu -- the ordered tail of greedy_sorted (local_max_seq.hpp:130-152) on the device.
//
// Variant::greedy runs as local-max rounds under the static order (weight descending, id ascending):
// every round takes all edges that come first among their live neighbours, which is exactly what
// greedy_sorted would take, many at a time.  The number of rounds is the dependency depth of the
// order -- a handful on random instances, but Theta(m) on a unit-weight path in natural order.  So
// after a bounded number of rounds the REST of the instance (edges neither matched nor touching a
// covered vertex) is finished the way the reference does it: sorted once by (weight descending, id
// ascending), then one ordered scan.  The scan is sequential by nature; one warp walks the sorted
// list, the lanes striding the pins of the edge at hand.  O(m log m + kappa) like the reference.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>

#include "hlm_engine.h"

namespace hlmb {

#define CU_CHECK(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return HLM_B200_ERR_CUDA;                                                            \
    }                                                                                      \
  } while (0)

// (caller id << 32 | resident row) of every edge that is still free: not matched, no pin covered
__global__ void __launch_bounds__(kBlock) k_greedy_collect(const EdgeCsr csr, const uint32_t* orig, uint32_t m,
                                                            const uint32_t* dead, const uint32_t* mbits,
                                                            unsigned long long* out, unsigned long long* count) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint32_t id = orig ? orig[e] : e;
    if ((mbits[id >> 5] >> (id & 31u)) & 1u) continue;
    uint64_t b;
    uint32_t s;
    csr.range(e, b, s);
    bool free = true;
    for (uint32_t i = 0; i < s && free; ++i) free = !vertex_dead(dead, csr.pins[b + i]);
    if (free) out[atomicAdd(count, 1ull)] = (static_cast<unsigned long long>(id) << 32) | e;
  }
}

// ascending sort key of "heavier first": the complement of the weight's bit pattern (weights are > 0)
__global__ void k_greedy_keys(const unsigned long long* vals, uint64_t count, const double* base,
                              unsigned long long* keys) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    keys[i] = ~static_cast<unsigned long long>(__double_as_longlong(base[vals[i] >> 32]));
}

// one warp: the edges in order; an edge all of whose pins are uncovered is taken (:140-149)
__global__ void __launch_bounds__(32) k_greedy_scan(const EdgeCsr csr, const unsigned long long* vals, uint64_t count,
                                                     uint32_t* dead, uint32_t* mbits, uint16_t* mround, uint32_t round) {
  const uint32_t lane = threadIdx.x;
  for (uint64_t i0 = 0; i0 < count; i0 += 32) {
    const unsigned long long mine = i0 + lane < count ? vals[i0 + lane] : 0ull;
    const uint32_t todo = static_cast<uint32_t>(min(static_cast<uint64_t>(32), count - i0));
    for (uint32_t k = 0; k < todo; ++k) {
      const unsigned long long v = __shfl_sync(0xffffffffu, mine, k);
      const uint32_t id = static_cast<uint32_t>(v >> 32), row = static_cast<uint32_t>(v);
      uint64_t b;
      uint32_t s;
      csr.range(row, b, s);
      bool free = true;
      for (uint32_t j = lane; j < s && free; j += 32u) free = !((__ldcg(dead + (csr.pins[b + j] >> 5)) >> (csr.pins[b + j] & 31u)) & 1u);
      if (!__all_sync(0xffffffffu, free)) continue;
      for (uint32_t j = lane; j < s; j += 32u) {
        const uint32_t u = csr.pins[b + j];
        atomicOr(dead + (u >> 5), 1u << (u & 31u));
      }
      if (lane == 0) {
        atomicOr(mbits + (id >> 5), 1u << (id & 31u));
        mround[id] = static_cast<uint16_t>(round);
      }
      __threadfence();
      __syncwarp();
    }
  }
}

int greedy_finish(Graph* g, uint32_t round, uint64_t* finished) {
  cudaStream_t s = g->stream;
  Workspace& w = g->ws;
  *finished = 0;
  if (g->m == 0) return HLM_B200_OK;
  unsigned long long *vals = nullptr, *vals2 = nullptr, *keys = nullptr, *keys2 = nullptr, *d_count = nullptr;
  void* tmp = nullptr;
  auto release = [&]() {
    pool_free(vals);
    pool_free(vals2);
    pool_free(keys);
    pool_free(keys2);
    pool_free(d_count);
    pool_free(tmp);
  };
  auto fail = [&](cudaError_t e, const char* what) {
    set_error("greedy tail: %s failed: %s", what, cudaGetErrorString(e));
    release();
    return HLM_B200_ERR_CUDA;
  };
  cudaError_t e = pool_malloc(reinterpret_cast<void**>(&vals), static_cast<size_t>(g->m) * 8);
  if (e == cudaSuccess) e = pool_malloc(reinterpret_cast<void**>(&d_count), 8);
  if (e != cudaSuccess) return fail(e, "allocation");
  CU_CHECK(cudaMemsetAsync(d_count, 0, 8, s));
  const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(static_cast<uint64_t>(g->num_sms) * 8, (g->m + kBlock - 1ull) / kBlock)));
  k_greedy_collect<<<grid, kBlock, 0, s>>>(g->csr(), g->orig, g->m, w.dead, w.mbits, vals, d_count);
  unsigned long long count = 0;
  CU_CHECK(cudaMemcpyAsync(&count, d_count, 8, cudaMemcpyDeviceToHost, s));
  CU_CHECK(cudaStreamSynchronize(s));
  *finished = count;
  if (count == 0) {
    release();
    return HLM_B200_OK;
  }
  // 1. ascending caller id (the high word); 2. stable sort by weight key: equal weights keep the id order
  e = pool_malloc(reinterpret_cast<void**>(&vals2), count * 8);
  if (e != cudaSuccess) return fail(e, "allocation");
  size_t tmp_bytes = 0;
  e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, vals, vals2, static_cast<int64_t>(count), 32, 64, s);
  if (e == cudaSuccess) e = pool_malloc(&tmp, std::max<size_t>(tmp_bytes, 16));
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, vals, vals2, static_cast<int64_t>(count), 32, 64, s);
  if (e != cudaSuccess) return fail(e, "sort by id");
  const unsigned long long* order = vals2;
  if (g->base) {
    e = pool_malloc(reinterpret_cast<void**>(&keys), count * 8);
    if (e == cudaSuccess) e = pool_malloc(reinterpret_cast<void**>(&keys2), count * 8);
    if (e != cudaSuccess) return fail(e, "allocation");
    k_greedy_keys<<<grid, kBlock, 0, s>>>(vals2, count, g->base, keys);
    size_t tmp2 = 0;
    e = cub::DeviceRadixSort::SortPairs(nullptr, tmp2, keys, keys2, vals2, vals, static_cast<int64_t>(count), 0, 64, s);
    if (e == cudaSuccess && tmp2 > tmp_bytes) {
      pool_free(tmp);
      tmp = nullptr;
      e = pool_malloc(&tmp, tmp2);
    }
    if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(tmp, tmp2, keys, keys2, vals2, vals, static_cast<int64_t>(count), 0, 64, s);
    if (e != cudaSuccess) return fail(e, "sort by weight");
    order = vals;
  }
  k_greedy_scan<<<1, 32, 0, s>>>(g->csr(), order, count, w.dead, w.mbits, w.mround, round);
  e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(e, "ordered scan");
  release();
  return HLM_B200_OK;
}

}  // namespace hlmb
