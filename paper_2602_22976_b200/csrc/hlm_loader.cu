// hlm_loader.cu -- device-side instance sources and CSR utilities of libhlm_b200.so:
//   * counter-based synthetic generators (the BASELINE.json configs 2-5; definitions in
//     DESIGN.md "Synthetic instances", CPU restatement in oracle/hlm_oracle.c orc_syn_*),
//   * the vertex-incidence CSR builder (counting sort of pins by vertex; the device analogue of
//     hypergraph.hpp:144-151),
//   * exclusive scan, download.
#include <cub/device/device_segmented_sort.cuh>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

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
#define ST_CHECK(expr)                \
  do {                                \
    int _s = (expr);                  \
    if (_s != HLM_B200_OK) return _s; \
  } while (0)

template <typename T>
static int dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = pool_malloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    set_error("cudaMalloc of %zu bytes failed: %s", count * sizeof(T), cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? HLM_B200_ERR_NOMEM : HLM_B200_ERR_CUDA;
  }
  return HLM_B200_OK;
}

static int grid_of(const Graph* g, uint64_t items, int per_block = kBlock) {
  const uint64_t want = (items + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(g->num_sms) * 8;
  return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

// ---------------------------------------------------------------------------------------------
// exclusive scan u32 -> u64 (three passes: chunk sums, one-block scan of the sums, rescan)
// ---------------------------------------------------------------------------------------------
constexpr int kScanItems = 16;
constexpr uint32_t kScanChunk = kBlock * kScanItems;

__global__ void __launch_bounds__(kBlock) k_scan_chunk_sums(const uint32_t* in, uint64_t count,
                                                            unsigned long long* sums) {
  __shared__ unsigned long long s_w[kWarpsPerBlock];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanChunk + threadIdx.x * kScanItems;
  unsigned long long acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < count) acc += in[base + k];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kWarpsPerBlock; ++w) t += s_w[w];
    sums[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_sums(unsigned long long* vals, uint64_t cnt,
                                                    unsigned long long* total) {
  __shared__ unsigned long long s_part[1024];
  const uint64_t per = (cnt + 1023) / 1024;
  const uint64_t b = threadIdx.x * per;
  const uint64_t e = min(cnt, b + per);
  unsigned long long acc = 0;
  for (uint64_t i = b; i < e; ++i) acc += vals[i];
  s_part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int i = 0; i < 1024; ++i) {
      const unsigned long long v = s_part[i];
      s_part[i] = run;
      run += v;
    }
    *total = run;
  }
  __syncthreads();
  unsigned long long run = s_part[threadIdx.x];
  for (uint64_t i = b; i < e; ++i) {
    const unsigned long long v = vals[i];
    vals[i] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(kBlock) k_scan_write(const uint32_t* in, uint64_t count,
                                                       const unsigned long long* sums,
                                                       unsigned long long* out) {
  __shared__ unsigned long long s_w[kWarpsPerBlock];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanChunk + threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  unsigned long long acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < count ? in[base + k] : 0u;
    acc += v[k];
  }
  // exclusive prefix of the per-thread totals across the block
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = acc;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  unsigned long long before = sums[blockIdx.x];
  for (uint32_t w = 0; w < warp; ++w) before += s_w[w];
  unsigned long long run = before + incl - acc;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < count) out[base + k] = run;
    run += v[k];
  }
}

// out has count+1 entries; out[count] = total.
int device_exclusive_scan_u32_to_u64(Graph* g, const uint32_t* in, uint64_t* out, uint64_t count,
                                     uint64_t* total) {
  cudaStream_t s = g->stream;
  const uint64_t chunks = (count + kScanChunk - 1) / kScanChunk;
  unsigned long long* sums = nullptr;
  ST_CHECK(dalloc(&sums, chunks + 1));
  uint64_t tot = 0;
  if (count) {
    k_scan_chunk_sums<<<static_cast<unsigned>(chunks), kBlock, 0, s>>>(in, count, sums);
    k_scan_sums<<<1, 1024, 0, s>>>(sums, chunks, sums + chunks);
    k_scan_write<<<static_cast<unsigned>(chunks), kBlock, 0, s>>>(
        in, count, sums, reinterpret_cast<unsigned long long*>(out));
    CU_CHECK(cudaMemcpyAsync(&tot, sums + chunks, 8, cudaMemcpyDeviceToHost, s));
  }
  CU_CHECK(cudaStreamSynchronize(s));
  CU_CHECK(cudaMemcpyAsync(out + count, &tot, 8, cudaMemcpyHostToDevice, s));
  CU_CHECK(cudaStreamSynchronize(s));
  pool_free(sums);
  CU_CHECK(cudaGetLastError());
  if (total) *total = tot;
  return HLM_B200_OK;
}

// ---------------------------------------------------------------------------------------------
// vertex-incidence CSR (order inside one vertex's list is unspecified; no matcher depends on it)
// ---------------------------------------------------------------------------------------------
// Both passes touch one word per pin at a random vertex.  Once the per-vertex array outgrows L2 those
// are random HBM sectors (2 G of them cost ~300 ms on the 8-uniform shard shape), so the pins are
// streamed several times instead, each time serving only the vertices of one window whose words
// stay in L2: [vlo, vhi).
__global__ void k_degree(const uint32_t* pins, uint64_t kappa, uint32_t vlo, uint32_t vhi, uint32_t* deg) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < kappa;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = __ldcs(pins + i);
    if (v >= vlo && v < vhi) atomicAdd(deg + v, 1u);
  }
}

__global__ void k_copy_u64(const unsigned long long* in, uint64_t count, unsigned long long* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

// pos[v] starts as voff[v]; the returning 64-bit add hands out the slots of v's list
// flag_mode != 0: two pins of every edge get a role, marked in the top bits of their entries -- bit 31 the
// PROPOSER, bit 30 the SECONDER.  The vertex-owned matching kernels look at an edge (read its row from HBM)
// only when the proposer names it as its argmax AND the seconder has said the same through a per-edge bit
// that stays in L2.  1: the first and the second pin; 2: the pins with the smallest and second smallest
// vertex ids, which on an instance renumbered by descending degree are the pins with the most incident
// edges, i.e. the ones least likely to name a given edge (fewest proposals to check).  An edge with a
// single pin plays both roles.
__device__ __forceinline__ void inc_roles(const EdgeCsr& csr, uint64_t b, uint32_t s, int flag_mode, uint32_t& proposer,
                                          uint32_t& seconder) {
  proposer = 0u;
  seconder = s > 1u ? 1u : 0u;
  if (flag_mode != 2) return;
  uint32_t best = 0xffffffffu, next = 0xffffffffu;
  for (uint32_t i = 0; i < s; ++i) {
    const uint32_t v = __ldg(csr.pins + b + i);
    if (v < best) {
      next = best;
      seconder = proposer;
      best = v;
      proposer = i;
    } else if (v < next) {
      next = v;
      seconder = i;
    }
  }
  if (s == 1u) seconder = proposer;
}

__device__ __forceinline__ uint32_t inc_entry(uint32_t id, uint32_t i, uint32_t proposer, uint32_t seconder, int flag_mode) {
  if (flag_mode == 0) return id;
  return id | (i == proposer ? 0x80000000u : 0u) | (i == seconder ? 0x40000000u : 0u);
}

__global__ void k_fill_incidence(const EdgeCsr csr, uint32_t m, uint32_t vlo, uint32_t vhi, unsigned long long* pos,
                                 const uint32_t* orig, uint32_t* vinc, int flag_mode) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    uint64_t b;
    uint32_t s;
    csr.range(e, b, s);
    uint32_t id = 0xffffffffu;  // incidence lists name edges by the caller's ids
    uint32_t proposer = 0, seconder = 0;
    inc_roles(csr, b, s, flag_mode, proposer, seconder);
    for (uint32_t i = 0; i < s; ++i) {
      const uint32_t v = __ldcs(csr.pins + b + i);
      if (v < vlo || v >= vhi) continue;
      if (id == 0xffffffffu) id = orig ? orig[e] : e;
      vinc[atomicAdd(pos + v, 1ull)] = inc_entry(id, i, proposer, seconder, flag_mode);
    }
  }
}

// ---- two-level slot fill ----
// The windowed fill above keeps the cursors in L2 but still scatters its 4-byte writes over a list region
// of hundreds of MB per pass (8-uniform shard shape: 235 ms for 2 G entries).  Here the (vertex, entry)
// pairs are first PARTITIONED by vertex range into buckets whose list region fits L2 (a radix pass: per-CTA
// histogram in shared memory, one range reservation per CTA and bucket, runs of pairs written back to
// back), then every bucket is filled on its own: its cursors and its slice of the list array stay in L2
// and reach HBM once.
constexpr uint32_t kIncMaxBuckets = 4096;
constexpr uint32_t kIncEdgesPerThread = 8;

__global__ void k_inc_bucket_cursors(const unsigned long long* voff, uint32_t n, uint32_t shift, uint32_t buckets,
                                     unsigned long long* bcur) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < buckets; b += gridDim.x * blockDim.x) {
    const unsigned long long first = static_cast<unsigned long long>(b) << shift;
    bcur[b] = voff[first < n ? first : n];
  }
}

__global__ void __launch_bounds__(kBlock) k_inc_partition(const EdgeCsr csr, uint32_t m, const uint32_t* orig, uint32_t shift,
                                                          uint32_t buckets, unsigned long long* bcur, int flag_mode,
                                                          unsigned long long* pairs) {
  extern __shared__ unsigned long long s_mem[];
  unsigned long long* s_base = s_mem;                                  // [buckets]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_mem + buckets);      // [buckets]
  const uint32_t per_block = kBlock * kIncEdgesPerThread;
  for (uint64_t e0 = static_cast<uint64_t>(blockIdx.x) * per_block; e0 < m; e0 += static_cast<uint64_t>(gridDim.x) * per_block) {
    for (uint32_t b = threadIdx.x; b < buckets; b += kBlock) s_cnt[b] = 0u;
    __syncthreads();
    for (uint32_t k = 0; k < kIncEdgesPerThread; ++k) {
      const uint64_t e = e0 + threadIdx.x + static_cast<uint64_t>(k) * kBlock;
      if (e >= m) break;
      uint64_t b;
      uint32_t s;
      csr.range(static_cast<uint32_t>(e), b, s);
      for (uint32_t i = 0; i < s; ++i) atomicAdd(s_cnt + (__ldg(csr.pins + b + i) >> shift), 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < buckets; b += kBlock) {
      const uint32_t c = s_cnt[b];
      s_base[b] = c ? atomicAdd(bcur + b, static_cast<unsigned long long>(c)) : 0ull;
      s_cnt[b] = 0u;
    }
    __syncthreads();
    for (uint32_t k = 0; k < kIncEdgesPerThread; ++k) {
      const uint64_t e = e0 + threadIdx.x + static_cast<uint64_t>(k) * kBlock;
      if (e >= m) break;
      uint64_t b;
      uint32_t s;
      csr.range(static_cast<uint32_t>(e), b, s);
      const uint32_t id = orig ? orig[e] : static_cast<uint32_t>(e);
      uint32_t proposer, seconder;
      inc_roles(csr, b, s, flag_mode, proposer, seconder);
      for (uint32_t i = 0; i < s; ++i) {
        const uint32_t v = __ldg(csr.pins + b + i);
        const uint32_t bk = v >> shift;
        const uint32_t raw = inc_entry(id, i, proposer, seconder, flag_mode);
        pairs[s_base[bk] + atomicAdd(s_cnt + bk, 1u)] = (static_cast<unsigned long long>(v) << 32) | raw;
      }
    }
    __syncthreads();
  }
}

// pairs [begin, end): the entries of the vertices of a few consecutive buckets
__global__ void __launch_bounds__(kBlock) k_inc_fill_bucket(const unsigned long long* pairs, unsigned long long begin,
                                                            unsigned long long end, unsigned long long* pos, uint32_t* vinc) {
  for (unsigned long long p = begin + blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x; p < end;
       p += static_cast<unsigned long long>(gridDim.x) * blockDim.x) {
    const unsigned long long pr = __ldcs(pairs + p);
    vinc[atomicAdd(pos + (pr >> 32), 1ull)] = static_cast<uint32_t>(pr);
  }
}

// true if the two-level fill ran (false: not enough memory for the pair array, or nothing to gain)
static int fill_incidence_partitioned(Graph* g, const EdgeCsr& csr, const uint64_t* voff, uint32_t* vinc, int flag_mode,
                                      bool* done) {
  *done = false;
  if (g->kappa < (1ull << 26) || std::getenv("HLM_B200_INCIDENCE_WINDOWED")) return HLM_B200_OK;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return HLM_B200_OK;
  const size_t need = g->kappa * 8 + static_cast<size_t>(g->n) * 8 + (64u << 20);
  if (need > free_b) return HLM_B200_OK;
  cudaStream_t s = g->stream;
  // buckets: list region of about a quarter of L2, at most kIncMaxBuckets of them (shared-memory histogram)
  const double avg = static_cast<double>(g->kappa) / std::max<uint32_t>(1, g->n);
  uint32_t shift = 10;
  while (shift < 31 && (static_cast<double>(1ull << shift) * avg * 4.0 < static_cast<double>(g->l2_bytes) / 4.0)) ++shift;
  while (((static_cast<uint64_t>(g->n) + (1ull << shift) - 1) >> shift) > kIncMaxBuckets) ++shift;
  const uint32_t buckets = static_cast<uint32_t>((static_cast<uint64_t>(g->n) + (1ull << shift) - 1) >> shift);
  unsigned long long *pairs = nullptr, *bcur = nullptr, *pos = nullptr;
  int rc = dalloc(&pairs, g->kappa);
  if (rc == HLM_B200_OK) rc = dalloc(&bcur, buckets);
  if (rc == HLM_B200_OK) rc = dalloc(&pos, g->n);
  if (rc != HLM_B200_OK) {
    pool_free(pairs);
    pool_free(bcur);
    pool_free(pos);
    cudaGetLastError();
    return HLM_B200_OK;  // fall back to the windowed fill
  }
  const unsigned long long* voffu = reinterpret_cast<const unsigned long long*>(voff);
  k_inc_bucket_cursors<<<grid_of(g, buckets), kBlock, 0, s>>>(voffu, g->n, shift, buckets, bcur);
  const size_t smem = static_cast<size_t>(buckets) * 12;
  cudaFuncSetAttribute(k_inc_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_inc_partition<<<g->num_sms * 4, kBlock, smem, s>>>(csr, g->m, g->orig, shift, buckets, bcur, flag_mode, pairs);
  k_copy_u64<<<grid_of(g, g->n), kBlock, 0, s>>>(voffu, g->n, pos);
  // bucket boundaries on the host: voff at every bucket start (bcur is done with: reuse it, + the end)
  std::vector<unsigned long long> bounds(static_cast<size_t>(buckets) + 1);
  k_inc_bucket_cursors<<<grid_of(g, buckets), kBlock, 0, s>>>(voffu, g->n, shift, buckets, bcur);
  CU_CHECK(cudaMemcpyAsync(bounds.data(), bcur, static_cast<size_t>(buckets) * 8, cudaMemcpyDeviceToHost, s));
  CU_CHECK(cudaMemcpyAsync(&bounds[buckets], voffu + g->n, 8, cudaMemcpyDeviceToHost, s));
  CU_CHECK(cudaStreamSynchronize(s));
  // fill: a few buckets per launch so that their list slices and cursors stay in L2 together
  const unsigned long long per_launch = static_cast<unsigned long long>(g->l2_bytes) / 2 / 4;  // entries
  for (uint32_t b = 0; b < buckets;) {
    uint32_t e = b + 1;
    while (e < buckets && bounds[e + 1] - bounds[b] <= per_launch) ++e;
    const unsigned long long cnt = bounds[e] - bounds[b];
    if (cnt) k_inc_fill_bucket<<<grid_of(g, cnt), kBlock, 0, s>>>(pairs, bounds[b], bounds[e], pos, vinc);
    b = e;
  }
  CU_CHECK(cudaStreamSynchronize(s));
  pool_free(pairs);
  pool_free(bcur);
  pool_free(pos);
  CU_CHECK(cudaGetLastError());
  *done = true;
  return HLM_B200_OK;
}

// voff (n+1) / vinc (kappa) of the CSR `csr` over n vertices; edges are named by orig[] when given
static int build_incidence_into(Graph* g, const EdgeCsr& csr, uint64_t* voff, uint32_t* vinc, int flag_mode = 0) {
  cudaStream_t s = g->stream;
  const bool trace = std::getenv("HLM_B200_TRACE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hlm_b200] incidence: %-20s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  uint32_t* deg = nullptr;
  ST_CHECK(dalloc(&deg, g->n));
  CU_CHECK(cudaMemsetAsync(deg, 0, static_cast<size_t>(g->n) * 4, s));
  // window sizes: half of L2 for the words the atomics hit (4 B per vertex, then 8 B per vertex)
  int l2 = 64 << 20;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device);
  uint64_t budget = std::max<uint64_t>(static_cast<uint64_t>(l2) / 2, 1u << 20);
  if (const char* wenv = std::getenv("HLM_B200_INCIDENCE_WINDOW_MB")) budget = std::max<uint64_t>(1, std::strtoull(wenv, nullptr, 10)) << 20;
  const uint32_t win4 = static_cast<uint32_t>(std::min<uint64_t>(0xffffffffu, budget / 4));
  const uint32_t win8 = static_cast<uint32_t>(std::min<uint64_t>(0xffffffffu, budget / 8));
  if (g->kappa)
    for (uint64_t lo = 0; lo < g->n; lo += win4)
      k_degree<<<grid_of(g, g->kappa), kBlock, 0, s>>>(csr.pins, g->kappa, static_cast<uint32_t>(lo),
                                                      static_cast<uint32_t>(std::min<uint64_t>(g->n, lo + win4)), deg);
  mark("degrees");
  int rc = device_exclusive_scan_u32_to_u64(g, deg, voff, g->n, nullptr);
  pool_free(deg);
  if (rc != HLM_B200_OK) return rc;
  mark("scan");
  bool partitioned = false;
  if (g->m && g->n) ST_CHECK(fill_incidence_partitioned(g, csr, voff, vinc, flag_mode, &partitioned));
  if (partitioned) mark("fill (two-level)");
  if (g->m && g->n && !partitioned) {
    unsigned long long* pos = nullptr;
    ST_CHECK(dalloc(&pos, g->n));
    k_copy_u64<<<grid_of(g, g->n), kBlock, 0, s>>>(reinterpret_cast<const unsigned long long*>(voff), g->n, pos);
    for (uint64_t lo = 0; lo < g->n; lo += win8)
      k_fill_incidence<<<grid_of(g, g->m), kBlock, 0, s>>>(csr, g->m, static_cast<uint32_t>(lo),
                                                           static_cast<uint32_t>(std::min<uint64_t>(g->n, lo + win8)), pos,
                                                           g->orig, vinc, flag_mode);
    CU_CHECK(cudaStreamSynchronize(s));
    mark("fill");
    pool_free(pos);
  }
  CU_CHECK(cudaStreamSynchronize(s));
  CU_CHECK(cudaGetLastError());
  return HLM_B200_OK;
}

// the resident instance's own incidence side (resident vertex numbering), kept for the CREW variant
int build_incidence(Graph* g) {
  if (g->voff) return HLM_B200_OK;
  ST_CHECK(dalloc(&g->voff, static_cast<size_t>(g->n) + 1));
  ST_CHECK(dalloc(&g->vinc, g->kappa + 16));  // padding: the vertex-owned sweep copies windows that end on a multiple of 16 entries
  g->device_bytes += (static_cast<uint64_t>(g->n) + 1) * 8 + g->kappa * 4;
  CU_CHECK(cudaMemsetAsync(g->vinc + g->kappa, 0xff, 64, g->stream));
  g->vinc_flagged = g->m < 0x3fffffffu;  // two role bits per entry
  // proposer of an edge: its highest-degree pin where vertex ids are degree ranks (renumbered, ragged
  // instances: an order of magnitude fewer proposals on skewed degrees), else its first pin
  g->vinc_first_pin = !(g->vold && !g->uniform_d) || std::getenv("HLM_B200_PROPOSER_FIRST") != nullptr;
  return build_incidence_into(g, g->csr(), g->voff, g->vinc, !g->vinc_flagged ? 0 : g->vinc_first_pin ? 1 : 2);
}

// ---------------------------------------------------------------------------------------------
// synthetic instances
// ---------------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t syn_hash(uint64_t seed, uint64_t tag, uint64_t e, uint64_t k) {
  return mix_splitmix(mix_splitmix(mix_splitmix(seed + tag) + e) + k);
}

struct SynParams {
  int32_t family;
  uint32_t n, d, scale;
  uint64_t seed;
  uint32_t edge_begin;  // global id of local edge 0
  uint32_t m_local;
  unsigned long long size_total;  // POWERLAW: sum of floor(2^40 / s^2), s = 2..64
};

__device__ __forceinline__ uint32_t syn_edge_size(const SynParams& p, uint32_t e) {
  if (p.family == HLM_B200_SYN_UNIFORM) return p.d;
  if (p.family == HLM_B200_SYN_RMAT) return 2;
  if (p.family == HLM_B200_SYN_POWERLAW) {
    unsigned long long x = syn_hash(p.seed, 1, e, 0) % p.size_total;
    for (unsigned long long s = 2; s <= 64; ++s) {
      const unsigned long long w = (1ull << 40) / (s * s);
      if (x < w) return static_cast<uint32_t>(s);
      x -= w;
    }
    return 64;
  }
  const uint64_t c = syn_hash(p.seed, 1, e, 0);
  if (c % 1000 == 0) {
    const uint32_t o = static_cast<uint32_t>((c >> 10) % 6);
    const uint32_t f = static_cast<uint32_t>((c >> 16) % (64u << o));
    uint32_t s = (64u << o) + f + 1;
    return s > p.n ? p.n : s;
  }
  const uint64_t gg = (c >> 10) & 0xFFFFFFFFull;
  uint64_t q = 1ull << 32;
  uint32_t k = 0;
  while (k < 30) {
    q = q * 3 / 5;
    if (gg >= q) break;
    ++k;
  }
  const uint32_t s = 2 + k;
  return s > p.n ? p.n : s;
}

__device__ __forceinline__ uint32_t syn_draw_vertex(const SynParams& p, uint32_t e, uint32_t j, uint32_t a) {
  const uint64_t h = syn_hash(p.seed, 2, e, (static_cast<uint64_t>(j) << 32) | a);
  if (p.family == HLM_B200_SYN_POWERLAW) {
    const uint64_t u = h >> 32;
    const uint64_t t1 = (u * u) >> 32;
    const uint64_t t2 = (t1 * u) >> 32;
    return static_cast<uint32_t>((t2 * static_cast<uint64_t>(p.n)) >> 32);
  }
  return static_cast<uint32_t>(__umul64hi(h, static_cast<uint64_t>(p.n)));
}

__global__ void k_syn_sizes(const SynParams p, uint32_t* sizes) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.m_local; i += gridDim.x * blockDim.x)
    sizes[i] = syn_edge_size(p, p.edge_begin + i);
}

// one thread per edge; `off` null means uniform size p.d (or 2 for RMAT)
__global__ void k_syn_pins(const SynParams p, const unsigned long long* off, uint32_t* pins) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.m_local; i += gridDim.x * blockDim.x) {
    const uint32_t e = p.edge_begin + i;
    if (p.family == HLM_B200_SYN_RMAT) {
      uint32_t u = 0, v = 0;
      for (uint32_t a = 0;; ++a) {
        u = 0;
        v = 0;
        uint64_t h = 0;
        for (uint32_t lvl = 0; lvl < p.scale; ++lvl) {
          if ((lvl & 3) == 0) h = syn_hash(p.seed, 2, e, (static_cast<uint64_t>(a) << 32) | (lvl >> 2));
          const uint32_t r = static_cast<uint32_t>((h >> (16 * (lvl & 3))) & 0xFFFFu);
          const uint32_t bu = r >= 49807u;
          const uint32_t bv = (r >= 37356u && r < 49807u) || r >= 62259u;
          u = (u << 1) | bu;
          v = (v << 1) | bv;
        }
        if (u != v) break;
      }
      reinterpret_cast<uint2*>(pins)[i] = make_uint2(u, v);
      continue;
    }
    uint64_t b;
    uint32_t s;
    if (off) {
      b = off[i];
      s = static_cast<uint32_t>(off[i + 1] - b);
    } else {
      b = static_cast<uint64_t>(i) * p.d;
      s = p.d;
    }
    uint32_t* pp = pins + b;
    for (uint32_t j = 0; j < s; ++j) {
      for (uint32_t a = 0;; ++a) {
        const uint32_t v = syn_draw_vertex(p, e, j, a);
        bool seen = false;
        for (uint32_t q = 0; q < j; ++q) seen |= (pp[q] == v);
        if (!seen) {
          pp[j] = v;
          break;
        }
      }
    }
  }
}

__global__ void k_syn_weights(const SynParams p, double* base) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < p.m_local; i += gridDim.x * blockDim.x)
    base[i] = static_cast<double>(1 + syn_hash(p.seed, 3, p.edge_begin + i, 0) % 100);
}

int generate(const hlm_b200_syn_spec* spec, int device, Graph** out) {
  *out = nullptr;
  const uint32_t n = spec->family == HLM_B200_SYN_RMAT ? (spec->scale < 32 ? 1u << spec->scale : 0u) : spec->n;
  if (spec->family < 0 || spec->family > 3 || n < 2 || spec->m == 0 ||
      (spec->family == HLM_B200_SYN_UNIFORM && (spec->d == 0 || spec->d > n || spec->d > 4096))) {
    set_error("bad synthetic instance spec");
    return HLM_B200_ERR_INPUT;
  }
  uint32_t begin = spec->edge_begin, m_local = spec->m_local;
  if (begin == 0 && m_local == 0) m_local = spec->m;
  if (static_cast<uint64_t>(begin) + m_local > spec->m) {
    set_error("edge shard [%u, %u + %u) exceeds m = %u", begin, begin, m_local, spec->m);
    return HLM_B200_ERR_INPUT;
  }
  Graph* g = nullptr;
  ST_CHECK(new_graph(device, &g));
  auto fail = [&](int rc) {
    delete g;
    return rc;
  };
  cudaStream_t s = g->stream;
  g->n = n;
  g->m = m_local;
  g->id_base = begin;
  SynParams p;
  p.family = spec->family;
  p.n = n;
  p.d = spec->d;
  p.scale = spec->scale;
  p.seed = spec->seed;
  p.edge_begin = begin;
  p.m_local = m_local;
  p.size_total = 0;
  for (unsigned long long q = 2; q <= 64; ++q) p.size_total += (1ull << 40) / (q * q);

  int rc;
  const bool uniform = spec->family == HLM_B200_SYN_UNIFORM || spec->family == HLM_B200_SYN_RMAT;
  uint64_t* off64 = nullptr;
  if ((rc = dalloc(&off64, static_cast<size_t>(m_local) + 1)) != HLM_B200_OK) return fail(rc);
  if (uniform) {
    const uint32_t d = spec->family == HLM_B200_SYN_RMAT ? 2u : spec->d;
    p.d = d;
    g->kappa = static_cast<uint64_t>(m_local) * d;
    if ((rc = dalloc(&g->pins, g->kappa)) != HLM_B200_OK) return fail(rc);
    g->device_bytes += g->kappa * 4;
    k_syn_pins<<<grid_of(g, m_local), kBlock, 0, s>>>(p, nullptr, g->pins);
    // uniform instances never materialise offsets
    pool_free(off64);
    g->uniform_d = d;
    g->max_edge_size = d;
    g->num_large = d > kLargeEdge ? m_local : 0;
    if (g->num_large) {
      set_error("uniform synthetic instances support d <= %u", kLargeEdge);
      return fail(HLM_B200_ERR_UNSUPPORTED);
    }
  } else {
    uint32_t* sizes = nullptr;
    if ((rc = dalloc(&sizes, m_local)) != HLM_B200_OK) return fail(rc);
    k_syn_sizes<<<grid_of(g, m_local), kBlock, 0, s>>>(p, sizes);
    rc = device_exclusive_scan_u32_to_u64(g, sizes, off64, m_local, &g->kappa);
    pool_free(sizes);
    if (rc != HLM_B200_OK) {
      pool_free(off64);
      return fail(rc);
    }
    if ((rc = dalloc(&g->pins, g->kappa)) != HLM_B200_OK) {
      pool_free(off64);
      return fail(rc);
    }
    g->device_bytes += g->kappa * 4;
    k_syn_pins<<<grid_of(g, m_local), kBlock, 0, s>>>(
        p, reinterpret_cast<const unsigned long long*>(off64), g->pins);
    if ((rc = finish_graph(g, off64, false)) != HLM_B200_OK) return fail(rc);
  }
  if (spec->int_weights) {
    if ((rc = dalloc(&g->base, m_local)) != HLM_B200_OK) return fail(rc);
    g->device_bytes += static_cast<uint64_t>(m_local) * 8;
    k_syn_weights<<<grid_of(g, m_local), kBlock, 0, s>>>(p, g->base);
    if ((rc = finish_weights(g)) != HLM_B200_OK) return fail(rc);
  } else {
    g->base = nullptr;
    g->base_const = g->base_min = g->base_max = 1.0;
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("synthetic generation failed: %s", cudaGetErrorString(e));
    return fail(HLM_B200_ERR_CUDA);
  }
  if (reorder_enabled() && renumber_enabled() && begin == 0 && m_local == spec->m &&
      (rc = renumber_by_degree(g)) != HLM_B200_OK)
    return fail(rc);
  if (reorder_enabled() && (rc = reorder_by_first_pin(g)) != HLM_B200_OK) return fail(rc);
  if ((rc = build_base_codes(g)) != HLM_B200_OK) return fail(rc);
  *out = g;
  return HLM_B200_OK;
}

// ---------------------------------------------------------------------------------------------
// download
// ---------------------------------------------------------------------------------------------
__global__ void k_widen_offsets(const EdgeCsr csr, uint32_t m, unsigned long long* out) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e <= m;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (csr.uniform_d)
      out[e] = e * csr.uniform_d;
    else if (csr.off32)
      out[e] = csr.off32[e];
    else
      out[e] = csr.off64[e];
  }
}

__global__ void k_map_pins(const uint32_t* pins, uint64_t kappa, const uint32_t* map, uint32_t* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < kappa;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = __ldg(map + pins[i]);
}

__global__ void k_fill_const(double* out, uint32_t m, double v) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) out[e] = v;
}

// ascending edge ids inside every vertex's list (cub segmented sort; not on the matching path)
static int sort_incidence_lists(Graph* g, const uint64_t* voff, uint32_t** vinc) {
  cudaStream_t s = g->stream;
  uint32_t* sorted = nullptr;
  ST_CHECK(dalloc(&sorted, g->kappa + 1));
  const unsigned long long* off = reinterpret_cast<const unsigned long long*>(voff);
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, *vinc, sorted, static_cast<int64_t>(g->kappa),
                                                     static_cast<int64_t>(g->n), off, off + 1, s);
  void* tmp = nullptr;
  if (e == cudaSuccess) e = pool_malloc(&tmp, std::max<size_t>(tmp_bytes, 16));
  if (e == cudaSuccess)
    e = cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, *vinc, sorted, static_cast<int64_t>(g->kappa),
                                           static_cast<int64_t>(g->n), off, off + 1, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  pool_free(tmp);
  if (e != cudaSuccess) {
    pool_free(sorted);
    set_error("sorting the incidence lists failed: %s", cudaGetErrorString(e));
    return HLM_B200_ERR_CUDA;
  }
  pool_free(*vinc);
  *vinc = sorted;
  return HLM_B200_OK;
}

int download(Graph* g, uint64_t* voff, uint32_t* vinc, uint64_t* eoff, uint32_t* pins, double* base) {
  CU_CHECK(cudaSetDevice(g->device));
  cudaStream_t s = g->stream;
  if (eoff) {
    unsigned long long* tmp = nullptr;
    ST_CHECK(dalloc(&tmp, static_cast<size_t>(g->m) + 1));
    k_widen_offsets<<<grid_of(g, g->m + 1ull), kBlock, 0, s>>>(g->csr(), g->m, tmp);
    CU_CHECK(cudaMemcpyAsync(eoff, tmp, (static_cast<size_t>(g->m) + 1) * 8, cudaMemcpyDeviceToHost, s));
    CU_CHECK(cudaStreamSynchronize(s));
    pool_free(tmp);
  }
  // the caller's vertex numbering: pins of the resident rows mapped back through vold[]
  uint32_t* old_pins = nullptr;  // resident edge order, caller's vertex ids
  if (g->vold && g->kappa && (pins || voff || vinc)) {
    ST_CHECK(dalloc(&old_pins, g->kappa));
    k_map_pins<<<grid_of(g, g->kappa), kBlock, 0, s>>>(g->pins, g->kappa, g->vold, old_pins);
  }
  if (pins && g->kappa) {
    const int rc = download_pins_original_order(g, old_pins ? old_pins : g->pins, pins);
    if (rc != HLM_B200_OK) return pool_free(old_pins), rc;
  }
  if (base && g->m) {
    if (g->base) {
      CU_CHECK(cudaMemcpyAsync(base, g->base, static_cast<size_t>(g->m) * 8, cudaMemcpyDeviceToHost, s));
    } else {
      double* tmp = nullptr;
      ST_CHECK(dalloc(&tmp, g->m));
      k_fill_const<<<grid_of(g, g->m), kBlock, 0, s>>>(tmp, g->m, g->base_const);
      CU_CHECK(cudaMemcpyAsync(base, tmp, static_cast<size_t>(g->m) * 8, cudaMemcpyDeviceToHost, s));
      CU_CHECK(cudaStreamSynchronize(s));
      pool_free(tmp);
    }
  }
  if (voff || vinc) {
    const uint64_t* d_voff = nullptr;
    const uint32_t* d_vinc = nullptr;
    uint64_t* t_voff = nullptr;
    uint32_t* t_vinc = nullptr;
    // Built on the fly in the caller's numbering and without the first-pin flags of the resident copy;
    // every list is then sorted ascending, which is what build_hypergraph (hypergraph.hpp:128-133)
    // produces (the slot fill by atomics leaves the order inside a list to chance).
    {
      int rc = dalloc(&t_voff, static_cast<size_t>(g->n) + 1);
      if (rc == HLM_B200_OK) rc = dalloc(&t_vinc, g->kappa + 1);
      if (rc == HLM_B200_OK) {
        EdgeCsr csr = g->csr();
        if (old_pins) csr.pins = old_pins;
        rc = build_incidence_into(g, csr, t_voff, t_vinc);
      }
      if (rc == HLM_B200_OK && vinc && g->kappa) rc = sort_incidence_lists(g, t_voff, &t_vinc);
      if (rc != HLM_B200_OK) return pool_free(old_pins), pool_free(t_voff), pool_free(t_vinc), rc;
      d_voff = t_voff;
      d_vinc = t_vinc;
    }
    if (voff) CU_CHECK(cudaMemcpyAsync(voff, d_voff, (static_cast<size_t>(g->n) + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (vinc && g->kappa) CU_CHECK(cudaMemcpyAsync(vinc, d_vinc, g->kappa * 4, cudaMemcpyDeviceToHost, s));
    CU_CHECK(cudaStreamSynchronize(s));
    pool_free(t_voff);
    pool_free(t_vinc);
  }
  CU_CHECK(cudaStreamSynchronize(s));
  pool_free(old_pins);
  CU_CHECK(cudaGetLastError());
  return HLM_B200_OK;
}

}  // namespace hlmb

// ---------------------------------------------------------------------------------------------
// Loader pass: sort the resident edges by their first pin (counting sort).  Edge order inside
// the instance is free (keys and results use the caller's ids), and with this
// order the pin-0 side of every sweep -- vertex-max, check, invalidate, in every round, because
// list compaction preserves order -- touches consecutive vkey slots: one or two 32-byte sectors
// per warp instead of 32.  Random 8-byte gathers are bounded by the L1 sector rate on B200
// (~0.7 sectors/clk/SM measured), so halving them for graphs halves the sweep time.
// ---------------------------------------------------------------------------------------------
namespace hlmb {

#define CU_CHECK2(expr)                                                                    \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return HLM_B200_ERR_CUDA;                                                            \
    }                                                                                      \
  } while (0)

__global__ void k_first_pin_hist(const uint32_t* pins, uint32_t m, uint32_t d, uint32_t* cnt) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
    atomicAdd(cnt + pins[static_cast<uint64_t>(e) * d], 1u);
}

__global__ void k_first_pin_scatter(const uint32_t* pins, const double* base, uint32_t m, uint32_t d,
                                    const unsigned long long* start, uint32_t* cursor,
                                    uint32_t* new_pins, uint32_t* orig, double* new_base) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint32_t* src = pins + static_cast<uint64_t>(e) * d;
    const uint32_t v = src[0];
    const uint64_t pos = start[v] + atomicAdd(cursor + v, 1u);
    uint32_t* dst = new_pins + pos * d;
    for (uint32_t i = 0; i < d; ++i) dst[i] = src[i];
    orig[pos] = e;
    if (base) new_base[pos] = base[e];
  }
}

__global__ void k_unpermute_rows(const uint32_t* pins, const uint32_t* orig, uint32_t m, uint32_t d,
                                 uint32_t* out) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint32_t* src = pins + static_cast<uint64_t>(e) * d;
    uint32_t* dst = out + static_cast<uint64_t>(orig[e]) * d;
    for (uint32_t i = 0; i < d; ++i) dst[i] = src[i];
  }
}

int reorder_by_first_pin(Graph* g) {
  if (g->orig || !g->uniform_d || g->m < 2) return HLM_B200_OK;
  // Only the CRCW sweeps gain from the order (coalesced first-pin filter words).  The vertex-owned
  // kernels look an edge's row up by its caller id: on a sorted instance that is one more random
  // read per candidate (id -> row), so instances they will run are left in the caller's order.
  if (!crcw_is_faster(g) && !std::getenv("HLM_B200_FORCE_REORDER")) return HLM_B200_OK;
  cudaStream_t s = g->stream;
  const uint32_t m = g->m, d = g->uniform_d;
  uint32_t *cnt = nullptr, *new_pins = nullptr, *orig = nullptr;
  uint64_t* start = nullptr;
  double* new_base = nullptr;
  auto cleanup = [&]() {
    pool_free(cnt);
    pool_free(start);
  };
  int rc;
  if ((rc = dalloc(&cnt, g->n)) != HLM_B200_OK) return rc;
  if ((rc = dalloc(&start, static_cast<size_t>(g->n) + 1)) != HLM_B200_OK) return cleanup(), rc;
  if ((rc = dalloc(&new_pins, g->kappa)) != HLM_B200_OK) return cleanup(), rc;
  if ((rc = dalloc(&orig, m)) != HLM_B200_OK) return cleanup(), pool_free(new_pins), rc;
  if (g->base && (rc = dalloc(&new_base, m)) != HLM_B200_OK)
    return cleanup(), pool_free(new_pins), pool_free(orig), rc;
  CU_CHECK2(cudaMemsetAsync(cnt, 0, static_cast<size_t>(g->n) * 4, s));
  k_first_pin_hist<<<grid_of(g, m), kBlock, 0, s>>>(g->pins, m, d, cnt);
  rc = device_exclusive_scan_u32_to_u64(g, cnt, start, g->n, nullptr);
  if (rc == HLM_B200_OK) {
    CU_CHECK2(cudaMemsetAsync(cnt, 0, static_cast<size_t>(g->n) * 4, s));
    k_first_pin_scatter<<<grid_of(g, m), kBlock, 0, s>>>(
        g->pins, g->base, m, d, reinterpret_cast<const unsigned long long*>(start), cnt, new_pins, orig,
        new_base);
    CU_CHECK2(cudaStreamSynchronize(s));
    CU_CHECK2(cudaGetLastError());
  }
  cleanup();
  if (rc != HLM_B200_OK) {
    pool_free(new_pins);
    pool_free(orig);
    pool_free(new_base);
    return rc;
  }
  pool_free(g->pins);
  g->pins = new_pins;
  g->orig = orig;
  g->base_run = new_base;  // null when the weights are constant
  g->device_bytes += static_cast<uint64_t>(m) * 4 + (new_base ? static_cast<uint64_t>(m) * 8 : 0);
  return HLM_B200_OK;
}

int download_pins_original_order(Graph* g, const uint32_t* resident_pins, uint32_t* host_pins) {
  cudaStream_t s = g->stream;
  if (!g->orig) {
    CU_CHECK2(cudaMemcpyAsync(host_pins, resident_pins, g->kappa * 4, cudaMemcpyDeviceToHost, s));
    CU_CHECK2(cudaStreamSynchronize(s));
    return HLM_B200_OK;
  }
  uint32_t* tmp = nullptr;
  ST_CHECK(dalloc(&tmp, g->kappa));
  k_unpermute_rows<<<grid_of(g, g->m), kBlock, 0, s>>>(resident_pins, g->orig, g->m, g->uniform_d, tmp);
  CU_CHECK2(cudaMemcpyAsync(host_pins, tmp, g->kappa * 4, cudaMemcpyDeviceToHost, s));
  CU_CHECK2(cudaStreamSynchronize(s));
  pool_free(tmp);
  return HLM_B200_OK;
}

}  // namespace hlmb

// ---------------------------------------------------------------------------------------------
// Loader pass: renumber the vertices by descending degree (counting sort on the capped degree).
// Vertex numbering is free (results name edges only).  With this order a vertex's id
// says how hot it is: the filter words and dead bits of the most frequently touched vertices are
// the first few hundred KB of their arrays and stay resident in the SM's L1 (loads of hot ids use
// ld.ca, cold ids bypass L1 with ld.cg so they cannot evict the hot window).  An L1 hit costs a
// third of an L2 sector request (scripts/micro/gather_bench.cu: 860 vs 285 G gathers/s), and the
// round sweeps are bound by exactly that rate.
// ---------------------------------------------------------------------------------------------
namespace hlmb {

constexpr uint32_t kDegCap = 65535;

__global__ void k_degree_hist(const uint32_t* deg, uint32_t n, uint32_t* hist) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t b = kDegCap - min(deg[v], kDegCap);  // bucket 0 = the highest degrees
    // warp-aggregated: low-degree buckets receive millions of increments
    const uint32_t peers = __match_any_sync(__activemask(), b);
    if ((__ffs(peers) - 1) == static_cast<int>(threadIdx.x & 31)) atomicAdd(hist + b, __popc(peers));
  }
}

__global__ void k_degree_rank(const uint32_t* deg, uint32_t n, const unsigned long long* start, uint32_t* cursor,
                              uint32_t* new_id, uint32_t* old_id) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t b = kDegCap - min(deg[v], kDegCap);
    const uint32_t peers = __match_any_sync(__activemask(), b);
    const uint32_t lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (leader == static_cast<int>(lane)) base = atomicAdd(cursor + b, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    const uint32_t id = static_cast<uint32_t>(start[b]) + base + __popc(peers & ((1u << lane) - 1u));
    new_id[v] = id;
    old_id[id] = v;
  }
}

__global__ void k_remap_pins(uint32_t* pins, uint64_t kappa, const uint32_t* new_id) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < kappa;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    pins[i] = __ldg(new_id + pins[i]);
}

int renumber_by_degree(Graph* g) {
  if (g->vold || g->n < 2 || g->kappa == 0) return HLM_B200_OK;
  cudaStream_t s = g->stream;
  uint32_t *deg = nullptr, *hist = nullptr, *new_id = nullptr;
  uint64_t* start = nullptr;
  const uint32_t nb = kDegCap + 1;
  int rc = HLM_B200_OK;
  auto cleanup = [&]() {
    pool_free(deg);
    pool_free(hist);
    pool_free(start);
    pool_free(new_id);
  };
  if ((rc = dalloc(&deg, g->n)) != HLM_B200_OK) return cleanup(), rc;
  if ((rc = dalloc(&hist, nb)) != HLM_B200_OK) return cleanup(), rc;
  if ((rc = dalloc(&start, static_cast<size_t>(nb) + 1)) != HLM_B200_OK) return cleanup(), rc;
  if ((rc = dalloc(&new_id, g->n)) != HLM_B200_OK) return cleanup(), rc;
  if ((rc = dalloc(&g->vold, g->n)) != HLM_B200_OK) return cleanup(), rc;
  g->device_bytes += static_cast<uint64_t>(g->n) * 4;
  CU_CHECK2(cudaMemsetAsync(deg, 0, static_cast<size_t>(g->n) * 4, s));
  CU_CHECK2(cudaMemsetAsync(hist, 0, static_cast<size_t>(nb) * 4, s));
  {  // windows of vertices whose counters stay in L2 (see build_incidence_into)
    int l2 = 64 << 20;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device);
    const uint32_t win = static_cast<uint32_t>(std::max(l2 / 2, 1 << 20) / 4);
    for (uint64_t lo = 0; lo < g->n; lo += win)
      k_degree<<<grid_of(g, g->kappa), kBlock, 0, s>>>(g->pins, g->kappa, static_cast<uint32_t>(lo),
                                                      static_cast<uint32_t>(std::min<uint64_t>(g->n, lo + win)), deg);
  }
  k_degree_hist<<<grid_of(g, g->n), kBlock, 0, s>>>(deg, g->n, hist);
  rc = device_exclusive_scan_u32_to_u64(g, hist, start, nb, nullptr);
  if (rc == HLM_B200_OK) {
    CU_CHECK2(cudaMemsetAsync(hist, 0, static_cast<size_t>(nb) * 4, s));
    k_degree_rank<<<grid_of(g, g->n), kBlock, 0, s>>>(deg, g->n, reinterpret_cast<const unsigned long long*>(start),
                                                      hist, new_id, g->vold);
    k_remap_pins<<<grid_of(g, g->kappa), kBlock, 0, s>>>(g->pins, g->kappa, new_id);
    CU_CHECK2(cudaStreamSynchronize(s));
    CU_CHECK2(cudaGetLastError());
  }
  cleanup();
  return rc;
}

}  // namespace hlmb
