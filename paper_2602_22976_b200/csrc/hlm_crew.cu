// hlm_crew.cu -- CREW variant on the device (reference: local_max_crew, local_max_par.hpp:258-338,
// inside the run_soft_delete skeleton :93-183).
//
// Every quantity is gathered by the task that owns it -- no atomics on priorities:
//   k_crew_refresh   per edge    : wkey[e] = bits(weight(e, r)) for active edges  (:126-135)
//   k_crew_argmax_*  per vertex  : T[v] = argmax over the incidence list under the full reference
//                                  comparator (weight, tie_hash, id) (:137-159); one thread per
//                                  light vertex, one warp (shuffle reduction) per mid vertex, one
//                                  CTA per hub -- "warp-segmented max over each vertex's
//                                  incidence list"
//   k_crew_agree     per edge    : matched iff T[v] == e at every pin (:270-285); matched edges
//                                  are vertex-disjoint, so completion marking (:289-299) is
//                                  exclusive and done in the same kernel
//   k_crew_invalidate per edge   : OR over the pins' dead flags (:301-321); vertex retire (:324-332)
//                                  is implicit in the flag
// Soft deletion like the reference's crew: the structure is swept in full every round.  Natively
// exact: ties are resolved inline, so there is no tie flag and no exact redo here.
// Per-edge state is indexed by the caller's edge ids (the incidence lists name edges that way).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hlm_comm.h"
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

constexpr uint32_t kNoEdge = 0xFFFFFFFFu;
constexpr uint32_t kLightDeg = 32;
constexpr uint32_t kMidDeg = 2048;

struct C2Ctl;
struct ShCtl;

// exchange arrays of an edge-partitioned run on one device (hlm_shard.inc); kept with the first shard
// of the device between matchings
struct ShDevMem {
  uint32_t n = 0;
  unsigned long long* gkey = nullptr;
  unsigned long long* g2 = nullptr;
  uint32_t* xv = nullptr;
  uint32_t* lbits = nullptr;
  uint32_t* lrank = nullptr;
  uint32_t* hmax = nullptr;
  uint32_t* bsum = nullptr;
  uint32_t* counters = nullptr;
  unsigned long long* c64 = nullptr;
  ShCtl* ctl = nullptr;
  ShCtl* h_ctl = nullptr;  // page-locked
  void release() {
    pool_free(gkey);
    pool_free(g2);
    pool_free(xv);
    pool_free(lbits);
    pool_free(lrank);
    pool_free(hmax);
    pool_free(bsum);
    pool_free(counters);
    pool_free(c64);
    pool_free(ctl);
    if (h_ctl) cudaFreeHost(h_ctl);
    *this = ShDevMem();
  }
};

struct CrewState {
  unsigned long long* wkey = nullptr;  // m: weight bits of active edges, 0 otherwise
  uint8_t* estat = nullptr;            // m: EdgeStatus (matching.hpp:50)
  uint32_t* top = nullptr;             // n: T[v] (work-optimal form: the raw incidence entry, id | first-pin flag)
  uint8_t* vdead = nullptr;            // n
  uint32_t* vlist[3] = {nullptr, nullptr, nullptr};  // light / mid / hub vertex ids
  uint32_t vcount[3] = {0, 0, 0};
  uint32_t* counters = nullptr;        // [0] matched this round, [1] deactivated this round
  // ---- work-optimal form (crew2_*) ----
  bool v2 = false;
  uint32_t* winc = nullptr;    // kappa: incidence lists compacted in place, round after round
  uint8_t* vw8 = nullptr;      // kappa: base weight of every incidence entry as a byte (integer weights 0..255)
  uint8_t* ww8 = nullptr;      // kappa: the same, moving with winc
  uint32_t* vlen = nullptr;    // n: live length of a light vertex's list (0: heavy, dead or isolated)
  uint32_t* alive = nullptr;   // m bits, caller edge ids
  uint32_t* vnew = nullptr;    // n bits: vertices covered in this round
  uint8_t* gflag = nullptr;    // n/32: 0 = no list of this 32-vertex group is live any more, else the group's class
  uint8_t* gclass = nullptr;   // n/32: 1 = per-vertex offsets (voff), 2 = group-packed and staged through shared memory
  uint32_t* inv = nullptr;     // m: caller id -> resident row (null: same order)
  uint32_t num_heavy = 0, num_tasks = 0;
  uint32_t* heavy_v = nullptr;      // heavy vertex ids
  uint32_t* heavy_first = nullptr;  // first task of a heavy vertex
  uint32_t* heavy_nt = nullptr;     // its number of tasks
  uint32_t* task_hv = nullptr;      // task -> index into heavy_v
  unsigned long long* task_begin = nullptr;  // first position of the task's chunk
  uint32_t* task_len0 = nullptr;    // chunk length at the start
  uint32_t* task_len = nullptr;     // live length
  unsigned long long* part_key = nullptr;  // per task: best key of the chunk
  uint32_t* part_id = nullptr;
  C2Ctl* rc = nullptr;         // device-resident loop state
  cudaGraph_t graph = nullptr;           // [round 1] -> WHILE { later rounds }
  cudaGraphExec_t graph_exec = nullptr;
  uint32_t graph_head_launches = 0, graph_body_launches = 0;
  int graph_km = -1;
  void* graph_params = nullptr;  // malloc'ed copy of the Crew2Params the graph was captured with
  // ---- edge-partitioned runs (hlm_shard.inc) ----
  unsigned long long* lkey = nullptr;  // n: this shard's maximum at every live vertex (live-slot order)
  uint32_t* mnow = nullptr;            // m bits: matched in the round in progress, not yet committed
  uint32_t* second = nullptr;          // m bits: the seconder of the edge named it in this round
  ShDevMem shdev;                      // the device's exchange arrays, when this is its first shard
};

struct CrewParams {
  EdgeCsr csr;
  const uint32_t* orig;
  const double* base;  // caller order, or null
  double base_const;
  uint32_t n, m, id_base;
  StreamParams stream;
  const unsigned long long* voff;
  const uint32_t* vinc;
  unsigned long long* wkey;
  uint8_t* estat;
  uint32_t* top;
  uint8_t* vdead;
  uint32_t* mbits;
  uint16_t* mround;
  uint32_t* counters;
  uint32_t id_mask;  // incidence entries carry two role flags (bits 31, 30) when the instance has < 2^30 edges
};

template <typename T>
static int calloc_dev(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = pool_malloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) {
    set_error("cudaMalloc of %zu bytes failed: %s", count * sizeof(T), cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? HLM_B200_ERR_NOMEM : HLM_B200_ERR_CUDA;
  }
  return HLM_B200_OK;
}

static int grid_c(const Graph* g, uint64_t items, int per_block = kBlock) {
  const uint64_t want = (items + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(g->num_sms) * 16;
  return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

// (ka, ida) beats (kb, idb) under weight_stream.hpp:105-113; ids are global caller ids
__device__ __forceinline__ bool crew_better(const StreamParams& s, uint32_t r, unsigned long long ka,
                                            uint32_t ida, unsigned long long kb, uint32_t idb) {
  if (ka != kb) return ka > kb;
  if (idb == kNoEdge) return true;
  const unsigned long long ha = tie_hash(s, ida, r), hb = tie_hash(s, idb, r);
  if (ha != hb) return ha > hb;
  return ida > idb;
}

__global__ void k_crew_classify(const unsigned long long* voff, uint32_t n, uint32_t* l0, uint32_t* l1,
                                uint32_t* l2, uint32_t* cnt) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const unsigned long long d = voff[v + 1] - voff[v];
    if (d == 0) continue;
    if (d <= kLightDeg)
      l0[atomicAdd(cnt + 0, 1u)] = v;
    else if (d <= kMidDeg)
      l1[atomicAdd(cnt + 1, 1u)] = v;
    else
      l2[atomicAdd(cnt + 2, 1u)] = v;
  }
}

__global__ void k_crew_refresh(const CrewParams P, uint32_t r) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < P.m; id += gridDim.x * blockDim.x) {
    if (P.estat[id] != 0) continue;
    const double b = P.base ? P.base[id] : P.base_const;
    P.wkey[id] = static_cast<unsigned long long>(__double_as_longlong(edge_weight(P.stream, id + P.id_base, r, b)));
  }
}

__global__ void k_crew_argmax_light(const CrewParams P, const uint32_t* list, uint32_t count, uint32_t r) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const uint32_t v = list[i];
    if (P.vdead[v]) continue;
    unsigned long long bk = 0;
    uint32_t bid = kNoEdge;
    for (unsigned long long p = P.voff[v]; p < P.voff[v + 1]; ++p) {
      const uint32_t id = P.vinc[p] & P.id_mask;
      const unsigned long long k = P.wkey[id];
      if (k != 0 && crew_better(P.stream, r, k, id + P.id_base, bk, bid == kNoEdge ? kNoEdge : bid + P.id_base)) {
        bk = k;
        bid = id;
      }
    }
    P.top[v] = bid;
  }
}

__device__ __forceinline__ void crew_combine(const CrewParams& P, uint32_t r, unsigned long long& bk,
                                             uint32_t& bid, unsigned long long ok, uint32_t oid) {
  if (oid == kNoEdge) return;
  if (bid == kNoEdge || crew_better(P.stream, r, ok, oid + P.id_base, bk, bid + P.id_base)) {
    bk = ok;
    bid = oid;
  }
}

// one warp per vertex: lanes stride the incidence list, butterfly reduction with the comparator
__global__ void __launch_bounds__(kBlock) k_crew_argmax_mid(const CrewParams P, const uint32_t* list,
                                                            uint32_t count, uint32_t r) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  for (uint32_t i = warp; i < count; i += nwarps) {
    const uint32_t v = list[i];
    if (P.vdead[v]) continue;
    unsigned long long bk = 0;
    uint32_t bid = kNoEdge;
    for (unsigned long long p = P.voff[v] + lane; p < P.voff[v + 1]; p += 32) {
      const uint32_t id = P.vinc[p] & P.id_mask;
      const unsigned long long k = P.wkey[id];
      if (k != 0) crew_combine(P, r, bk, bid, k, id);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const uint32_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
      crew_combine(P, r, bk, bid, ok, oid);
    }
    if (lane == 0) P.top[v] = bid;
  }
}

// one CTA per hub vertex
__global__ void __launch_bounds__(kBlock) k_crew_argmax_hub(const CrewParams P, const uint32_t* list,
                                                            uint32_t count, uint32_t r) {
  __shared__ unsigned long long s_k[kWarpsPerBlock];
  __shared__ uint32_t s_id[kWarpsPerBlock];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = blockIdx.x; i < count; i += gridDim.x) {
    const uint32_t v = list[i];
    if (P.vdead[v]) continue;  // uniform across the CTA
    unsigned long long bk = 0;
    uint32_t bid = kNoEdge;
    for (unsigned long long p = P.voff[v] + threadIdx.x; p < P.voff[v + 1]; p += kBlock) {
      const uint32_t id = P.vinc[p] & P.id_mask;
      const unsigned long long k = P.wkey[id];
      if (k != 0) crew_combine(P, r, bk, bid, k, id);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const uint32_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
      crew_combine(P, r, bk, bid, ok, oid);
    }
    __syncthreads();
    if (lane == 0) {
      s_k[warp] = bk;
      s_id[warp] = bid;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kWarpsPerBlock; ++w) crew_combine(P, r, bk, bid, s_k[w], s_id[w]);
      P.top[v] = bid;
    }
  }
}

// PHASE 0: agreement + match + completion marking; PHASE 1: invalidation by segmented OR
template <int PHASE>
__global__ void k_crew_edges(const CrewParams P, uint32_t r) {
  uint32_t local = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < P.m; e += gridDim.x * blockDim.x) {
    const uint32_t id = P.orig ? P.orig[e] : e;
    if (P.estat[id] != 0) continue;
    uint64_t b;
    uint32_t s;
    P.csr.range(e, b, s);
    const uint32_t* pp = P.csr.pins + b;
    if (PHASE == 0) {
      bool all = true;
      for (uint32_t i = 0; i < s && all; ++i) all = (P.top[pp[i]] == id);
      if (all) {
        P.estat[id] = 1;
        P.wkey[id] = 0;
        P.mround[id] = static_cast<uint16_t>(r);
        atomicOr(P.mbits + (id >> 5), 1u << (id & 31));
        for (uint32_t i = 0; i < s; ++i) P.vdead[pp[i]] = 1;
        ++local;
      }
    } else {
      bool touched = false;
      for (uint32_t i = 0; i < s && !touched; ++i) touched = P.vdead[pp[i]] != 0;
      if (touched) {
        P.estat[id] = 2;
        P.wkey[id] = 0;
        ++local;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(P.counters + PHASE, local);
}

void crew_release(Graph* g) {
  CrewState* c = g->crew;
  if (!c) return;
  pool_free(c->wkey);
  pool_free(c->estat);
  pool_free(c->top);
  pool_free(c->vdead);
  for (auto& l : c->vlist) pool_free(l);
  pool_free(c->counters);
  pool_free(c->winc);
  pool_free(c->vw8);
  pool_free(c->ww8);
  pool_free(c->vlen);
  pool_free(c->alive);
  pool_free(c->vnew);
  pool_free(c->gflag);
  pool_free(c->gclass);
  pool_free(c->inv);
  pool_free(c->heavy_v);
  pool_free(c->heavy_first);
  pool_free(c->heavy_nt);
  pool_free(c->task_hv);
  pool_free(c->task_begin);
  pool_free(c->task_len0);
  pool_free(c->task_len);
  pool_free(c->part_key);
  pool_free(c->part_id);
  pool_free(c->rc);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  std::free(c->graph_params);
  pool_free(c->lkey);
  pool_free(c->mnow);
  pool_free(c->second);
  c->shdev.release();
  delete c;
  g->crew = nullptr;
}

static int crew_setup(Graph* g) {
  if (g->crew && !g->crew->v2) return HLM_B200_OK;
  if (g->crew) crew_release(g);
  ST_CHECK(build_incidence(g));
  CrewState* c = new CrewState();
  g->crew = c;
  ST_CHECK(calloc_dev(&c->wkey, g->m));
  ST_CHECK(calloc_dev(&c->estat, g->m));
  ST_CHECK(calloc_dev(&c->top, g->n));
  ST_CHECK(calloc_dev(&c->vdead, g->n));
  for (auto& l : c->vlist) ST_CHECK(calloc_dev(&l, g->n));
  ST_CHECK(calloc_dev(&c->counters, 4));
  g->device_bytes += static_cast<uint64_t>(g->m) * 9 + static_cast<uint64_t>(g->n) * 17;
  cudaStream_t s = g->stream;
  CU_CHECK(cudaMemsetAsync(c->counters, 0, 16, s));
  if (g->n)
    k_crew_classify<<<grid_c(g, g->n), kBlock, 0, s>>>(reinterpret_cast<const unsigned long long*>(g->voff), g->n,
                                                      c->vlist[0], c->vlist[1], c->vlist[2], c->counters);
  CU_CHECK(cudaMemcpyAsync(c->vcount, c->counters, 12, cudaMemcpyDeviceToHost, s));
  CU_CHECK(cudaStreamSynchronize(s));
  CU_CHECK(cudaGetLastError());
  return HLM_B200_OK;
}

static int match_crew_soft(Graph* g, const hlm_b200_stream* st, const hlm_b200_config* cfg, hlm_b200_result* out,
                           int report_variant) {
  const uint32_t requested = cfg->max_rounds ? cfg->max_rounds : default_max_rounds(g->m);
  const uint32_t max_rounds = std::min(requested, 65000u);  // 16-bit round record; see match_crcw
  ST_CHECK(ensure_workspace(g, max_rounds));
  ST_CHECK(crew_setup(g));
  Workspace& w = g->ws;
  CrewState* c = g->crew;
  cudaStream_t s = g->stream;

  CrewParams P;
  std::memset(&P, 0, sizeof(P));
  P.csr = g->csr();
  P.orig = g->orig;
  P.base = g->base;
  P.base_const = g->base_const;
  P.n = g->n;
  P.m = g->m;
  P.id_base = g->id_base;
  P.stream.seed = st->seed;
  P.stream.kind = st->kind;
  P.stream.mode = st->mode;
  P.stream.lo = st->noise_low;
  P.stream.hi = st->noise_high;
  P.stream.width = st->noise_high - st->noise_low;
  P.voff = reinterpret_cast<const unsigned long long*>(g->voff);
  P.vinc = g->vinc;
  P.id_mask = g->vinc_flagged ? 0x3fffffffu : 0xffffffffu;
  P.wkey = c->wkey;
  P.estat = c->estat;
  P.top = c->top;
  P.vdead = c->vdead;
  P.mbits = w.mbits;
  P.mround = w.mround;
  P.counters = c->counters;

  CU_CHECK(cudaEventRecord(w.ev0, s));
  CU_CHECK(cudaMemsetAsync(c->wkey, 0, static_cast<size_t>(g->m) * 8, s));
  CU_CHECK(cudaMemsetAsync(c->estat, 0, g->m, s));
  CU_CHECK(cudaMemsetAsync(c->vdead, 0, g->n, s));
  CU_CHECK(cudaMemsetAsync(w.mbits, 0, static_cast<size_t>(w.mbits_words) * 4, s));
  CU_CHECK(cudaMemsetAsync(w.matched_cnt, 0, static_cast<size_t>(w.rounds_cap) * 4, s));
  CU_CHECK(cudaMemsetAsync(w.deact_cnt, 0, static_cast<size_t>(w.rounds_cap) * 4, s));

  uint32_t active = g->m, round = 0, launches = 0;
  bool limit = false;
  std::vector<uint32_t> matched_r, dropped_r;
  const int egrid = grid_c(g, g->m);
  while (active > 0) {  // local_max_par.hpp:117
    ++round;
    if (round > max_rounds) {  // :119-124
      limit = true;
      --round;
      break;
    }
    CU_CHECK(cudaMemsetAsync(c->counters, 0, 8, s));
    k_crew_refresh<<<egrid, kBlock, 0, s>>>(P, round);
    if (c->vcount[0])
      k_crew_argmax_light<<<grid_c(g, c->vcount[0]), kBlock, 0, s>>>(P, c->vlist[0], c->vcount[0], round);
    if (c->vcount[1])
      k_crew_argmax_mid<<<grid_c(g, c->vcount[1], kWarpsPerBlock), kBlock, 0, s>>>(P, c->vlist[1], c->vcount[1], round);
    if (c->vcount[2])
      k_crew_argmax_hub<<<grid_c(g, c->vcount[2], 1), kBlock, 0, s>>>(P, c->vlist[2], c->vcount[2], round);
    k_crew_edges<0><<<egrid, kBlock, 0, s>>>(P, round);
    k_crew_edges<1><<<egrid, kBlock, 0, s>>>(P, round);
    launches += 3 + (c->vcount[0] != 0) + (c->vcount[1] != 0) + (c->vcount[2] != 0);
    uint32_t cnt[2] = {0, 0};
    CU_CHECK(cudaMemcpyAsync(cnt, c->counters, 8, cudaMemcpyDeviceToHost, s));
    CU_CHECK(cudaStreamSynchronize(s));
    matched_r.push_back(cnt[0]);
    dropped_r.push_back(cnt[0] + cnt[1]);  // assemble_result subtracts the matched ones again
    active -= cnt[0] + cnt[1];
  }
  CU_CHECK(cudaGetLastError());
  if (round) {
    CU_CHECK(cudaMemcpyAsync(w.matched_cnt + 1, matched_r.data(), round * 4ull, cudaMemcpyHostToDevice, s));
    CU_CHECK(cudaMemcpyAsync(w.deact_cnt + 1, dropped_r.data(), round * 4ull, cudaMemcpyHostToDevice, s));
  }
  out->kernel_launches = launches;
  out->engine = HLM_B200_ENGINE_VERTEX_OWNED;
  out->device_edge_visits = static_cast<uint64_t>(g->m) * round;
  int rc = assemble_result(g, round, cfg, report_variant, out);
  if (rc != HLM_B200_OK) return rc;
  if (limit && requested > max_rounds) {
    set_error("the run needs more than %u rounds (16-bit round record)", max_rounds);
    return HLM_B200_ERR_UNSUPPORTED;
  }
  return limit ? HLM_B200_ERR_ROUND_LIMIT : HLM_B200_OK;
}

#include "hlm_crew2.inc"
#include "hlm_shard.inc"

int match_crew(Graph* g, const hlm_b200_stream* st, const hlm_b200_config* cfg, hlm_b200_result* out, int report_variant) {
  const char* env = std::getenv("HLM_B200_CREW_SOFT");
  // the work-optimal form needs the two role flags of the incidence entries (bits 31, 30: < 2^30 edges)
  if ((env && env[0] == '1') || g->m >= 0x3fffffffu) return match_crew_soft(g, st, cfg, out, report_variant);
  return match_crew_compacting(g, st, cfg, out, report_variant);
}

}  // namespace hlmb

using namespace hlmb;

extern "C" {

int hlm_b200_match_sharded(hlm_b200_graph* const* shards, int num_shards, hlm_b200_comm* comm,
                           const hlm_b200_stream* stream, const hlm_b200_config* cfg, hlm_b200_result* results,
                           hlm_b200_shard_report* report) {
  return match_sharded(reinterpret_cast<Graph* const*>(shards), num_shards, reinterpret_cast<Comm*>(comm), stream, cfg,
                       results, report);
}

void hlm_b200_shard_report_free(hlm_b200_shard_report* report) {
  if (!report) return;
  std::free(report->collective_bytes_per_round);
  std::free(report->live_vertices_per_round);
  report->collective_bytes_per_round = nullptr;
  report->live_vertices_per_round = nullptr;
}

}  // extern "C"
