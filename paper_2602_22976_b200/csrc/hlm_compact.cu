// hlm_compact.cu -- compact (local_max_par.hpp:350-454) on the device: rebuild both CSRs over the
// active vertices and edges, renumbered densely and order-preserving by exclusive prefix sums over
// the activity flags (the reference's exclusive_scan, parallel.hpp:83-119, is
// device_exclusive_scan_u32_to_u64 here).  The matching path itself only compacts its active-edge
// lists; this is the reference's public building block of the work-optimal variant as
// a stand-alone operation behind the C-ABI, with the same result, maps, error and WorkCounters.
#include <cstdlib>
#include <cstring>

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

constexpr uint32_t kInvalid = 0xFFFFFFFFu;

// new degree of every active vertex = its incident active edges (:357-366); keep flag = active and
// still incident to something
__global__ void k_cmp_degree(const unsigned long long* voff, const uint32_t* vinc, uint32_t n, const uint8_t* vact,
                             const uint8_t* eact, uint32_t* new_deg, uint32_t* vkeep) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    uint32_t deg = 0;
    if (vact[v])
      for (unsigned long long i = voff[v]; i < voff[v + 1]; ++i) deg += eact[vinc[i]] ? 1u : 0u;
    new_deg[v] = deg;
    vkeep[v] = deg > 0 ? 1u : 0u;
  }
}

__global__ void k_cmp_flags(const uint8_t* act, uint32_t count, uint32_t* keep) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) keep[i] = act[i] ? 1u : 0u;
}

// old id -> new id or kInvalid (:378-388), and the size of every kept item at its new position
__global__ void k_cmp_map(const uint32_t* keep, const unsigned long long* pos, uint32_t count, uint32_t* map,
                          const uint32_t* size_by_old, const unsigned long long* off_by_old, uint32_t* size_by_new) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    if (!keep[i]) {
      map[i] = kInvalid;
      continue;
    }
    const uint32_t id = static_cast<uint32_t>(pos[i]);
    map[i] = id;
    size_by_new[id] = size_by_old ? size_by_old[i] : static_cast<uint32_t>(off_by_old[i + 1] - off_by_old[i]);
  }
}

// incidence rewrite (:420-429): the surviving edges of a kept vertex, in their old order
__global__ void k_cmp_write_incidence(const unsigned long long* voff, const uint32_t* vinc, uint32_t n, const uint32_t* vmap,
                                      const uint32_t* emap, const unsigned long long* new_voff, uint32_t* new_vinc) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (vmap[v] == kInvalid) continue;
    unsigned long long pos = new_voff[vmap[v]];
    for (unsigned long long i = voff[v]; i < voff[v + 1]; ++i) {
      const uint32_t e = emap[vinc[i]];
      if (e != kInvalid) new_vinc[pos++] = e;
    }
  }
}

// member rewrite (:430-443); an active edge with an inactive vertex is the reference's input_error
__global__ void k_cmp_write_members(const unsigned long long* eoff, const uint32_t* pins, const double* base, uint32_t m,
                                    const uint8_t* vact, const uint32_t* vmap, const uint32_t* emap,
                                    const unsigned long long* new_eoff, uint32_t* new_pins, double* new_base,
                                    unsigned long long* bad) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    if (emap[e] == kInvalid) continue;
    unsigned long long pos = new_eoff[emap[e]];
    for (unsigned long long i = eoff[e]; i < eoff[e + 1]; ++i) {
      const uint32_t v = pins[i];
      if (!vact[v]) {
        atomicMin(bad, (static_cast<unsigned long long>(e) << 32) | v);  // the first offender, like the reference's message
        continue;
      }
      new_pins[pos++] = vmap[v];
    }
    new_base[emap[e]] = base[e];
  }
}

namespace {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() { pool_free(p); }
  int alloc(size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = pool_malloc(reinterpret_cast<void**>(&p), count * sizeof(T));
    if (e != cudaSuccess) {
      set_error("device allocation of %zu bytes failed: %s", count * sizeof(T), cudaGetErrorString(e));
      return e == cudaErrorMemoryAllocation ? HLM_B200_ERR_NOMEM : HLM_B200_ERR_CUDA;
    }
    return HLM_B200_OK;
  }
};

int grid_of(const Graph* g, uint64_t items) {
  const uint64_t want = (items + kBlock - 1) / kBlock, cap = static_cast<uint64_t>(g->num_sms) * 8;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

template <typename T>
T* host_alloc(size_t count) {
  return static_cast<T*>(std::malloc(sizeof(T) * (count + 1)));
}

int run_compact(Graph* g, const hlm_b200_csr_view* h, const uint8_t* vact_h, const uint8_t* eact_h, hlm_b200_host_graph* out,
                uint32_t** vmap_out, uint32_t** emap_out, hlm_b200_compact_work* work) {
  cudaStream_t s = g->stream;
  const uint32_t n = h->num_vertices, m = h->num_edges;
  const uint64_t kappa = m ? h->edge_offsets[m] : 0;
  DevBuf<unsigned long long> voff, eoff, vpos, epos, new_voff, new_eoff, bad;
  DevBuf<uint32_t> vinc, pins, new_deg, vkeep, ekeep, vmap, emap, vsizes, esizes, new_vinc, new_pins;
  DevBuf<uint8_t> vact, eact;
  DevBuf<double> base, new_base;
  ST_CHECK(voff.alloc(n + 1ull));
  ST_CHECK(eoff.alloc(m + 1ull));
  ST_CHECK(vinc.alloc(kappa));
  ST_CHECK(pins.alloc(kappa));
  ST_CHECK(base.alloc(m));
  ST_CHECK(vact.alloc(n));
  ST_CHECK(eact.alloc(m));
  ST_CHECK(new_deg.alloc(n));
  ST_CHECK(vkeep.alloc(n));
  ST_CHECK(ekeep.alloc(m));
  ST_CHECK(vpos.alloc(n + 1ull));
  ST_CHECK(epos.alloc(m + 1ull));
  ST_CHECK(vmap.alloc(n));
  ST_CHECK(emap.alloc(m));
  ST_CHECK(bad.alloc(1));
  const unsigned long long zero_off = 0, no_bad = ~0ull;
  CU_CHECK(cudaMemcpyAsync(voff.p, n ? h->vertex_offsets : reinterpret_cast<const uint64_t*>(&zero_off), (n + 1ull) * 8, cudaMemcpyHostToDevice, s));
  CU_CHECK(cudaMemcpyAsync(eoff.p, m ? h->edge_offsets : reinterpret_cast<const uint64_t*>(&zero_off), (m + 1ull) * 8, cudaMemcpyHostToDevice, s));
  if (kappa) {
    CU_CHECK(cudaMemcpyAsync(vinc.p, h->vertex_incidence, kappa * 4, cudaMemcpyHostToDevice, s));
    CU_CHECK(cudaMemcpyAsync(pins.p, h->edge_members, kappa * 4, cudaMemcpyHostToDevice, s));
  }
  if (m) {
    CU_CHECK(cudaMemcpyAsync(base.p, h->base_weights, m * 8ull, cudaMemcpyHostToDevice, s));
    CU_CHECK(cudaMemcpyAsync(eact.p, eact_h, m, cudaMemcpyHostToDevice, s));
  }
  if (n) CU_CHECK(cudaMemcpyAsync(vact.p, vact_h, n, cudaMemcpyHostToDevice, s));
  CU_CHECK(cudaMemcpyAsync(bad.p, &no_bad, 8, cudaMemcpyHostToDevice, s));

  if (n) k_cmp_degree<<<grid_of(g, n), kBlock, 0, s>>>(voff.p, vinc.p, n, vact.p, eact.p, new_deg.p, vkeep.p);
  if (m) k_cmp_flags<<<grid_of(g, m), kBlock, 0, s>>>(eact.p, m, ekeep.p);
  uint64_t kept_v = 0, kept_e = 0, new_kappa_v = 0, new_kappa_e = 0;
  ST_CHECK(device_exclusive_scan_u32_to_u64(g, vkeep.p, reinterpret_cast<uint64_t*>(vpos.p), n, &kept_v));  // P_V
  ST_CHECK(device_exclusive_scan_u32_to_u64(g, ekeep.p, reinterpret_cast<uint64_t*>(epos.p), m, &kept_e));  // P_E
  ST_CHECK(vsizes.alloc(kept_v));
  ST_CHECK(esizes.alloc(kept_e));
  ST_CHECK(new_voff.alloc(kept_v + 1));
  ST_CHECK(new_eoff.alloc(kept_e + 1));
  if (n) k_cmp_map<<<grid_of(g, n), kBlock, 0, s>>>(vkeep.p, vpos.p, n, vmap.p, new_deg.p, nullptr, vsizes.p);
  if (m) k_cmp_map<<<grid_of(g, m), kBlock, 0, s>>>(ekeep.p, epos.p, m, emap.p, nullptr, eoff.p, esizes.p);
  ST_CHECK(device_exclusive_scan_u32_to_u64(g, vsizes.p, reinterpret_cast<uint64_t*>(new_voff.p), kept_v, &new_kappa_v));
  ST_CHECK(device_exclusive_scan_u32_to_u64(g, esizes.p, reinterpret_cast<uint64_t*>(new_eoff.p), kept_e, &new_kappa_e));
  ST_CHECK(new_vinc.alloc(new_kappa_v));
  ST_CHECK(new_pins.alloc(new_kappa_e));
  ST_CHECK(new_base.alloc(kept_e));
  if (n) k_cmp_write_incidence<<<grid_of(g, n), kBlock, 0, s>>>(voff.p, vinc.p, n, vmap.p, emap.p, new_voff.p, new_vinc.p);
  if (m)
    k_cmp_write_members<<<grid_of(g, m), kBlock, 0, s>>>(eoff.p, pins.p, base.p, m, vact.p, vmap.p, emap.p, new_eoff.p,
                                                        new_pins.p, new_base.p, bad.p);
  unsigned long long first_bad = ~0ull;
  CU_CHECK(cudaMemcpyAsync(&first_bad, bad.p, 8, cudaMemcpyDeviceToHost, s));
  CU_CHECK(cudaStreamSynchronize(s));
  CU_CHECK(cudaGetLastError());
  if (first_bad != ~0ull) {
    set_error("active edge %u references inactive vertex %u", static_cast<uint32_t>(first_bad >> 32),
              static_cast<uint32_t>(first_bad & 0xFFFFFFFFu));
    return HLM_B200_ERR_INPUT;
  }

  out->num_vertices = static_cast<uint32_t>(kept_v);
  out->num_edges = static_cast<uint32_t>(kept_e);
  out->vertex_offsets = host_alloc<uint64_t>(kept_v + 1);
  out->vertex_incidence = host_alloc<uint32_t>(new_kappa_v);
  out->edge_offsets = host_alloc<uint64_t>(kept_e + 1);
  out->edge_members = host_alloc<uint32_t>(new_kappa_e);
  out->base_weights = host_alloc<double>(kept_e);
  *vmap_out = host_alloc<uint32_t>(n);
  *emap_out = host_alloc<uint32_t>(m);
  if (!out->vertex_offsets || !out->vertex_incidence || !out->edge_offsets || !out->edge_members || !out->base_weights ||
      !*vmap_out || !*emap_out) {
    set_error("host allocation of the compacted hypergraph failed");
    return HLM_B200_ERR_NOMEM;
  }
  CU_CHECK(cudaMemcpyAsync(out->vertex_offsets, new_voff.p, (kept_v + 1) * 8, cudaMemcpyDeviceToHost, s));
  CU_CHECK(cudaMemcpyAsync(out->edge_offsets, new_eoff.p, (kept_e + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (new_kappa_v) CU_CHECK(cudaMemcpyAsync(out->vertex_incidence, new_vinc.p, new_kappa_v * 4, cudaMemcpyDeviceToHost, s));
  if (new_kappa_e) CU_CHECK(cudaMemcpyAsync(out->edge_members, new_pins.p, new_kappa_e * 4, cudaMemcpyDeviceToHost, s));
  if (kept_e) CU_CHECK(cudaMemcpyAsync(out->base_weights, new_base.p, kept_e * 8, cudaMemcpyDeviceToHost, s));
  if (n) CU_CHECK(cudaMemcpyAsync(*vmap_out, vmap.p, n * 4ull, cudaMemcpyDeviceToHost, s));
  if (m) CU_CHECK(cudaMemcpyAsync(*emap_out, emap.p, m * 4ull, cudaMemcpyDeviceToHost, s));
  CU_CHECK(cudaStreamSynchronize(s));
  if (work) {  // local_max_par.hpp:446-453
    work->prefix_sum_invocations = 4;
    work->compactions = 1;
    work->total_pin_visits = 2 * kappa + 3 * new_kappa_e;
    work->total_edge_visits = m;
  }
  return HLM_B200_OK;
}

}  // namespace
}  // namespace hlmb

using namespace hlmb;

extern "C" int hlm_b200_compact(const hlm_b200_csr_view* h, const uint8_t* vertex_active, const uint8_t* edge_active,
                                int device, hlm_b200_host_graph* out, uint32_t** vertex_map, uint32_t** edge_map,
                                hlm_b200_compact_work* work) {
  if (!h || !out || !vertex_map || !edge_map) return HLM_B200_ERR_INPUT;
  std::memset(out, 0, sizeof(*out));
  *vertex_map = *edge_map = nullptr;
  if ((h->num_vertices && (!vertex_active || !h->vertex_offsets)) ||
      (h->num_edges && (!edge_active || !h->edge_offsets || !h->base_weights)) ||
      (h->num_edges && h->edge_offsets[h->num_edges] && (!h->edge_members || !h->vertex_incidence))) {
    set_error("compact needs both CSR sides of the hypergraph and both flag arrays");
    return HLM_B200_ERR_INPUT;
  }
  Graph* g = nullptr;
  int rc = new_graph(device, &g);
  if (rc != HLM_B200_OK) return rc;
  rc = run_compact(g, h, vertex_active, edge_active, out, vertex_map, edge_map, work);
  delete g;
  if (rc != HLM_B200_OK) {
    hlm_b200_host_graph_free(out);
    std::free(*vertex_map);
    std::free(*edge_map);
    *vertex_map = *edge_map = nullptr;
  }
  return rc;
}
