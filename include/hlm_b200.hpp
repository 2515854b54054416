// hlm_b200.hpp -- header-only C++ shim: the reference's matching API on top of the C-ABI.
//
// Include it AFTER the reference's headers ("hlm/hlm.hpp" or "hlm/local_max_par.hpp") and link
// libhlm_b200.so.  It provides, in namespace hlm::b200, functions with the reference's own
// signatures that fill real hlm::MatchResult objects and throw the reference's exception types:
//
//   hlm::MatchResult hlm::b200::run_variant(const Hypergraph&, const WeightStream&, const ParallelConfig&)
//       replaces hlm::run_variant           (local_max_par.hpp:586)
//   hlm::b200::local_max_crcw / local_max_crew
//       replace hlm::local_max_crcw / local_max_crew (local_max_par.hpp:190,258)
//   hlm::VerificationReport hlm::b200::verify_matching(const Hypergraph&, const Matching&)
//       replaces hlm::verify_matching       (exact.hpp:115)
//   class hlm::b200::ResidentHypergraph     -- upload once, match many times (bench protocol)
//
// Errors: HLM_B200_ERR_INPUT -> hlm::input_error; HLM_B200_ERR_ROUND_LIMIT ->
// hlm::round_limit_error carrying the partial matching and report (matching.hpp:77-85);
// anything else -> std::runtime_error.  ParallelConfig::workers / grain are ignored (the device
// decides its own parallelism; results never depend on them, test_par.cpp:32-55).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "hlm_b200.h"

#ifndef HLM_B200_NO_REFERENCE_HEADERS
#include "hlm/exact.hpp"
#include "hlm/local_max_par.hpp"
#endif

namespace hlm {
namespace b200 {

namespace detail {

inline hlm_b200_csr_view view_of(const Hypergraph& h) {
  hlm_b200_csr_view v;
  v.num_vertices = h.num_vertices;
  v.num_edges = h.num_edges;
  v.vertex_offsets = h.vertex_offsets.data();
  v.vertex_incidence = h.vertex_incidence.data();
  v.edge_offsets = h.edge_offsets.data();
  v.edge_members = h.edge_members.data();
  v.base_weights = h.base_weights.data();
  return v;
}

inline hlm_b200_stream stream_of(const WeightStream& s) {
  hlm_b200_stream c;
  c.seed = s.seed;
  c.kind = static_cast<int32_t>(s.kind);
  c.mode = static_cast<int32_t>(s.mode);
  c.noise_low = s.noise_low;
  c.noise_high = s.noise_high;
  return c;
}

inline hlm_b200_config config_of(const ParallelConfig& cfg) {
  hlm_b200_config c;
  c.variant = static_cast<int32_t>(cfg.variant);
  c.max_rounds = cfg.max_rounds;
  c.loop_mode = HLM_B200_LOOP_AUTO;
  c.tie_mode = HLM_B200_TIES_AUTO;
  c.flags = 0;
  c.num_gpus = 0;
  return c;
}

// hlm_b200_result -> hlm::MatchResult (matching.hpp:15-48); frees the C result.
inline MatchResult take(hlm_b200_result& r) {
  MatchResult out;
  Matching& m = out.matching;
  RunReport& rep = out.report;
  m.matched_edges.assign(r.matched_edges, r.matched_edges + r.num_matched);
  m.total_weight = r.total_weight;
  m.rounds_used = r.rounds;
  m.per_round_matched.assign(r.per_round_matched, r.per_round_matched + r.rounds);
  rep.rounds = r.rounds;
  rep.matched_per_round_count = m.per_round_matched;
  rep.deactivated_per_round.assign(r.per_round_deactivated, r.per_round_deactivated + r.rounds);
  rep.matched_per_round.assign(r.rounds, {});
  for (std::uint32_t q = 0; q < r.rounds; ++q) rep.matched_per_round[q].reserve(m.per_round_matched[q]);
  if (r.matched_round)
    for (std::uint64_t i = 0; i < r.num_matched; ++i)  // ids ascend, so every per-round list does too
      rep.matched_per_round[r.matched_round[i] - 1].push_back(r.matched_edges[i]);
  rep.work.rounds = r.rounds;
  rep.work.total_edge_visits = r.total_edge_visits;
  rep.work.total_pin_visits = r.total_pin_visits;
  rep.work.prefix_sum_invocations = r.prefix_sum_invocations;
  rep.work.compactions = r.compactions;
  rep.wall_time_ms = r.wall_time_ms;
  rep.write_conflicts = r.write_conflicts;
  hlm_b200_result_free(&r);
  return out;
}

inline MatchResult finish(int status, hlm_b200_result& r) {
  if (status == HLM_B200_OK) return take(r);
  if (status == HLM_B200_ERR_ROUND_LIMIT) {
    MatchResult partial = take(r);
    throw round_limit_error(std::move(partial.matching), std::move(partial.report));
  }
  const std::string msg = hlm_b200_last_error();
  hlm_b200_result_free(&r);
  if (status == HLM_B200_ERR_INPUT) throw input_error(msg);
  throw std::runtime_error("hlm_b200: " + msg);
}

}  // namespace detail

// run_variant (local_max_par.hpp:586): upload + match + release in one synchronous call.
// num_gpus > 1 (B200 extension): the edge rows are cut into that many blocks over the visible devices
// (hlm_b200_config::num_gpus); the result is the same for every value.
inline MatchResult run_variant(const Hypergraph& h, const WeightStream& stream, const ParallelConfig& cfg,
                               int device = 0, unsigned num_gpus = 0) {
  const hlm_b200_csr_view v = detail::view_of(h);
  const hlm_b200_stream s = detail::stream_of(stream);
  hlm_b200_config c = detail::config_of(cfg);
  c.num_gpus = num_gpus;
  hlm_b200_result r;
  const int st = hlm_b200_match_host(&v, &s, &c, device, &r);
  return detail::finish(st, r);
}

inline MatchResult local_max_crcw(const Hypergraph& h, const WeightStream& stream, ParallelConfig cfg = {}) {
  cfg.variant = Variant::crcw;
  return ::hlm::b200::run_variant(h, stream, cfg, 0);
}

inline MatchResult local_max_crew(const Hypergraph& h, const WeightStream& stream, ParallelConfig cfg = {}) {
  cfg.variant = Variant::crew;
  return ::hlm::b200::run_variant(h, stream, cfg, 0);
}

// local_max_work_optimal (local_max_par.hpp:460): same matching, the variant's own WorkCounters
inline MatchResult local_max_work_optimal(const Hypergraph& h, const WeightStream& stream, ParallelConfig cfg = {}) {
  cfg.variant = Variant::work_optimal;
  return ::hlm::b200::run_variant(h, stream, cfg, 0);
}

// local_max_sequential (local_max_seq.hpp:94)
inline MatchResult local_max_sequential(const Hypergraph& h, const WeightStream& stream, std::uint32_t max_rounds = 0) {
  ParallelConfig cfg;
  cfg.variant = Variant::seq;
  cfg.max_rounds = max_rounds;
  return ::hlm::b200::run_variant(h, stream, cfg, 0);
}

// greedy_sorted (local_max_seq.hpp:130): Matching only, like the reference
inline Matching greedy_sorted(const Hypergraph& h) {
  ParallelConfig cfg;
  cfg.variant = Variant::greedy;
  return ::hlm::b200::run_variant(h, WeightStream{}, cfg, 0).matching;
}

namespace detail {
inline Hypergraph take_host_graph(hlm_b200_host_graph& g) {
  Hypergraph h;
  const std::uint64_t kappa = g.num_edges ? g.edge_offsets[g.num_edges] : 0;
  h.num_vertices = g.num_vertices;
  h.num_edges = g.num_edges;
  h.vertex_offsets.assign(g.vertex_offsets, g.vertex_offsets + g.num_vertices + 1);
  h.vertex_incidence.assign(g.vertex_incidence, g.vertex_incidence + kappa);
  h.edge_offsets.assign(g.edge_offsets, g.edge_offsets + g.num_edges + 1);
  h.edge_members.assign(g.edge_members, g.edge_members + kappa);
  h.base_weights.assign(g.base_weights, g.base_weights + g.num_edges);
  hlm_b200_host_graph_free(&g);
  return h;
}
}  // namespace detail

// generate_random / random_weights_1_100 (generators.hpp:65-101) through the library's host code
#ifndef HLM_B200_NO_REFERENCE_HEADERS
inline Hypergraph generate_random(const RandomInstanceSpec& spec) {
  hlm_b200_host_graph g;
  const int st = hlm_b200_generate_random(spec.num_vertices, spec.num_edges, spec.min_edge_size, spec.max_edge_size,
                                          spec.seed, &g);
  if (st == HLM_B200_ERR_INPUT) throw input_error(hlm_b200_last_error());
  if (st != HLM_B200_OK) throw std::runtime_error(std::string("hlm_b200: ") + hlm_b200_last_error());
  return detail::take_host_graph(g);
}
#endif

inline std::vector<double> random_weights_1_100(std::uint32_t num_edges, std::uint64_t seed) {
  std::vector<double> w(num_edges);
  hlm_b200_random_weights_1_100(num_edges, seed, w.data());
  return w;
}

// compact (local_max_par.hpp:350-454) on the device
inline CompactResult compact(const Hypergraph& h, std::span<const std::uint8_t> vertex_active,
                             std::span<const std::uint8_t> edge_active, unsigned /*workers*/ = 1,
                             WorkCounters* wc = nullptr, int device = 0) {
  const hlm_b200_csr_view v = detail::view_of(h);
  hlm_b200_host_graph g;
  std::uint32_t *vmap = nullptr, *emap = nullptr;
  hlm_b200_compact_work work;
  const int st = hlm_b200_compact(&v, vertex_active.data(), edge_active.data(), device, &g, &vmap, &emap, &work);
  if (st == HLM_B200_ERR_INPUT) throw input_error(hlm_b200_last_error());
  if (st != HLM_B200_OK) throw std::runtime_error(std::string("hlm_b200: ") + hlm_b200_last_error());
  CompactResult out;
  const std::uint64_t kv = g.num_vertices ? g.vertex_offsets[g.num_vertices] : 0;
  const std::uint64_t ke = g.num_edges ? g.edge_offsets[g.num_edges] : 0;
  out.graph.num_vertices = g.num_vertices;
  out.graph.num_edges = g.num_edges;
  out.graph.vertex_offsets.assign(g.vertex_offsets, g.vertex_offsets + g.num_vertices + 1);
  out.graph.vertex_incidence.assign(g.vertex_incidence, g.vertex_incidence + kv);
  out.graph.edge_offsets.assign(g.edge_offsets, g.edge_offsets + g.num_edges + 1);
  out.graph.edge_members.assign(g.edge_members, g.edge_members + ke);
  out.graph.base_weights.assign(g.base_weights, g.base_weights + g.num_edges);
  out.vertex_map.assign(vmap, vmap + h.num_vertices);
  out.edge_map.assign(emap, emap + h.num_edges);
  hlm_b200_host_graph_free(&g);
  hlm_b200_text_free(vmap);
  hlm_b200_text_free(emap);
  if (wc) {
    wc->prefix_sum_invocations += work.prefix_sum_invocations;
    wc->compactions += work.compactions;
    wc->total_pin_visits += work.total_pin_visits;
    wc->total_edge_visits += work.total_edge_visits;
  }
  return out;
}

// An instance resident in HBM: the loader's output.  Matching it repeatedly excludes the
// host-to-device copy, which is the paper's timing protocol.
class ResidentHypergraph {
 public:
  explicit ResidentHypergraph(const Hypergraph& h, int device = 0) {
    const hlm_b200_csr_view v = detail::view_of(h);
    const int st = hlm_b200_graph_upload(&v, device, &g_);
    if (st == HLM_B200_ERR_INPUT) throw input_error(hlm_b200_last_error());
    if (st != HLM_B200_OK) throw std::runtime_error(std::string("hlm_b200: ") + hlm_b200_last_error());
  }
  ResidentHypergraph(const ResidentHypergraph&) = delete;
  ResidentHypergraph& operator=(const ResidentHypergraph&) = delete;
  ~ResidentHypergraph() { hlm_b200_graph_release(g_); }

  MatchResult run_variant(const WeightStream& stream, const ParallelConfig& cfg) const {
    const hlm_b200_stream s = detail::stream_of(stream);
    const hlm_b200_config c = detail::config_of(cfg);
    hlm_b200_result r;
    const int st = hlm_b200_match(g_, &s, &c, &r);
    return detail::finish(st, r);
  }

  // B200 extension (HLM_B200_VARIANT_AUTO): Variant::crcw as far as the caller can tell -- the same
  // matching, report and WorkCounters -- on whichever engine is faster for this instance.
  MatchResult run_fastest(const WeightStream& stream, const ParallelConfig& cfg = ParallelConfig{}) const {
    const hlm_b200_stream s = detail::stream_of(stream);
    hlm_b200_config c = detail::config_of(cfg);
    c.variant = HLM_B200_VARIANT_AUTO;
    hlm_b200_result r;
    const int st = hlm_b200_match(g_, &s, &c, &r);
    return detail::finish(st, r);
  }

  VerificationReport verify_matching(const Matching& m) const {
    int disjoint = 0, maximal = 0;
    double weight = 0.0;
    const int st = hlm_b200_verify(g_, m.matched_edges.data(), m.matched_edges.size(), &disjoint, &maximal, &weight);
    if (st == HLM_B200_ERR_INPUT) throw input_error(hlm_b200_last_error());  // exact.hpp:117
    if (st != HLM_B200_OK) throw std::runtime_error(std::string("hlm_b200: ") + hlm_b200_last_error());
    VerificationReport rep;
    rep.disjoint = disjoint != 0;
    rep.maximal = maximal != 0;
    rep.weight = weight;
    return rep;
  }

 private:
  hlm_b200_graph* g_ = nullptr;
};

inline VerificationReport verify_matching(const Hypergraph& h, const Matching& m, int device = 0) {
  return ResidentHypergraph(h, device).verify_matching(m);
}

}  // namespace b200
}  // namespace hlm
