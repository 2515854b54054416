// ref_driver.cpp -- thin C-ABI wrapper that compiles the UNMODIFIED reference headers where
// they lie (/root/reference/proj/include, passed with -I by oracle/Makefile) into
// oracle/_ref/libhlm_ref.so.  TEST INFRASTRUCTURE ONLY: used to pin the C restatement
// (hlm_oracle.c), to generate tests/golden/*.json, and as bench.py's `--impl reference` /
// cpu_baseline "reference" arm.  No reference source is copied into this repo; this file only
// calls the reference's public API (local_max_par.hpp:586 run_variant, generators.hpp:65,96,
// exact.hpp:115, weight_stream.hpp:78,86).
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>

#include "hlm/hlm.hpp"
#include "hlm_oracle.h"

namespace {

hlm::WeightStream to_stream(const orc_stream* s) {
  hlm::WeightStream w;
  w.seed = s->seed;
  w.kind = static_cast<hlm::GeneratorKind>(s->kind);
  w.mode = static_cast<hlm::WeightMode>(s->mode);
  w.noise_low = s->noise_low;
  w.noise_high = s->noise_high;
  return w;
}

template <typename T>
T* dup_array(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() + 1)));
  if (p && !v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

void export_graph(const hlm::Hypergraph& h, orc_owned_graph* out) {
  out->n = h.num_vertices;
  out->m = h.num_edges;
  out->kappa = h.pin_count();
  out->vertex_offsets = dup_array(h.vertex_offsets);
  out->vertex_incidence = dup_array(h.vertex_incidence);
  out->edge_offsets = dup_array(h.edge_offsets);
  out->edge_members = dup_array(h.edge_members);
  out->base_weights = dup_array(h.base_weights);
}

void fill_result(const hlm::Matching& m, const hlm::RunReport& r, orc_result* out) {
  std::memset(out, 0, sizeof(*out));
  out->num_matched = m.matched_edges.size();
  out->matched_edges = dup_array(m.matched_edges);
  out->matched_round = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (out->num_matched + 1)));
  // round of each matched edge, recovered from the per-round id lists
  {
    std::vector<uint32_t> round_of(m.matched_edges.size(), 0);
    for (std::size_t q = 0; q < r.matched_per_round.size(); ++q)
      for (hlm::edge_id e : r.matched_per_round[q]) {
        auto it = std::lower_bound(m.matched_edges.begin(), m.matched_edges.end(), e);
        round_of[static_cast<std::size_t>(it - m.matched_edges.begin())] =
            static_cast<uint32_t>(q + 1);
      }
    if (!round_of.empty())
      std::memcpy(out->matched_round, round_of.data(), sizeof(uint32_t) * round_of.size());
  }
  out->total_weight = m.total_weight;
  out->rounds = r.rounds;
  out->per_round_matched = dup_array(r.matched_per_round_count);
  out->per_round_deactivated = dup_array(r.deactivated_per_round);
  out->edge_visits = r.work.total_edge_visits;
  out->pin_visits = r.work.total_pin_visits;
  out->wall_ms = r.wall_time_ms;
}

}  // namespace

extern "C" {

// Opaque handle owning a reference hlm::Hypergraph (so repeated timed runs do not re-copy).
void* ref_graph_create(uint32_t n, uint32_t m, const uint64_t* voff, const uint32_t* vinc,
                       const uint64_t* eoff, const uint32_t* pins, const double* base) {
  auto* h = new (std::nothrow) hlm::Hypergraph();
  if (!h) return nullptr;
  const uint64_t kappa = m ? eoff[m] : 0;
  h->num_vertices = n;
  h->num_edges = m;
  h->vertex_offsets.assign(voff, voff + n + 1);
  h->vertex_incidence.assign(vinc, vinc + kappa);
  h->edge_offsets.assign(eoff, eoff + m + 1);
  h->edge_members.assign(pins, pins + kappa);
  h->base_weights.assign(base, base + m);
  return h;
}

void ref_graph_destroy(void* handle) { delete static_cast<hlm::Hypergraph*>(handle); }

unsigned ref_hardware_workers(void) { return hlm::hardware_workers(); }

// variant: hlm::Variant order (local_max_par.hpp:34): 0 seq, 1 crcw, 2 crew, 3 work_optimal, 4 greedy.
// Returns ORC_OK / ORC_INPUT_ERROR / ORC_ROUND_LIMIT (partial result filled) / -1 (other exception).
int ref_run(void* handle, int variant, const orc_stream* s, unsigned workers, uint32_t max_rounds,
            orc_result* out) {
  const auto& h = *static_cast<hlm::Hypergraph*>(handle);
  hlm::ParallelConfig cfg;
  cfg.workers = workers;
  cfg.variant = static_cast<hlm::Variant>(variant);
  cfg.max_rounds = max_rounds;
  try {
    hlm::MatchResult r = hlm::run_variant(h, to_stream(s), cfg);
    fill_result(r.matching, r.report, out);
    return ORC_OK;
  } catch (const hlm::round_limit_error& e) {
    fill_result(e.partial, e.report, out);
    return ORC_ROUND_LIMIT;
  } catch (const hlm::input_error&) {
    std::memset(out, 0, sizeof(*out));
    return ORC_INPUT_ERROR;
  } catch (...) {
    std::memset(out, 0, sizeof(*out));
    return -1;
  }
}

int ref_verify(void* handle, const uint32_t* matched, uint64_t count, int* disjoint, int* maximal,
               double* weight) {
  const auto& h = *static_cast<hlm::Hypergraph*>(handle);
  hlm::Matching m;
  m.matched_edges.assign(matched, matched + count);
  try {
    const hlm::VerificationReport v = hlm::verify_matching(h, m);
    *disjoint = v.disjoint;
    *maximal = v.maximal;
    *weight = v.weight;
    return ORC_OK;
  } catch (const hlm::input_error&) {
    return ORC_INPUT_ERROR;
  }
}

int ref_generate_random(uint32_t nv, uint32_t ne, uint32_t min_size, uint32_t max_size,
                        uint64_t seed, orc_owned_graph* out) {
  std::memset(out, 0, sizeof(*out));
  hlm::RandomInstanceSpec spec;
  spec.num_vertices = nv;
  spec.num_edges = ne;
  spec.min_edge_size = min_size;
  spec.max_edge_size = max_size;
  spec.seed = seed;
  try {
    export_graph(hlm::generate_random(spec), out);
    return ORC_OK;
  } catch (const hlm::input_error&) {
    return ORC_INPUT_ERROR;
  }
}

void ref_random_weights_1_100(uint32_t m, uint64_t seed, double* out) {
  const std::vector<double> w = hlm::random_weights_1_100(m, seed);
  if (m) std::memcpy(out, w.data(), sizeof(double) * m);
}

int ref_tight_family(uint32_t d, double eps, orc_owned_graph* out) {
  std::memset(out, 0, sizeof(*out));
  try {
    export_graph(hlm::generate_tight_family(d, eps), out);
    return ORC_OK;
  } catch (const hlm::input_error&) {
    return ORC_INPUT_ERROR;
  }
}

void ref_eval_stream(const orc_stream* s, const uint32_t* edges, const uint32_t* rounds,
                     const double* base, size_t count, double* w_out, uint64_t* t_out) {
  const hlm::WeightStream w = to_stream(s);
  for (size_t i = 0; i < count; ++i) {
    if (w_out) w_out[i] = w.weight(edges[i], rounds[i], base ? base[i] : 1.0);
    if (t_out) t_out[i] = w.tie_hash(edges[i], rounds[i]);
  }
}

int ref_tie_break(double wa, uint32_t ida, double wb, uint32_t idb, const orc_stream* s,
                  uint32_t round) {
  const auto c = hlm::tie_break(wa, ida, wb, idb, to_stream(s), round);
  return c < 0 ? -1 : (c > 0 ? 1 : 0);
}

uint32_t ref_default_max_rounds(uint32_t m) { return hlm::default_max_rounds(m); }

// ---- io.hpp: the reference's own parsers and writers, for the text-format parity tests ----------
static hlm::ParseOptions parse_options(int degree_zero, std::vector<std::string>* warnings) {
  hlm::ParseOptions o;
  o.degree_zero = degree_zero ? hlm::DegreeZeroPolicy::drop_and_renumber : hlm::DegreeZeroPolicy::reject;
  o.warnings = warnings;
  return o;
}

int ref_parse_hgr(const char* text, size_t len, int degree_zero, orc_owned_graph* out, uint32_t* num_warnings) {
  std::memset(out, 0, sizeof(*out));
  std::vector<std::string> warnings;
  try {
    export_graph(hlm::parse_hgr(std::string(text, len), parse_options(degree_zero, &warnings)), out);
    if (num_warnings) *num_warnings = static_cast<uint32_t>(warnings.size());
    return ORC_OK;
  } catch (const hlm::input_error&) {
    return ORC_INPUT_ERROR;
  }
}

int ref_parse_metis_graph(const char* text, size_t len, int degree_zero, orc_owned_graph* out) {
  std::memset(out, 0, sizeof(*out));
  try {
    export_graph(hlm::parse_metis_graph(std::string(text, len), parse_options(degree_zero, nullptr)), out);
    return ORC_OK;
  } catch (const hlm::input_error&) {
    return ORC_INPUT_ERROR;
  }
}

static char* dup_text(const std::string& s, size_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = 0;
  *len = s.size();
  return p;
}

char* ref_write_hgr(void* handle, size_t* len) {
  std::ostringstream out;
  hlm::write_hgr(*static_cast<hlm::Hypergraph*>(handle), out);
  return dup_text(out.str(), len);
}

char* ref_write_matching(const uint32_t* matched, uint64_t count, double total_weight, uint32_t rounds, size_t* len) {
  hlm::Matching m;
  m.matched_edges.assign(matched, matched + count);
  m.total_weight = total_weight;
  m.rounds_used = rounds;
  std::ostringstream out;
  hlm::write_matching(m, out);
  return dup_text(out.str(), len);
}

int ref_parse_matching(const char* text, size_t len, uint32_t** ids, uint64_t* count) {
  try {
    std::istringstream in(std::string(text, len));
    const std::vector<hlm::edge_id> v = hlm::parse_matching(in);
    *ids = dup_array(v);
    *count = v.size();
    return ORC_OK;
  } catch (const hlm::input_error&) {
    return ORC_INPUT_ERROR;
  }
}

void ref_free_text(void* p) { std::free(p); }

// compact (local_max_par.hpp:350-454): vmap / emap are caller arrays of n / m entries; counters[4] =
// {edge visits, pin visits, prefix sums, compactions} added by this one call
int ref_compact(void* handle, const uint8_t* vact, const uint8_t* eact, unsigned workers, orc_owned_graph* out,
                uint32_t* vmap, uint32_t* emap, uint64_t* counters) {
  std::memset(out, 0, sizeof(*out));
  const auto& h = *static_cast<hlm::Hypergraph*>(handle);
  try {
    hlm::WorkCounters wc;
    hlm::CompactResult c = hlm::compact(h, std::span<const std::uint8_t>(vact, h.num_vertices),
                                        std::span<const std::uint8_t>(eact, h.num_edges), workers, &wc);
    export_graph(c.graph, out);
    if (h.num_vertices) std::memcpy(vmap, c.vertex_map.data(), sizeof(uint32_t) * h.num_vertices);
    if (h.num_edges) std::memcpy(emap, c.edge_map.data(), sizeof(uint32_t) * h.num_edges);
    counters[0] = wc.total_edge_visits;
    counters[1] = wc.total_pin_visits;
    counters[2] = wc.prefix_sum_invocations;
    counters[3] = wc.compactions;
    return ORC_OK;
  } catch (const hlm::input_error&) {
    return ORC_INPUT_ERROR;
  }
}

void ref_free_graph(orc_owned_graph* g) {
  std::free(g->vertex_offsets);
  std::free(g->vertex_incidence);
  std::free(g->edge_offsets);
  std::free(g->edge_members);
  std::free(g->base_weights);
  std::memset(g, 0, sizeof(*g));
}

void ref_free_result(orc_result* r) {
  std::free(r->matched_edges);
  std::free(r->matched_round);
  std::free(r->per_round_matched);
  std::free(r->per_round_deactivated);
  std::memset(r, 0, sizeof(*r));
}

}  // extern "C"
