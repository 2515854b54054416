// Drop-in check of include/hlm_b200.hpp: the reference's own call sites (test_par.cpp:32-55,
// test_seq.cpp:115-134 style) with hlm::b200:: substituted for the parallel matchers, compared
// against the reference's sequential matcher in the same process.
// Built in the container (needs /root/reference headers) by tests/test_shim.py into
// tests/cpp/_build/shim_parity; run on the GPU box by the gpu-marked test.
#include <cstdio>

#include "hlm/hlm.hpp"
#include "hlm_b200.hpp"

using namespace hlm;

static int failures = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

int main() {
  for (std::uint64_t seed = 1; seed <= 20; ++seed) {
    RandomInstanceSpec spec;
    spec.num_vertices = 40 + 25 * static_cast<std::uint32_t>(seed);
    spec.num_edges = 60 + 40 * static_cast<std::uint32_t>(seed);
    spec.min_edge_size = 2;
    spec.max_edge_size = 4;
    spec.seed = seed;
    Hypergraph h = generate_random(spec);
    if (seed % 3 == 0) h.base_weights = random_weights_1_100(h.num_edges, seed);
    WeightStream s;
    s.seed = seed * 7;
    if (seed % 2 == 0) s.mode = WeightMode::replace_uniform;
    if (seed % 5 == 0) s.noise_high = 0.0;
    const MatchResult seq = local_max_sequential(h, s);
    for (Variant v : {Variant::crcw, Variant::crew}) {
      ParallelConfig cfg;
      cfg.variant = v;
      cfg.workers = 8;
      const MatchResult got = b200::run_variant(h, s, cfg);
      CHECK(got.matching.matched_edges == seq.matching.matched_edges);
      CHECK(got.matching.total_weight == seq.matching.total_weight);
      CHECK(got.report.rounds == seq.report.rounds);
      CHECK(got.report.matched_per_round == seq.report.matched_per_round);
      CHECK(got.report.deactivated_per_round == seq.report.deactivated_per_round);
      CHECK(got.report.matched_per_round_count == seq.report.matched_per_round_count);
      const VerificationReport ver = b200::verify_matching(h, got.matching);
      CHECK(ver.valid());
      CHECK(ver.weight == verify_matching(h, got.matching).weight);
    }
    {  // resident instance: upload once, match on the engine the library picks
      const b200::ResidentHypergraph dev(h);
      const MatchResult fast = dev.run_fastest(s);
      ParallelConfig crcw;
      crcw.variant = Variant::crcw;
      const MatchResult plain = dev.run_variant(s, crcw);
      CHECK(fast.matching.matched_edges == seq.matching.matched_edges);
      CHECK(fast.report.matched_per_round == seq.report.matched_per_round);
      CHECK(fast.report.work.total_pin_visits == plain.report.work.total_pin_visits);
      CHECK(fast.report.work.total_edge_visits == plain.report.work.total_edge_visits);
    }
    // every other entry point with the reference's signature
    {
      const MatchResult opt = b200::local_max_work_optimal(h, s);
      ParallelConfig two;
      two.workers = 2;
      const MatchResult ref_opt = local_max_work_optimal(h, s, two);
      CHECK(opt.matching.matched_edges == seq.matching.matched_edges);
      CHECK(opt.report.work.total_pin_visits == ref_opt.report.work.total_pin_visits);
      CHECK(opt.report.work.total_edge_visits == ref_opt.report.work.total_edge_visits);
      CHECK(opt.report.work.compactions == ref_opt.report.work.compactions);
      CHECK(opt.report.work.prefix_sum_invocations == ref_opt.report.work.prefix_sum_invocations);
      CHECK(b200::local_max_sequential(h, s).matching.matched_edges == seq.matching.matched_edges);
      const Matching greedy = b200::greedy_sorted(h), ref_greedy = greedy_sorted(h);
      CHECK(greedy.matched_edges == ref_greedy.matched_edges);
      CHECK(greedy.total_weight == ref_greedy.total_weight);
      CHECK(greedy.per_round_matched == ref_greedy.per_round_matched);
      // compact on the flags left by the first round
      std::vector<std::uint8_t> v_active(h.num_vertices, 1), e_active(h.num_edges, 1);
      for (edge_id e : seq.report.matched_per_round[0])
        for (vertex_id v : h.members_of(e)) v_active[v] = 0;
      for (edge_id e = 0; e < h.num_edges; ++e)
        for (vertex_id v : h.members_of(e))
          if (!v_active[v]) e_active[e] = 0;
      WorkCounters wa, wb;
      const CompactResult ca = b200::compact(h, v_active, e_active, 1, &wa);
      const CompactResult cb = compact(h, v_active, e_active, 2, &wb);
      CHECK(ca.graph == cb.graph);
      CHECK(ca.vertex_map == cb.vertex_map);
      CHECK(ca.edge_map == cb.edge_map);
      CHECK(wa.total_pin_visits == wb.total_pin_visits && wa.total_edge_visits == wb.total_edge_visits);
      CHECK(wa.compactions == wb.compactions && wa.prefix_sum_invocations == wb.prefix_sum_invocations);
    }
    // work counters follow the reference formulas
    ParallelConfig one;
    one.workers = 1;
    CHECK(b200::local_max_crcw(h, s).report.work.total_pin_visits ==
          local_max_crcw(h, s, one).report.work.total_pin_visits);
    CHECK(b200::local_max_crcw(h, s).report.work.total_edge_visits ==
          local_max_crcw(h, s, one).report.work.total_edge_visits);
  }
  // round cap: same exception type, same partial matching (test_par.cpp:86-99)
  {
    std::vector<std::vector<vertex_id>> lists;
    std::vector<double> weights;
    for (vertex_id i = 0; i < 12; ++i) {
      lists.push_back({i, i + 1});
      weights.push_back(1.0 + i);
    }
    Hypergraph h = build_hypergraph(lists, weights);
    WeightStream z;
    z.noise_high = 0.0;
    ParallelConfig cfg;
    cfg.max_rounds = 2;
    bool thrown = false;
    try {
      b200::local_max_crcw(h, z, cfg);
    } catch (const round_limit_error& e) {
      thrown = true;
      CHECK(e.report.rounds == 2);
      try {
        local_max_crcw(h, z, cfg);
      } catch (const round_limit_error& ref) {
        CHECK(e.partial.matched_edges == ref.partial.matched_edges);
        CHECK(e.report.matched_per_round == ref.report.matched_per_round);
      }
    }
    CHECK(thrown);
    WeightStream bad;
    bad.noise_low = 3.0;
    bad.noise_high = 1.0;
    bool input = false;
    try {
      b200::local_max_crcw(h, bad);
    } catch (const input_error&) {
      input = true;
    }
    CHECK(input);
  }
  std::printf(failures ? "shim parity: %d failures\n" : "shim parity: ok\n", failures);
  return failures ? 1 : 0;
}
