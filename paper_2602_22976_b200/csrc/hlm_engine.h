// hlm_engine.h -- host-side types shared by the translation units of libhlm_b200.so.
#pragma once
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include <vector>

#include "../../include/hlm_b200.h"
#include "hlm_types.cuh"

namespace hlmb {

struct Graph;

// Per-instance scratch in HBM, allocated on the first match and reused by later ones.
struct Workspace {
  Ctrl* ctrl = nullptr;
  unsigned long long* vkey = nullptr;
  uint32_t* vtop = nullptr;
  uint32_t* dead = nullptr;
  uint16_t* mround = nullptr;
  uint32_t* mbits = nullptr;
  uint32_t mbits_words = 0;
  uint32_t* seg_ids[2] = {nullptr, nullptr};
  uint32_t* seg_cnt[2] = {nullptr, nullptr};
  uint32_t nseg = 0, seg_cap = 0;
  uint8_t* large_state = nullptr;
  uint32_t* bat_pin0 = nullptr;  // first pin per 32-edge batch, first-pin sorted uniform instances only
  uint32_t* cand_ids = nullptr;
  uint32_t* cand_cnt = nullptr;
  uint32_t* matched_cnt = nullptr;
  uint32_t* deact_cnt = nullptr;
  uint32_t rounds_cap = 0;
  // exact tie path
  unsigned long long* va = nullptr;
  unsigned long long* vb = nullptr;
  uint32_t* vc = nullptr;
  // result assembly
  uint32_t* chunk_cnt = nullptr;
  uint32_t num_chunks = 0;
  unsigned long long* scan_total = nullptr;
  uint32_t* out_ids = nullptr;
  uint16_t* out_round = nullptr;
  double* out_w = nullptr;
  uint64_t out_cap = 0;
  unsigned long long* int_sum = nullptr;
  // pinned host staging of the matched base weights (ordered FP64 sum on the host)
  void* pin_w = nullptr;
  uint64_t pin_cap = 0;
  // CUDA-graph WHILE loop over the round body
  // [0]: round 1 (specialised sweep) followed by the WHILE node; [1]: the WHILE node alone, used
  // to resume after a tie redo or a tag wrap handled by the host
  cudaGraph_t graph[2] = {nullptr, nullptr};
  cudaGraphExec_t graph_exec[2] = {nullptr, nullptr};
  RoundParams graph_key = {};
  uint32_t graph_head_launches = 0;  // round 1 (ahead of the WHILE node)
  uint32_t graph_body_launches = 0;  // one iteration of the WHILE body
  uint32_t launches = 0;
  unsigned long long pins_matched = 0;  // ragged instances: pins of the matched edges of the last run
  // one-launch matching of small instances (k_rounds_fused)
  uint32_t* fused_block_cnt = nullptr;
  unsigned long long* fused_block_isum = nullptr;
  hlmb::FusedSummary* fused_sum = nullptr;  // page-locked host memory
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void drop_graphs();
  void release();
};

struct CrewState;  // hlm_crew.cu

// HLM_B200_TRACE=1: phase times of the loader / a matching on stderr (host clock; `sync` waits for the stream first)
struct PhaseTrace {
  bool on = std::getenv("HLM_B200_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char* what, cudaStream_t sync = nullptr) {
    if (!on) return;
    if (sync) cudaStreamSynchronize(sync);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hlm_b200] %-28s %8.2f ms  (+%.2f)\n", what,
                 std::chrono::duration<double, std::milli>(now - t0).count(),
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

// An instance resident in HBM (pin-CSR as 32-bit arrays, optional incidence-CSR).
struct Graph {
  int device = 0;
  int num_sms = 148;
  int l2_bytes = 126 << 20;
  bool one_shot = false;  // created by hlm_b200_match_host: lives for one matching
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  uint32_t n = 0, m = 0;
  uint32_t id_base = 0;  // global id of local edge 0 (edge shard of a larger instance)
  uint64_t kappa = 0;
  uint32_t* pins = nullptr;
  uint32_t* off32 = nullptr;
  uint64_t* off64 = nullptr;
  uint32_t uniform_d = 0;
  uint32_t max_edge_size = 0;
  uint32_t num_large = 0;
  uint32_t* large_list = nullptr;
  double* base = nullptr;  // null: all weights equal base_const (caller's edge order)
  uint32_t* vold = nullptr;     // resident vertex v is the caller's vertex vold[v] (null: same numbering)
  uint32_t* orig = nullptr;     // resident edge e is the caller's edge orig[e] (null: same order)
  double* base_run = nullptr;   // base weights in resident order when orig != null
  uint8_t* base8 = nullptr;     // resident order, integer weights 0..255: what the gathers of rounds >= 2 read
  double base_const = 1.0;
  double base_min = 1.0, base_max = 1.0;
  bool base_integral = true;  // every base weight is an integer below 2^32 (order-free exact sums)
  // vertex -> incident edges, built on the device when a variant (crew) or a download needs it
  uint64_t* voff = nullptr;  // n+1
  uint32_t* vinc = nullptr;  // kappa
  bool vinc_flagged = false;  // bit 31 of an entry: the list's vertex is the proposer of that edge (m < 2^31)
  bool vinc_first_pin = true;  // the proposer is the edge's first pin (else: its pin with the smallest vertex id)
  uint64_t device_bytes = 0;
  uint64_t h2d_bytes = 0;
  int round_grid = 0, sweep_grid = 0, check_grid = 0, large_grid = 0, fused_grid = 0;
  bool fused_off = false;  // a cooperative launch was refused (SM-limited context): the graph loop from then on
  Workspace ws;
  CrewState* crew = nullptr;
  EdgeCsr csr() const;
  ~Graph();
};

// HBM allocations go through the device's stream-ordered pool with an unlimited release
// threshold: a freed instance's memory stays mapped and the next upload reuses it (plain
// cudaMalloc after a multi-GB cudaFree costs ~0.1 s per GB on this platform).
cudaError_t pool_malloc(void** p, size_t bytes);
void pool_free(void* p);

void set_error(const char* fmt, ...);
void* host_result_alloc(size_t bytes);
void host_result_free(void* p);
uint32_t default_max_rounds(uint32_t m);
int new_graph(int device, Graph** out);
int finish_graph(Graph* g, uint64_t* off64_dev, bool check_pins);
struct WeightStats;
// known: statistics the loader already has (from the packed byte codes); null = one pass over g->base
int finish_weights(Graph* g, const WeightStats* known = nullptr);
int weight_stats(Graph* g, double lo, WeightStats* out);
int build_incidence(Graph* g);
int ensure_workspace(Graph* g, uint32_t max_rounds);
bool reorder_enabled();
bool renumber_enabled();
int reorder_by_first_pin(Graph* g);
bool crcw_is_faster(const Graph* g);
// Rounds first_round.. of a matching on the CRCW kernels, continuing what the vertex-owned engine started
// (hlm_crew2.inc hands over when few edges are left).  Expects in the workspace: seg_ids[0] / seg_cnt[0] =
// the alive class-0 edges (ascending inside every region), large_state, dead = all covered vertices, and
// mbits / mround / matched_cnt / deact_cnt of the rounds so far.
struct CrcwTailOut {
  uint32_t rounds_done = 0, tie_redo = 0, launches = 0, graph_launches = 0;
  bool limit = false;
  std::vector<float> t_filter, t_check;
};
int crcw_tail(Graph* g, const hlm_b200_stream* st, const hlm_b200_config* cfg, uint32_t first_round, uint32_t max_rounds,
              uint32_t alive_small, uint32_t alive_large, CrcwTailOut* out);
// the rest of greedy_sorted as one ordered scan over the still-free edges (hlm_greedy.cu)
int greedy_finish(Graph* g, uint32_t round, uint64_t* finished);
int renumber_by_degree(Graph* g);
int build_base_codes(Graph* g);
int download_pins_original_order(Graph* g, const uint32_t* resident_pins, uint32_t* host_pins);
int generate(const hlm_b200_syn_spec* spec, int device, Graph** out);
int download(Graph* g, uint64_t* voff, uint32_t* vinc, uint64_t* eoff, uint32_t* pins, double* base);
// report_variant: whose WorkCounters formulas the result carries (CREW, or CRCW when AUTO chose this engine)
int match_crew(Graph* g, const hlm_b200_stream* st, const hlm_b200_config* cfg, hlm_b200_result* out,
               int report_variant = HLM_B200_VARIANT_CREW);
void crew_release(Graph* g);
struct Comm;  // hlm_comm.h
int match_sharded(Graph* const* graphs, int num_shards, Comm* comm, const hlm_b200_stream* st, const hlm_b200_config* cfg,
                  hlm_b200_result* results, hlm_b200_shard_report* report);
// result arrays the fused kernel filled before assemble_result runs (page-locked, from host_result_alloc)
struct PreAssembled {
  const hlmb::FusedSummary* sum = nullptr;
  uint32_t* ids = nullptr;
  uint16_t* round = nullptr;
};
int assemble_result(Graph* g, uint32_t rounds, const hlm_b200_config* cfg, int variant,
                    hlm_b200_result* out, double weight_before = 0.0, const PreAssembled* pre = nullptr);
int device_exclusive_scan_u32_to_u64(Graph* g, const uint32_t* in, uint64_t* out, uint64_t count,
                                     uint64_t* total);

}  // namespace hlmb
