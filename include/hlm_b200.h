/*
 * hlm_b200.h -- C-ABI of the B200-native local-max hypergraph matcher (libhlm_b200.so).
 *
 * This is the drop-in boundary for the reference's CPU matching path.  Every entry point names
 * the reference interface it replaces (file:line relative to /root/reference/proj/include/hlm/).
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.  The C++ shim with
 * the reference's own signatures is include/hlm_b200.hpp; the Python binding is
 * paper_2602_22976_b200/_lib.py; the reference-side glue is shown in INTEGRATION.md.
 *
 * All entry points return an hlm_b200_status.  On failure hlm_b200_last_error() holds a
 * message (thread-local).  There is no CPU fallback: without a CUDA device every compute entry
 * point fails with HLM_B200_ERR_CUDA.
 */
#ifndef HLM_B200_H
#define HLM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HLM_B200_ABI_VERSION 3

typedef enum {
  HLM_B200_OK = 0,
  HLM_B200_ERR_INPUT = 1,       /* hlm::input_error   (common.hpp:18)  */
  HLM_B200_ERR_ROUND_LIMIT = 2, /* hlm::round_limit_error (matching.hpp:77); partial result filled */
  HLM_B200_ERR_CUDA = 3,        /* CUDA runtime failure / no device */
  HLM_B200_ERR_NOMEM = 4,
  HLM_B200_ERR_UNSUPPORTED = 5, /* e.g. a Variant this library does not implement */
  HLM_B200_ERR_NCCL = 6         /* libnccl.so.2 missing, or a collective failed */
} hlm_b200_status;

/* hlm::GeneratorKind / hlm::WeightMode (weight_stream.hpp:17-22), same enumerator order. */
enum { HLM_B200_GEN_XORSHIFT = 0, HLM_B200_GEN_PARK_MILLER = 1, HLM_B200_GEN_SPLITMIX = 2 };
enum { HLM_B200_MODE_PERTURB_BASE = 0, HLM_B200_MODE_REPLACE_UNIFORM = 1 };

/* hlm::Variant (local_max_par.hpp:34), same enumerator order.  CRCW and CREW have their own device
 * kernels.  SEQ and WORK_OPTIMAL are accepted and executed by the CRCW kernels (all variants return
 * the same matching by contract, tests/test_par.cpp:32-55; the CRCW path already compacts its
 * active lists every round, which is what work_optimal is for); their WorkCounters follow the
 * reference's own per-variant formulas.  GREEDY (greedy_sorted, local_max_seq.hpp:130) is the
 * lexicographically first maximal matching under (weight descending, id ascending): it runs on the
 * exact three-level path with that static order as the key and reports like the reference does.
 * AUTO (B200 extension, not in the reference's enum) is CRCW as far as the caller can tell -- the same
 * matching, the same report, CRCW's WorkCounters -- with the engine chosen by the library: the
 * vertex-owned CREW kernels when the per-vertex words of the instance outgrow L2 or its edges are
 * ragged / long (there the atomics and the random filter-word reads of the CRCW kernels cost 1.7-3x),
 * the CRCW kernels otherwise and always for the one-shot hlm_b200_match_host (the incidence side
 * the CREW kernels need is built once per resident instance). */
enum {
  HLM_B200_VARIANT_SEQ = 0,
  HLM_B200_VARIANT_CRCW = 1,
  HLM_B200_VARIANT_CREW = 2,
  HLM_B200_VARIANT_WORK_OPTIMAL = 3,
  HLM_B200_VARIANT_GREEDY = 4,
  HLM_B200_VARIANT_AUTO = 5
};

/* Borrowed view of hlm::Hypergraph (hypergraph.hpp:19-27): exactly its five arrays.  The vertex
 * side may be NULL: the library derives the incidence CSR on the device when a variant needs it. */
typedef struct {
  uint32_t num_vertices;
  uint32_t num_edges;
  const uint64_t* vertex_offsets;   /* n+1, or NULL */
  const uint32_t* vertex_incidence; /* kappa, or NULL */
  const uint64_t* edge_offsets;     /* m+1 */
  const uint32_t* edge_members;     /* kappa = edge_offsets[m] */
  const double* base_weights;       /* m, all > 0 */
} hlm_b200_csr_view;

/* hlm::WeightStream (weight_stream.hpp:56-61). */
typedef struct {
  uint64_t seed;
  int32_t kind;
  int32_t mode;
  double noise_low;
  double noise_high;
} hlm_b200_stream;

enum { HLM_B200_LOOP_AUTO = 0, HLM_B200_LOOP_HOST = 1, HLM_B200_LOOP_GRAPH = 2 };
enum { HLM_B200_TIES_AUTO = 0, HLM_B200_TIES_EXACT = 1 };

/* hlm::ParallelConfig (local_max_par.hpp:36-42).  workers / grain have no meaning on a GPU and
 * are absent; assert_exclusive_writes maps to compute-sanitizer runs. */
typedef struct {
  int32_t variant;      /* HLM_B200_VARIANT_* */
  uint32_t max_rounds;  /* 0 selects hlm::default_max_rounds (matching.hpp:87) */
  int32_t loop_mode;    /* HLM_B200_LOOP_*: host-driven rounds or one CUDA-graph WHILE launch */
  int32_t tie_mode;     /* HLM_B200_TIES_AUTO: 64-bit keys + detection + exact redo of a tied round;
                           HLM_B200_TIES_EXACT: three-level (w, tie_hash, id) keys every round */
  uint32_t flags;       /* HLM_B200_FLAG_* */
  uint32_t num_gpus;    /* hlm_b200_match_host only: 0 / 1 = one device; k > 1 = the edge rows are cut into k
                           blocks, block i goes to device (first + i) mod hlm_b200_device_count(), and the
                           blocks are matched as one instance by hlm_b200_match_sharded (blocks that share a
                           device run as co-located shards).  The result does not depend on k -- the
                           reference's "independent of workers" (tests/test_par.cpp:32-55). */
} hlm_b200_config;

#define HLM_B200_FLAG_NO_ROUND_OF 1u   /* do not return matched_round */
#define HLM_B200_FLAG_KERNEL_TIMES 2u  /* host loop only: CUDA-event time of every round kernel */

/* hlm::MatchResult = Matching + RunReport (matching.hpp:15-48), flattened.  Arrays are owned by
 * the library; release with hlm_b200_result_free.  report.matched_per_round[r] is
 * { matched_edges[i] : matched_round[i] == r+1 } (already ascending). */
typedef struct {
  uint32_t* matched_edges;         /* ascending original ids */
  uint16_t* matched_round;         /* parallel to matched_edges, 1-based */
  uint64_t num_matched;
  double total_weight;             /* sum of base weights in ascending-id order */
  uint32_t rounds;
  uint32_t* per_round_matched;     /* rounds entries */
  uint32_t* per_round_deactivated; /* rounds entries */
  uint64_t total_edge_visits;      /* WorkCounters by the reference's per-variant formulas */
  uint64_t total_pin_visits;
  uint64_t device_edge_visits;     /* what the device really swept: sum over rounds of m_r */
  uint64_t device_pin_visits;      /* sum over rounds of kappa_r (pins of the edges active in round r) */
  double wall_time_ms;             /* host clock around the matching (upload excluded) */
  double device_ms;                /* CUDA events around the round loop + result assembly */
  uint32_t tie_redo_rounds;        /* rounds that were redone on the exact three-level path */
  uint32_t kernel_launches;        /* kernels of this library launched by the call */
  uint32_t graph_launches;         /* CUDA-graph launches, or launches of the one-kernel form of small instances (each runs many rounds) */
  uint32_t write_conflicts;        /* always 0 (RunReport::write_conflicts) */
  /* HLM_B200_FLAG_KERNEL_TIMES: rounds + 1 entries each (the last filter launch finds the empty
   * list); NULL otherwise.  CRCW engine: filter = the round sweep (invalidate + compact + vertex-max, all
   * classes), check = k_check_commit.  Vertex-owned engine: filter = the vertex-max sweep (k_c2_argmax_*),
   * check = agreement + deactivation (k_c2_check, k_c2_kill_*, k_c2_count_alive). */
  float* round_filter_ms;
  float* round_check_ms;
  uint64_t h2d_bytes;              /* hlm_b200_match_host: bytes the loader moved host -> device */
  uint32_t prefix_sum_invocations; /* WorkCounters (matching.hpp:27-33): non-zero for WORK_OPTIMAL only */
  uint32_t compactions;
  uint32_t engine;                 /* HLM_B200_ENGINE_*: which kernels ran (what HLM_B200_VARIANT_AUTO chose) */
  uint32_t engine_switch_round;    /* HLM_B200_ENGINE_VERTEX_THEN_CRCW: first round on the CRCW kernels, else 0 */
} hlm_b200_result;

enum { HLM_B200_ENGINE_CRCW = 1, HLM_B200_ENGINE_VERTEX_OWNED = 2, HLM_B200_ENGINE_VERTEX_THEN_CRCW = 3,
       HLM_B200_ENGINE_SHARDED = 4 };

typedef struct hlm_b200_graph hlm_b200_graph; /* opaque: instance resident in HBM */

typedef struct {
  uint32_t num_vertices;
  uint32_t num_edges;
  uint64_t num_pins;
  uint32_t uniform_size;   /* d if every edge has d pins, else 0 */
  uint32_t max_edge_size;
  uint32_t num_large_edges; /* edges handled warp-per-edge (size > 32) */
  int32_t unit_weights;    /* all base weights equal */
  int32_t device;
  uint64_t device_bytes;   /* HBM held by the instance + workspace */
} hlm_b200_graph_info;

/* Synthetic instances generated on the device; the CPU
 * restatement lives in oracle/hlm_oracle.c (orc_syn_generate) and is checked bit-for-bit. */
enum { HLM_B200_SYN_UNIFORM = 0, HLM_B200_SYN_RMAT = 1, HLM_B200_SYN_POWERLAW = 2, HLM_B200_SYN_NETLIST = 3 };
typedef struct {
  int32_t family;
  uint32_t n;
  uint32_t m;
  uint32_t d;
  uint32_t scale;
  uint64_t seed;
  int32_t int_weights;
  /* edge-partition for multi-GPU runs: this graph holds edges [edge_begin, edge_begin + m_local)
   * of the m-edge instance; 0/0 = the whole instance. */
  uint32_t edge_begin;
  uint32_t m_local;
} hlm_b200_syn_spec;

int hlm_b200_abi_version(void);
const char* hlm_b200_last_error(void);
int hlm_b200_device_count(void);

/* Loader: replaces the in-memory hand-over of hlm::Hypergraph to run_variant
 * (tools/hlm_app.hpp:156-165).  Narrows offsets, detects uniform edge size / unit weights, bins
 * large edges, uploads to HBM.  The host arrays are not retained. */
int hlm_b200_graph_upload(const hlm_b200_csr_view* host, int device, hlm_b200_graph** out);
/* The same for one shard of an edge-partitioned instance: `rows` holds the edges [edge_begin, edge_begin +
 * rows->num_edges) of the instance (offsets rebased to 0, vertex ids global); see hlm_b200_match_sharded. */
int hlm_b200_graph_upload_shard(const hlm_b200_csr_view* rows, uint32_t edge_begin, int device, hlm_b200_graph** out);
int hlm_b200_graph_generate(const hlm_b200_syn_spec* spec, int device, hlm_b200_graph** out);
int hlm_b200_graph_info_get(const hlm_b200_graph* g, hlm_b200_graph_info* info);
/* Copies the instance back into caller-allocated host arrays (any pointer may be NULL);
 * vertex side is produced by the device incidence builder. */
int hlm_b200_graph_download(hlm_b200_graph* g, uint64_t* vertex_offsets, uint32_t* vertex_incidence,
                            uint64_t* edge_offsets, uint32_t* edge_members, double* base_weights);
void hlm_b200_graph_release(hlm_b200_graph* g);
/* Runs all later work of this instance on the caller's CUDA stream (a cudaStream_t, e.g. the
 * stream a framework is timing with its own events); NULL restores the instance's own stream. */
int hlm_b200_graph_set_stream(hlm_b200_graph* g, void* cuda_stream);

/* run_variant / local_max_crcw / local_max_crew (local_max_par.hpp:586,190,258) on a resident
 * instance.  Synchronous and re-entrant per graph handle. */
int hlm_b200_match(hlm_b200_graph* g, const hlm_b200_stream* stream, const hlm_b200_config* cfg,
                   hlm_b200_result* out);
/* Same with host arrays in, result out: upload + match + release (the end-to-end drop-in call). */
int hlm_b200_match_host(const hlm_b200_csr_view* host, const hlm_b200_stream* stream,
                        const hlm_b200_config* cfg, int device, hlm_b200_result* out);
void hlm_b200_result_free(hlm_b200_result* r);

/* verify_matching (exact.hpp:115-140) on the device. */
int hlm_b200_verify(hlm_b200_graph* g, const uint32_t* matched, uint64_t count, int* disjoint,
                    int* maximal, double* weight);

/* WeightStream::weight / tie_hash (weight_stream.hpp:78,86) evaluated by the device code the
 * kernels use; host arrays in and out.  For bit-exactness tests of the priority keys. */
int hlm_b200_eval_stream(const hlm_b200_stream* stream, const uint32_t* edges, const uint32_t* rounds,
                         const double* base, size_t count, double* w_out, uint64_t* t_out, int device);

/* ---- edge-partitioned (multi-GPU) runs: round driver in C++, collectives by NCCL --------------
 * No reference counterpart (the reference is single-process; PAPER.md:418 only sketches it).  The round loop, the collectives and the tie handling
 * all live behind one call; the host waits for the device once per round (a 32-byte read-back).
 * Every shard holds the edge rows [edge_begin, edge_begin + m_local) of the instance and the
 * incidence lists of its own edges; per round the ranks all-reduce(max) one uint64 per LIVE vertex
 * and all-reduce(sum) the covered-vertex bitmap (csrc/hlm_shard.inc has the protocol).
 *
 * hlm_b200_comm: one rank of an NCCL communicator (one process per GPU).  Rank 0 calls
 * hlm_b200_comm_unique_id and ships the 128 bytes to the other ranks by any means (bench.py:
 * torch.distributed broadcast); every rank then calls hlm_b200_comm_create.  libnccl.so.2 is bound
 * at run time (the copy already loaded in the process, if any). */
#define HLM_B200_UNIQUE_ID_BYTES 128
typedef struct hlm_b200_comm hlm_b200_comm;
int hlm_b200_comm_unique_id(uint8_t* id /* HLM_B200_UNIQUE_ID_BYTES */);
int hlm_b200_comm_create(const uint8_t* id, int rank, int nranks, int device, hlm_b200_comm** out);
int hlm_b200_comm_info(const hlm_b200_comm* comm, int* rank, int* nranks, int* device, int* nccl_version);
void hlm_b200_comm_destroy(hlm_b200_comm* comm);

typedef struct {
  uint32_t rounds;
  uint32_t num_local_shards;
  uint32_t num_processes;
  uint32_t tie_redo_rounds;  /* rounds resolved by the three-level comparator across ranks */
  uint32_t host_syncs;       /* stream synchronisations inside the round loop: rounds + tie_redo_rounds */
  uint32_t kernel_launches;
  uint32_t nccl_calls;
  uint64_t num_edges_global;
  uint64_t collective_bytes;             /* payload handed to the collectives by one rank, all rounds */
  uint64_t* collective_bytes_per_round;  /* rounds entries: shrinks with the live-vertex set */
  uint32_t* live_vertices_per_round;     /* rounds entries: vertices whose maxima were exchanged */
} hlm_b200_shard_report;

/* run_variant (local_max_par.hpp:586) over the shards `shards[0 .. num_shards)` of this process (ascending
 * edge-id ranges; shards on one device are co-located "virtual ranks") and, if `comm` is given, the shards
 * of the other processes.  results[i] receives shard i's slice (global edge ids, ascending) together with
 * the GLOBAL rounds, per-round counts and total_weight; concatenating the slices in rank order gives the
 * reference's matched_edges.  HLM_B200_TIES_EXACT in cfg resolves every round by the three-level comparator. */
int hlm_b200_match_sharded(hlm_b200_graph* const* shards, int num_shards, hlm_b200_comm* comm,
                           const hlm_b200_stream* stream, const hlm_b200_config* cfg, hlm_b200_result* results,
                           hlm_b200_shard_report* report);
void hlm_b200_shard_report_free(hlm_b200_shard_report* report);

/* ---- text formats (host only, no device needed) ------------------------------------------------
 * io.hpp of the reference: hMetis .hgr hypergraphs (parse_hgr :79, write_hgr :146), METIS graphs
 * as 2-uniform hypergraphs (parse_metis_graph :176), the matching file (write_matching :240,
 * parse_matching :249), on top of build_hypergraph (hypergraph.hpp:78-153).  Same inputs accepted
 * and rejected (HLM_B200_ERR_INPUT = hlm::input_error), same CSR and the same text out. */
typedef struct {          /* an hlm::Hypergraph owned by the library: all five arrays, malloc'ed */
  uint32_t num_vertices;
  uint32_t num_edges;
  uint64_t* vertex_offsets;
  uint32_t* vertex_incidence;
  uint64_t* edge_offsets;
  uint32_t* edge_members;
  double* base_weights;
  uint32_t num_warnings;  /* ParseOptions::warnings->size(): 1 if a vertex-weight block was skipped */
} hlm_b200_host_graph;

/* hlm::DegreeZeroPolicy (hypergraph.hpp:56-59) */
enum { HLM_B200_DEGREE_ZERO_REJECT = 0, HLM_B200_DEGREE_ZERO_DROP = 1 };

int hlm_b200_parse_hgr(const char* text, size_t len, int degree_zero, hlm_b200_host_graph* out);
int hlm_b200_parse_metis_graph(const char* text, size_t len, int degree_zero, hlm_b200_host_graph* out);
void hlm_b200_host_graph_free(hlm_b200_host_graph* g);
/* Instance generators of the reference (generators.hpp), host only, bit-identical output:
 * generate_random (:65-93; BASELINE config 1 = {1000000, 1000000, 4, 4, seed 1}), generate_tight_family
 * (:37-54) and random_weights_1_100 (:96-101; `out` holds num_edges doubles).  Release the graphs with
 * hlm_b200_host_graph_free.  Bad parameters are HLM_B200_ERR_INPUT with the reference's messages. */
int hlm_b200_generate_random(uint32_t num_vertices, uint32_t num_edges, uint32_t min_edge_size, uint32_t max_edge_size,
                             uint64_t seed, hlm_b200_host_graph* out);
int hlm_b200_generate_tight_family(uint32_t d, double epsilon, hlm_b200_host_graph* out);
int hlm_b200_random_weights_1_100(uint32_t num_edges, uint64_t seed, double* out);
/* *text is NUL-terminated, *len excludes the NUL; release with hlm_b200_text_free */
int hlm_b200_write_hgr(const hlm_b200_csr_view* h, char** text, size_t* len);
int hlm_b200_write_matching(const uint32_t* matched, uint64_t count, double total_weight, uint32_t rounds,
                            char** text, size_t* len);
int hlm_b200_parse_matching(const char* text, size_t len, uint32_t** ids, uint64_t* count);
void hlm_b200_text_free(void* p); /* texts and id arrays returned by the three calls above */

/* compact (local_max_par.hpp:350-454) on the device: both CSRs rebuilt over the active vertices and
 * edges (dense, order-preserving renumbering by exclusive scans over the flags); active vertices
 * left without an active edge are dropped.  *vertex_map / *edge_map: old id -> new id or 0xFFFFFFFF
 * (release with hlm_b200_text_free).  An active edge touching an inactive vertex is
 * HLM_B200_ERR_INPUT (the reference's input_error).  `work`, if given, receives what the reference
 * adds to its WorkCounters for one compaction (:446-453). */
typedef struct {
  uint64_t total_edge_visits;
  uint64_t total_pin_visits;
  uint32_t prefix_sum_invocations;
  uint32_t compactions;
} hlm_b200_compact_work;
int hlm_b200_compact(const hlm_b200_csr_view* h, const uint8_t* vertex_active, const uint8_t* edge_active, int device,
                     hlm_b200_host_graph* out, uint32_t** vertex_map, uint32_t** edge_map, hlm_b200_compact_work* work);

/* default_max_rounds (matching.hpp:87-89). */
uint32_t hlm_b200_default_max_rounds(uint32_t num_edges);

#ifdef __cplusplus
}
#endif
#endif /* HLM_B200_H */
