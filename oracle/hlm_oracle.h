/*
 * hlm_oracle.h -- CPU restatement (plain C) of the reference's local-max
 * hypergraph matching path.
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, bench.py's
 * cpu_baseline / --impl reference legs and __graft_entry__.smoke() may load
 * it.  The product path (paper_2602_22976_b200/) never links, imports or
 * calls anything in oracle/.
 *
 * Parity status: PINNED.  tests/test_oracle_*.py check this restatement
 * against (a) the literal known answers in the reference's own tests
 * (proj/tests/test_seq.cpp:7-65, test_par.cpp:20-30), (b) golden vectors
 * produced by the unmodified reference compiled in this container
 * (oracle/_ref, recipe in oracle/Makefile; fixtures in tests/golden/), and
 * (c) live differential runs against oracle/_ref when that library exists.
 *
 * Every function cites the reference file:line (relative to
 * /root/reference/proj/include/hlm/) whose behaviour it restates.
 */
#ifndef HLM_ORACLE_H
#define HLM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* weight_stream.hpp:17-22 -- enum orders are the reference's. */
enum { ORC_GEN_XORSHIFT = 0, ORC_GEN_PARK_MILLER = 1, ORC_GEN_SPLITMIX = 2 };
enum { ORC_MODE_PERTURB_BASE = 0, ORC_MODE_REPLACE_UNIFORM = 1 };

/* weight_stream.hpp:56-61 */
typedef struct {
  uint64_t seed;
  int32_t kind;
  int32_t mode;
  double noise_low;
  double noise_high;
} orc_stream;

/* hypergraph.hpp:19-27 (borrowed arrays) */
typedef struct {
  uint32_t n;
  uint32_t m;
  const uint64_t* vertex_offsets;   /* n+1 */
  const uint32_t* vertex_incidence; /* kappa */
  const uint64_t* edge_offsets;     /* m+1 */
  const uint32_t* edge_members;     /* kappa */
  const double* base_weights;       /* m */
} orc_graph;

/* an owned instance, as produced by the generators below */
typedef struct {
  uint32_t n;
  uint32_t m;
  uint64_t kappa;
  uint64_t* vertex_offsets;
  uint32_t* vertex_incidence;
  uint64_t* edge_offsets;
  uint32_t* edge_members;
  double* base_weights;
} orc_owned_graph;

/* matching.hpp:15-48 flattened */
typedef struct {
  uint32_t* matched_edges;        /* ascending original ids */
  uint32_t* matched_round;        /* 1-based round each of them matched in */
  uint64_t num_matched;
  double total_weight;
  uint32_t rounds;
  uint32_t* per_round_matched;    /* rounds entries */
  uint32_t* per_round_deactivated;
  uint64_t edge_visits;
  uint64_t pin_visits;
  double wall_ms;
} orc_result;

enum { ORC_OK = 0, ORC_INPUT_ERROR = 1, ORC_ROUND_LIMIT = 2, ORC_NOMEM = 3 };

/* ---- priority stream (weight_stream.hpp) ---- */
uint64_t orc_mix_splitmix(uint64_t x);
uint64_t orc_mix_xorshift(uint64_t x);
uint64_t orc_mix_park_miller(uint64_t x);
double orc_unit_noise(const orc_stream* s, uint32_t e, uint32_t round);
double orc_weight(const orc_stream* s, uint32_t e, uint32_t round, double base);
uint64_t orc_tie_hash(const orc_stream* s, uint32_t e, uint32_t round);
int orc_tie_break(double wa, uint32_t ida, double wb, uint32_t idb, const orc_stream* s,
                  uint32_t round);
int orc_check_noise_interval(const orc_stream* s);
void orc_eval_stream(const orc_stream* s, const uint32_t* edges, const uint32_t* rounds,
                     const double* base, size_t count, double* w_out, uint64_t* t_out);

/* ---- matcher (local_max_seq.hpp) ---- */
uint32_t orc_default_max_rounds(uint32_t m);
int orc_local_max(const orc_graph* g, const orc_stream* s, uint32_t max_rounds, orc_result* out);
void orc_free_result(orc_result* r);

/* ---- verification (exact.hpp:115-140) ---- */
int orc_verify_matching(const orc_graph* g, const uint32_t* matched, uint64_t count,
                        int* disjoint, int* maximal, double* weight);

/* ---- instance sources (generators.hpp, hypergraph.hpp) ---- */
int orc_build_incidence(uint32_t n, uint32_t m, const uint64_t* edge_offsets,
                        const uint32_t* edge_members, uint64_t* vertex_offsets,
                        uint32_t* vertex_incidence);
int orc_generate_random(uint32_t num_vertices, uint32_t num_edges, uint32_t min_size,
                        uint32_t max_size, uint64_t seed, orc_owned_graph* out);
void orc_random_weights_1_100(uint32_t m, uint64_t seed, double* out);
int orc_tight_family(uint32_t d, double epsilon, orc_owned_graph* out);
void orc_free_graph(orc_owned_graph* g);

/* FNV-1a-64 over the little-endian bytes of each id */
uint64_t orc_fnv1a_ids(const uint32_t* ids, uint64_t count);

/* ---- synthetic bench instances (this repo's own counter-based definitions,
 *      DESIGN.md section "Synthetic instances"; no reference counterpart) ---- */
enum { ORC_SYN_UNIFORM = 0, ORC_SYN_RMAT = 1, ORC_SYN_POWERLAW = 2, ORC_SYN_NETLIST = 3 };
typedef struct {
  int32_t family;
  uint32_t n;        /* vertices (RMAT: 1 << scale) */
  uint32_t m;        /* edges */
  uint32_t d;        /* UNIFORM: edge size */
  uint32_t scale;    /* RMAT */
  uint64_t seed;
  int32_t int_weights; /* 0: unit weights, 1: integers 1..100 from a hash of (seed, e) */
} orc_syn_spec;
int orc_syn_generate(const orc_syn_spec* spec, orc_owned_graph* out);
uint32_t orc_syn_edge_size(const orc_syn_spec* spec, uint32_t e);
void orc_syn_edge_pins(const orc_syn_spec* spec, uint32_t e, uint32_t size, uint32_t* pins);
double orc_syn_weight(const orc_syn_spec* spec, uint32_t e);

#ifdef __cplusplus
}
#endif
#endif
