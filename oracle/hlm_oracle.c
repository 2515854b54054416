/*
 * hlm_oracle.c -- CPU restatement of the reference hot path in plain C.
 * TEST INFRASTRUCTURE ONLY (see hlm_oracle.h).  Parity status: PINNED
 * (known answers + reference-generated goldens + live oracle/_ref diffs).
 *
 * Build WITHOUT -march=native / -ffast-math and WITH -ffp-contract=off: the
 * reference is built with plain -O2 (proj/CMakeLists.txt:3-8), so its weight
 * expression rounds twice (no FMA) and the bit patterns depend on that.
 *
 * File:line citations are relative to /root/reference/proj/include/hlm/.
 */
#define _POSIX_C_SOURCE 200809L
#ifdef _OPENMP
#include <omp.h>
#endif
#include "hlm_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_INVALID 0xFFFFFFFFu

/* ------------------------------------------------------------------ */
/* priority stream                                                      */
/* ------------------------------------------------------------------ */

/* weight_stream.hpp:26-31 */
uint64_t orc_mix_splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* weight_stream.hpp:33-39 */
uint64_t orc_mix_xorshift(uint64_t x) {
  x *= 0x9E3779B97F4A7C15ull;
  x ^= x >> 12;
  x ^= x << 25;
  x ^= x >> 27;
  return x * 0x2545F4914F6CDD1Dull;
}

/* weight_stream.hpp:42-47 */
uint64_t orc_mix_park_miller(uint64_t x) {
  uint64_t s = x % 2147483646ull + 1ull;
  s = (s * 16807ull) % 2147483647ull;
  s = (s * 16807ull) % 2147483647ull;
  return s;
}

/* weight_stream.hpp:49-52 */
static double unit_from_bits(uint64_t bits) {
  return ((double)(bits >> 11) + 0.5) * 0x1.0p-53;
}

/* weight_stream.hpp:91-93 */
static uint64_t stream_counter(const orc_stream* s, uint32_t e, uint32_t round) {
  return s->seed ^ ((uint64_t)round << 40) ^ (uint64_t)e;
}

/* weight_stream.hpp:64-75 */
double orc_unit_noise(const orc_stream* s, uint32_t e, uint32_t round) {
  const uint64_t key = stream_counter(s, e, round);
  switch (s->kind) {
    case ORC_GEN_SPLITMIX:
      return unit_from_bits(orc_mix_splitmix(key));
    case ORC_GEN_XORSHIFT:
      return unit_from_bits(orc_mix_xorshift(key));
    case ORC_GEN_PARK_MILLER:
      return (double)orc_mix_park_miller(key) / 2147483647.0;
  }
  return 0.5;
}

/* weight_stream.hpp:78-83 */
double orc_weight(const orc_stream* s, uint32_t e, uint32_t round, double base) {
  if (s->mode == ORC_MODE_REPLACE_UNIFORM) return orc_unit_noise(s, e, round);
  const double width = s->noise_high - s->noise_low;
  if (width == 0.0) return base + s->noise_low;
  return base + s->noise_low + orc_unit_noise(s, e, round) * width;
}

/* weight_stream.hpp:86-88 */
uint64_t orc_tie_hash(const orc_stream* s, uint32_t e, uint32_t round) {
  return orc_mix_splitmix(stream_counter(s, e, round) ^ 0x6A09E667F3BCC909ull);
}

/* weight_stream.hpp:105-113; returns <0, 0, >0 */
int orc_tie_break(double wa, uint32_t ida, double wb, uint32_t idb, const orc_stream* s,
                  uint32_t round) {
  if (wa < wb) return -1;
  if (wa > wb) return 1;
  const uint64_t ha = orc_tie_hash(s, ida, round);
  const uint64_t hb = orc_tie_hash(s, idb, round);
  if (ha != hb) return ha < hb ? -1 : 1;
  return ida < idb ? -1 : (ida > idb ? 1 : 0);
}

/* weight_stream.hpp:96-100 */
int orc_check_noise_interval(const orc_stream* s) {
  if (s->noise_low < 0.0 || s->noise_high < s->noise_low) return ORC_INPUT_ERROR;
  return ORC_OK;
}

void orc_eval_stream(const orc_stream* s, const uint32_t* edges, const uint32_t* rounds,
                     const double* base, size_t count, double* w_out, uint64_t* t_out) {
  for (size_t i = 0; i < count; ++i) {
    if (w_out) w_out[i] = orc_weight(s, edges[i], rounds[i], base ? base[i] : 1.0);
    if (t_out) t_out[i] = orc_tie_hash(s, edges[i], rounds[i]);
  }
}

/* ------------------------------------------------------------------ */
/* matcher                                                              */
/* ------------------------------------------------------------------ */

/* common.hpp:27-35, matching.hpp:87-89 */
uint32_t orc_default_max_rounds(uint32_t m) {
  const uint64_t x = (uint64_t)m + 2;
  uint32_t r = 0;
  uint64_t p = 1;
  while (p < x) {
    p <<= 1;
    ++r;
  }
  return 64 + 4 * r;
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

void orc_free_result(orc_result* r) {
  if (!r) return;
  free(r->matched_edges);
  free(r->matched_round);
  free(r->per_round_matched);
  free(r->per_round_deactivated);
  memset(r, 0, sizeof(*r));
}

/*
 * local_max_seq.hpp:94-126 (driver) and :22-70 (one round, phases A-D).
 * Status bytes follow matching.hpp:50 (0 active, 1 matched, 2 inactive).
 * On ORC_ROUND_LIMIT the partial matching is still filled in
 * (local_max_seq.hpp:109-113).
 */
int orc_local_max(const orc_graph* g, const orc_stream* s, uint32_t max_rounds, orc_result* out) {
  memset(out, 0, sizeof(*out));
  if (orc_check_noise_interval(s) != ORC_OK) return ORC_INPUT_ERROR;
  const uint32_t n = g->n, m = g->m;
  const uint64_t kappa = m ? g->edge_offsets[m] : 0;
  if (max_rounds == 0) max_rounds = orc_default_max_rounds(m);
  const double t0 = now_ms();

  uint32_t* top = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
  uint32_t* agree = (uint32_t*)calloc((size_t)m + 1, sizeof(uint32_t));
  uint8_t* status = (uint8_t*)calloc((size_t)m + 1, 1);
  uint8_t* vactive = (uint8_t*)malloc((size_t)n + 1);
  uint8_t* newly = (uint8_t*)calloc((size_t)n + 1, 1);
  double* w = (double*)calloc((size_t)m + 1, sizeof(double));
  uint32_t* mround = (uint32_t*)calloc((size_t)m + 1, sizeof(uint32_t));
  uint32_t cap = 16;
  uint32_t* prm = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  uint32_t* prd = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  if (!top || !agree || !status || !vactive || !newly || !w || !mround || !prm || !prd)
    return ORC_NOMEM;
  memset(vactive, 1, (size_t)n + 1);

  uint32_t active_edges = m;
  uint32_t round = 0;
  uint64_t total_matched = 0;
  int rc = ORC_OK;

  while (active_edges > 0) {
    ++round;
    if (round > max_rounds) {
      rc = ORC_ROUND_LIMIT;
      --round;
      break;
    }
    /* weight_stream.hpp:117-123 */
    for (uint32_t e = 0; e < m; ++e)
      if (status[e] == 0) w[e] = orc_weight(s, e, round, g->base_weights[e]);
    out->edge_visits += m;

    /* phase A, local_max_seq.hpp:28-38 */
    for (uint32_t v = 0; v < n; ++v) {
      if (!vactive[v]) continue;
      uint32_t best = ORC_INVALID;
      for (uint64_t i = g->vertex_offsets[v]; i < g->vertex_offsets[v + 1]; ++i) {
        const uint32_t e = g->vertex_incidence[i];
        if (status[e] != 0) continue;
        if (best == ORC_INVALID || orc_tie_break(w[e], e, w[best], best, s, round) > 0) best = e;
      }
      top[v] = best;
    }
    /* phase B, :40-42 */
    memset(agree, 0, sizeof(uint32_t) * (size_t)m);
    for (uint32_t v = 0; v < n; ++v)
      if (vactive[v] && top[v] != ORC_INVALID) ++agree[top[v]];
    /* phase C, :44-50 */
    uint32_t matched_now = 0;
    for (uint32_t e = 0; e < m; ++e) {
      if (status[e] != 0) continue;
      const uint64_t b = g->edge_offsets[e], en = g->edge_offsets[e + 1];
      if (agree[e] != (uint32_t)(en - b)) continue;
      status[e] = 1;
      mround[e] = round;
      ++matched_now;
      for (uint64_t i = b; i < en; ++i) newly[g->edge_members[i]] = 1;
    }
    /* phase D, :52-62 */
    uint32_t deactivated = 0;
    for (uint32_t v = 0; v < n; ++v) {
      if (!vactive[v] || !newly[v]) continue;
      for (uint64_t i = g->vertex_offsets[v]; i < g->vertex_offsets[v + 1]; ++i) {
        const uint32_t e = g->vertex_incidence[i];
        if (status[e] == 0) {
          status[e] = 2;
          ++deactivated;
        }
      }
      vactive[v] = 0;
      newly[v] = 0;
    }
    /* :64-68 */
    out->pin_visits += 3 * kappa;
    out->edge_visits += 2 * (uint64_t)m;

    active_edges -= matched_now + deactivated;
    total_matched += matched_now;
    if (round > cap) {
      cap *= 2;
      prm = (uint32_t*)realloc(prm, sizeof(uint32_t) * cap);
      prd = (uint32_t*)realloc(prd, sizeof(uint32_t) * cap);
      if (!prm || !prd) return ORC_NOMEM;
    }
    prm[round - 1] = matched_now;
    prd[round - 1] = deactivated;
  }

  /* finish_matching, local_max_seq.hpp:74-83: ascending ids, weight summed in id order */
  out->rounds = round;
  out->num_matched = total_matched;
  out->matched_edges = (uint32_t*)malloc(sizeof(uint32_t) * (total_matched + 1));
  out->matched_round = (uint32_t*)malloc(sizeof(uint32_t) * (total_matched + 1));
  uint64_t k = 0;
  double total = 0.0;
  for (uint32_t e = 0; e < m; ++e)
    if (status[e] == 1) {
      out->matched_edges[k] = e;
      out->matched_round[k] = mround[e];
      total += g->base_weights[e];
      ++k;
    }
  out->total_weight = total;
  out->per_round_matched = prm;
  out->per_round_deactivated = prd;
  out->wall_ms = now_ms() - t0;

  free(top);
  free(agree);
  free(status);
  free(vactive);
  free(newly);
  free(w);
  free(mround);
  return rc;
}

/* exact.hpp:115-140 */
int orc_verify_matching(const orc_graph* g, const uint32_t* matched, uint64_t count,
                        int* disjoint, int* maximal, double* weight) {
  for (uint64_t i = 0; i < count; ++i)
    if (matched[i] >= g->m) return ORC_INPUT_ERROR;
  uint8_t* covered = (uint8_t*)calloc((size_t)g->n + 1, 1);
  uint8_t* inm = (uint8_t*)calloc((size_t)g->m + 1, 1);
  if (!covered || !inm) return ORC_NOMEM;
  int dis = 1, mx = 1;
  double wsum = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t e = matched[i];
    for (uint64_t p = g->edge_offsets[e]; p < g->edge_offsets[e + 1]; ++p) {
      const uint32_t v = g->edge_members[p];
      if (covered[v]) dis = 0;
      covered[v] = 1;
    }
    wsum += g->base_weights[e];
    inm[e] = 1;
  }
  for (uint32_t e = 0; e < g->m && mx; ++e) {
    if (inm[e]) continue;
    int any = 0;
    for (uint64_t p = g->edge_offsets[e]; p < g->edge_offsets[e + 1]; ++p)
      any |= covered[g->edge_members[p]];
    if (!any) mx = 0;
  }
  free(covered);
  free(inm);
  *disjoint = dis;
  *maximal = mx;
  *weight = wsum;
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* instance sources                                                     */
/* ------------------------------------------------------------------ */

void orc_free_graph(orc_owned_graph* g) {
  if (!g) return;
  free(g->vertex_offsets);
  free(g->vertex_incidence);
  free(g->edge_offsets);
  free(g->edge_members);
  free(g->base_weights);
  memset(g, 0, sizeof(*g));
}

/* hypergraph.hpp:144-151: counting sort of pins by vertex; incidence lists come out
 * in ascending edge order. */
int orc_build_incidence(uint32_t n, uint32_t m, const uint64_t* edge_offsets,
                        const uint32_t* edge_members, uint64_t* vertex_offsets,
                        uint32_t* vertex_incidence) {
  const uint64_t kappa = m ? edge_offsets[m] : 0;
  memset(vertex_offsets, 0, sizeof(uint64_t) * ((size_t)n + 1));
  /* Large instances (the full BASELINE configs for bench.py's reference arm): every thread owns a
   * range of vertices and walks all pins, so counters and cursors are private to their owner and a
   * list is filled in ascending edge order, exactly like the sequential form below. */
  int bad = 0;
#ifdef _OPENMP
  if (kappa >= (1ull << 22)) {
#pragma omp parallel
    {
      const uint32_t nt = (uint32_t)omp_get_num_threads(), t = (uint32_t)omp_get_thread_num();
      const uint32_t lo = (uint32_t)((uint64_t)n * t / nt), hi = (uint32_t)((uint64_t)n * (t + 1) / nt);
      for (uint64_t i = 0; i < kappa; ++i) {
        const uint32_t v = edge_members[i];
        if (v >= n) {
          if (t == 0) bad = 1;
        } else if (v >= lo && v < hi) {
          ++vertex_offsets[v + 1];
        }
      }
    }
    if (bad) return ORC_INPUT_ERROR;
    for (uint32_t v = 0; v < n; ++v) vertex_offsets[v + 1] += vertex_offsets[v];
    uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    if (!cur) return ORC_NOMEM;
    memcpy(cur, vertex_offsets, sizeof(uint64_t) * (size_t)n);
#pragma omp parallel
    {
      const uint32_t nt = (uint32_t)omp_get_num_threads(), t = (uint32_t)omp_get_thread_num();
      const uint32_t lo = (uint32_t)((uint64_t)n * t / nt), hi = (uint32_t)((uint64_t)n * (t + 1) / nt);
      for (uint32_t e = 0; e < m; ++e)
        for (uint64_t i = edge_offsets[e]; i < edge_offsets[e + 1]; ++i) {
          const uint32_t v = edge_members[i];
          if (v >= lo && v < hi) vertex_incidence[cur[v]++] = e;
        }
    }
    free(cur);
    return ORC_OK;
  }
#endif
  for (uint64_t i = 0; i < kappa; ++i) {
    if (edge_members[i] >= n) return ORC_INPUT_ERROR;
    ++vertex_offsets[edge_members[i] + 1];
  }
  for (uint32_t v = 0; v < n; ++v) vertex_offsets[v + 1] += vertex_offsets[v];
  uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  if (!cursor) return ORC_NOMEM;
  memcpy(cursor, vertex_offsets, sizeof(uint64_t) * (size_t)n);
  for (uint32_t e = 0; e < m; ++e)
    for (uint64_t i = edge_offsets[e]; i < edge_offsets[e + 1]; ++i)
      vertex_incidence[cursor[edge_members[i]]++] = e;
  free(cursor);
  return ORC_OK;
}

/* generators.hpp:19-30 */
typedef struct {
  uint64_t state;
} seq_rng;
static uint64_t seq_next(seq_rng* r) {
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static int alloc_graph(orc_owned_graph* g, uint32_t n, uint32_t m, uint64_t kappa) {
  memset(g, 0, sizeof(*g));
  g->n = n;
  g->m = m;
  g->kappa = kappa;
  g->vertex_offsets = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  g->vertex_incidence = (uint32_t*)malloc(sizeof(uint32_t) * (kappa + 1));
  g->edge_offsets = (uint64_t*)calloc((size_t)m + 1, sizeof(uint64_t));
  g->edge_members = (uint32_t*)malloc(sizeof(uint32_t) * (kappa + 1));
  g->base_weights = (double*)malloc(sizeof(double) * ((size_t)m + 1));
  if (!g->vertex_offsets || !g->vertex_incidence || !g->edge_offsets || !g->edge_members ||
      !g->base_weights) {
    orc_free_graph(g);
    return ORC_NOMEM;
  }
  return ORC_OK;
}

/*
 * generators.hpp:65-93 followed by build_hypergraph with drop_and_renumber
 * (hypergraph.hpp:78-153): one size draw per edge (consumed even when the span
 * is 1), then vertex draws until `size` distinct ones are collected; unused
 * vertices are dropped and the rest renumbered densely; unit weights.
 */
int orc_generate_random(uint32_t num_vertices, uint32_t num_edges, uint32_t min_size,
                        uint32_t max_size, uint64_t seed, orc_owned_graph* out) {
  memset(out, 0, sizeof(*out));
  if (num_vertices == 0 || num_edges == 0) return ORC_INPUT_ERROR;
  if (min_size == 0 || min_size > max_size) return ORC_INPUT_ERROR;
  if (max_size > num_vertices) return ORC_INPUT_ERROR;

  seq_rng rng = {seed};
  const uint32_t span = max_size - min_size + 1;
  uint64_t* eoff = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)num_edges + 1));
  uint32_t* raw = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)num_edges * max_size);
  uint32_t* degree = (uint32_t*)calloc(num_vertices, sizeof(uint32_t));
  if (!eoff || !raw || !degree) return ORC_NOMEM;
  uint64_t pos = 0;
  for (uint32_t e = 0; e < num_edges; ++e) {
    const uint32_t size = min_size + (uint32_t)(seq_next(&rng) % span);
    eoff[e] = pos;
    uint32_t have = 0;
    while (have < size) {
      const uint32_t v = (uint32_t)(seq_next(&rng) % num_vertices);
      int seen = 0;
      for (uint32_t i = 0; i < have; ++i) seen |= (raw[pos + i] == v);
      if (!seen) raw[pos + have++] = v;
    }
    for (uint32_t i = 0; i < size; ++i) ++degree[raw[pos + i]];
    pos += size;
  }
  eoff[num_edges] = pos;

  uint32_t kept = 0;
  uint32_t* remap = (uint32_t*)malloc(sizeof(uint32_t) * num_vertices);
  if (!remap) return ORC_NOMEM;
  for (uint32_t v = 0; v < num_vertices; ++v) remap[v] = degree[v] ? kept++ : ORC_INVALID;

  int rc = alloc_graph(out, kept, num_edges, pos);
  if (rc != ORC_OK) return rc;
  memcpy(out->edge_offsets, eoff, sizeof(uint64_t) * ((size_t)num_edges + 1));
  for (uint64_t i = 0; i < pos; ++i) out->edge_members[i] = remap[raw[i]];
  for (uint32_t e = 0; e < num_edges; ++e) out->base_weights[e] = 1.0;
  rc = orc_build_incidence(kept, num_edges, out->edge_offsets, out->edge_members,
                           out->vertex_offsets, out->vertex_incidence);
  free(eoff);
  free(raw);
  free(degree);
  free(remap);
  return rc;
}

/* generators.hpp:96-101 */
void orc_random_weights_1_100(uint32_t m, uint64_t seed, double* out) {
  seq_rng rng = {seed ^ 0x517CC1B727220A95ull};
  for (uint32_t e = 0; e < m; ++e) out[e] = (double)(1 + seq_next(&rng) % 100);
}

/* generators.hpp:37-52: d pair edges {i, d+i} of weight 1, then one rank-d edge
 * {0..d-1} of weight 1+epsilon. */
int orc_tight_family(uint32_t d, double epsilon, orc_owned_graph* out) {
  memset(out, 0, sizeof(*out));
  if (d < 2 || !(epsilon > 0.0)) return ORC_INPUT_ERROR;
  int rc = alloc_graph(out, 2 * d, d + 1, 3 * (uint64_t)d);
  if (rc != ORC_OK) return rc;
  uint64_t pos = 0;
  for (uint32_t i = 0; i < d; ++i) {
    out->edge_offsets[i] = pos;
    out->edge_members[pos++] = i;
    out->edge_members[pos++] = d + i;
    out->base_weights[i] = 1.0;
  }
  out->edge_offsets[d] = pos;
  for (uint32_t i = 0; i < d; ++i) out->edge_members[pos++] = i;
  out->edge_offsets[d + 1] = pos;
  out->base_weights[d] = 1.0 + epsilon;
  return orc_build_incidence(2 * d, d + 1, out->edge_offsets, out->edge_members,
                             out->vertex_offsets, out->vertex_incidence);
}

uint64_t orc_fnv1a_ids(const uint32_t* ids, uint64_t count) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t x = ids[i];
    for (int b = 0; b < 4; ++b) {
      h ^= (uint64_t)((x >> (8 * b)) & 0xFFu);
      h *= 1099511628211ull;
    }
  }
  return h;
}

/* ------------------------------------------------------------------ */
/* synthetic bench instances (this repo's definitions)       */
/* ------------------------------------------------------------------ */

static uint64_t syn_hash(uint64_t seed, uint64_t tag, uint64_t e, uint64_t k) {
  return orc_mix_splitmix(orc_mix_splitmix(orc_mix_splitmix(seed + tag) + e) + k);
}

static uint64_t mulhi64(uint64_t a, uint64_t b) {
  return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
}

enum { SYN_TAG_SIZE = 1, SYN_TAG_PIN = 2, SYN_TAG_WEIGHT = 3 };

double orc_syn_weight(const orc_syn_spec* spec, uint32_t e) {
  if (!spec->int_weights) return 1.0;
  return (double)(1 + syn_hash(spec->seed, SYN_TAG_WEIGHT, e, 0) % 100);
}

uint32_t orc_syn_edge_size(const orc_syn_spec* spec, uint32_t e) {
  switch (spec->family) {
    case ORC_SYN_UNIFORM:
      return spec->d;
    case ORC_SYN_RMAT:
      return 2;
    case ORC_SYN_POWERLAW: {
      /* P(s) proportional to floor(2^40 / s^2), s in [2, 64] */
      uint64_t total = 0;
      for (uint64_t s = 2; s <= 64; ++s) total += (1ull << 40) / (s * s);
      uint64_t x = syn_hash(spec->seed, SYN_TAG_SIZE, e, 0) % total;
      for (uint64_t s = 2; s <= 64; ++s) {
        const uint64_t w = (1ull << 40) / (s * s);
        if (x < w) return (uint32_t)s;
        x -= w;
      }
      return 64;
    }
    case ORC_SYN_NETLIST: {
      const uint64_t c = syn_hash(spec->seed, SYN_TAG_SIZE, e, 0);
      if (c % 1000 == 0) {
        /* one edge in a thousand is a large net: uniform inside a random octave of [64, 4096] */
        const uint32_t o = (uint32_t)((c >> 10) % 6);
        const uint32_t f = (uint32_t)((c >> 16) % (64u << o));
        uint32_t s = (64u << o) + f + 1;
        if (s > spec->n) s = spec->n;
        return s;
      }
      /* 2 + geometric (P(K >= k) = 0.6^k by integer recurrence), capped at 32 */
      const uint64_t g = (c >> 10) & 0xFFFFFFFFull;
      uint64_t q = 1ull << 32;
      uint32_t k = 0;
      while (k < 30) {
        q = q * 3 / 5;
        if (g >= q) break;
        ++k;
      }
      uint32_t s = 2 + k;
      if (s > spec->n) s = spec->n;
      return s;
    }
  }
  return 0;
}

static uint32_t syn_draw_vertex(const orc_syn_spec* spec, uint32_t e, uint32_t j, uint32_t a) {
  const uint64_t h = syn_hash(spec->seed, SYN_TAG_PIN, e, ((uint64_t)j << 32) | a);
  if (spec->family == ORC_SYN_POWERLAW) {
    /* v = floor(n * u^3) in 32.32 fixed point: density proportional to v^(-2/3) */
    const uint64_t u = h >> 32;
    const uint64_t t1 = (u * u) >> 32;
    const uint64_t t2 = (t1 * u) >> 32;
    return (uint32_t)((t2 * (uint64_t)spec->n) >> 32);
  }
  return (uint32_t)mulhi64(h, spec->n);
}

void orc_syn_edge_pins(const orc_syn_spec* spec, uint32_t e, uint32_t size, uint32_t* pins) {
  if (spec->family == ORC_SYN_RMAT) {
    /* (a,b,c,d) = (0.57,0.19,0.19,0.05) on 16-bit draws: 37356 / 49807 / 62259 */
    for (uint32_t a = 0;; ++a) {
      uint32_t u = 0, v = 0;
      for (uint32_t lvl = 0; lvl < spec->scale; ++lvl) {
        const uint64_t h = syn_hash(spec->seed, SYN_TAG_PIN, e, ((uint64_t)a << 32) | (lvl >> 2));
        const uint32_t r = (uint32_t)((h >> (16 * (lvl & 3))) & 0xFFFFu);
        const uint32_t bu = r >= 49807u;
        const uint32_t bv = (r >= 37356u && r < 49807u) || r >= 62259u;
        u = (u << 1) | bu;
        v = (v << 1) | bv;
      }
      if (u != v) {
        pins[0] = u;
        pins[1] = v;
        return;
      }
    }
  }
  for (uint32_t j = 0; j < size; ++j) {
    for (uint32_t a = 0;; ++a) {
      const uint32_t v = syn_draw_vertex(spec, e, j, a);
      int seen = 0;
      for (uint32_t i = 0; i < j; ++i) seen |= (pins[i] == v);
      if (!seen) {
        pins[j] = v;
        break;
      }
    }
  }
}

int orc_syn_generate(const orc_syn_spec* spec, orc_owned_graph* out) {
  memset(out, 0, sizeof(*out));
  const uint32_t n = spec->family == ORC_SYN_RMAT ? (1u << spec->scale) : spec->n;
  if (n < 2 || spec->m == 0) return ORC_INPUT_ERROR;
  if (spec->family == ORC_SYN_UNIFORM && (spec->d == 0 || spec->d > n)) return ORC_INPUT_ERROR;
  orc_syn_spec sp = *spec;
  sp.n = n;
  /* counter-based: every edge is a pure function of (seed, e), so the rows are filled in parallel
   * (OpenMP; the full BASELINE configs are generated on the host for the reference arm of bench.py) */
  uint32_t* sizes = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)sp.m);
  if (!sizes) return ORC_NOMEM;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < (int64_t)sp.m; ++e) sizes[e] = orc_syn_edge_size(&sp, (uint32_t)e);
  uint64_t kappa = 0;
  for (uint32_t e = 0; e < sp.m; ++e) kappa += sizes[e];
  int rc = alloc_graph(out, n, sp.m, kappa);
  if (rc != ORC_OK) {
    free(sizes);
    return rc;
  }
  uint64_t pos = 0;
  for (uint32_t e = 0; e < sp.m; ++e) {
    out->edge_offsets[e] = pos;
    pos += sizes[e];
  }
  out->edge_offsets[sp.m] = pos;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t e = 0; e < (int64_t)sp.m; ++e) {
    orc_syn_edge_pins(&sp, (uint32_t)e, sizes[e], out->edge_members + out->edge_offsets[e]);
    out->base_weights[e] = orc_syn_weight(&sp, (uint32_t)e);
  }
  free(sizes);
  return orc_build_incidence(n, sp.m, out->edge_offsets, out->edge_members, out->vertex_offsets,
                             out->vertex_incidence);
}
