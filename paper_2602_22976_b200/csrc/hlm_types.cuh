// hlm_types.cuh -- device-side types and helpers shared by the translation units of
// libhlm_b200.so.  Reference semantics: local_max_par.hpp:93-253 (run_soft_delete +
// local_max_crcw) and local_max_seq.hpp:22-90; DESIGN.md maps reference phases onto kernels.
//
// Round r on the device (one iteration of the CUDA-graph WHILE body):
//   k_filter_vmax  -- for every edge that was active in round r-1: drop it if it matched, drop it
//                     (counted as deactivated) if one of its pins died, otherwise keep it in the
//                     round-r active list and atomicMax its round-tagged key into vkey[pin].
//                     (reference: deactivation :229-248, collect :163, weight refresh :126-135,
//                     vertex argmax :137-159 -- fused into one pass over the pins)
//   k_check_commit -- an active edge is matched iff its key is the maximum at every pin
//                     (== agreement count == |e|, :202-224); matched edges record their round
//                     and set the dead bit of their pins (completion marking :221).
//   k_advance      -- one thread: round bookkeeping, termination, round cap, tie / epoch exits.
// All of it is memory-bound integer work: no tensor cores.
//
// Active lists (class 0 = edges with <= 32 pins, one thread per edge) are SEGMENTED: the edge-id
// space is cut into nseg regions of seg_cap ids; a CTA claims a region by ticket, filters it and
// writes the survivors back into the same region of the other buffer.  No global scan, no
// contended append counter, and the lists stay in ascending-id order (deterministic content,
// monotone pin addresses).  Class 1 (larger edges, one warp per edge) keeps a state byte per edge.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hlm_priority.cuh"

namespace hlmb {

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;
constexpr uint32_t kLargeEdge = 32;  // edges with more pins are handled warp-per-edge

enum LoopStatus : uint32_t {
  ST_RUNNING = 0,
  ST_DONE = 1,
  ST_ROUND_LIMIT = 2,
  ST_TIE = 3,    // a vertex saw two equal keys: redo this round on the exact path
  ST_EPOCH = 4,  // round tags wrapped: vkey must be cleared before continuing
  ST_HANDOVER = 5,  // vertex-owned engine: few edges are left, the CRCW kernels finish the run
};

// Device-resident loop state.
struct Ctrl {
  uint32_t round;        // round being processed (1-based)
  uint32_t parity;       // list buffer holding the previous round's active lists
  uint32_t ticket_f;     // region tickets of the filter kernel
  uint32_t ticket_c;     // region tickets of the check kernel
  uint32_t active_small; // class-0 edges active in this round (sum of region counts)
  uint32_t count1[2];    // [buffer] active class-1 (large) edges
  uint32_t tie_flag;
  uint32_t status;
  uint32_t max_rounds;
  uint32_t rounds_done;
  uint32_t active_prev;  // class-0 edges in the list the next sweep reads (0 before round 2)
  uint32_t blocks_done;  // fused kernel: CTAs that finished this round's check
  uint32_t pad0;
  unsigned long long edges_swept;  // sum over rounds of the active-list lengths (sum of m_r)
  unsigned long long pins_swept;   // sum over rounds of the pins of the active edges (sum of kappa_r)
  unsigned long long pins_round;   // ragged instances: pins of the edges kept by this round's sweeps
  unsigned long long pins_matched; // ragged instances: pins of all matched edges so far
};

// One-launch matching of a small instance (k_rounds_fused): what the kernel leaves in page-locked host
// memory for the caller -- nothing else crosses the bus, and nothing is read back before the one final sync.
constexpr uint32_t kFusedRounds = 254;
struct FusedSummary {
  Ctrl ctrl;                 // the final control block
  unsigned long long total;  // matched edges
  unsigned long long isum;   // sum of their (integer) base weights, when asked for
  uint32_t assembled;        // 1: ids / rounds / per-round counts below are in place
  uint32_t pad;
  uint32_t matched[kFusedRounds + 2];  // [r] edges matched in round r
  uint32_t dropped[kFusedRounds + 2];  // [r] edges dropped from the list after round r
  unsigned long long trace[64];        // -DHLM_FUSED_TRACE: globaltimer of block 0 at every phase boundary
};

struct FusedExtra {
  Ctrl c0;                 // init: the control block of a fresh run
  uint32_t init;           // zero the per-call state (filter words, keys, bitmaps, counters) first
  uint32_t rounds_cap;     // entries of matched_cnt / deact_cnt
  uint32_t mbits_words;
  uint32_t out_cap;        // entries of out_ids / out_round
  uint32_t* block_cnt;     // [grid] scratch of the assembly phase
  unsigned long long* block_isum;  // [grid]
  uint32_t* dev_ids;       // [out_cap + 4] device staging of the result (the bus wants full-line writes)
  uint16_t* dev_round;     // [out_cap + 8]
  uint32_t* out_ids;       // page-locked host memory, same sizes (or null together with sum)
  uint16_t* out_round;     // may be null
  const double* base_int;  // non-null: integer base weights (caller-id indexed), summed on the device
  FusedSummary* sum;       // page-locked host memory; null: rounds only, no assembly
};

struct EdgeCsr {
  const uint32_t* pins;
  const uint32_t* off32;  // m+1 or null
  const uint64_t* off64;  // m+1 or null
  uint32_t uniform_d;     // >0: every edge has exactly this many pins, offsets implicit
  __device__ __forceinline__ void range(uint32_t e, uint64_t& begin, uint32_t& size) const {
    if (uniform_d) {
      begin = static_cast<uint64_t>(e) * uniform_d;
      size = uniform_d;
    } else if (off32) {
      const uint32_t b = __ldg(off32 + e);
      begin = b;
      size = __ldg(off32 + e + 1) - b;
    } else {
      const uint64_t b = __ldg(off64 + e);
      begin = b;
      size = static_cast<uint32_t>(__ldg(off64 + e + 1) - b);
    }
  }
};

struct RoundParams {
  EdgeCsr csr;
  const double* base;  // null: every edge weighs base_const
  const uint8_t* base8;  // same weights, one byte each, when all are integers in 0..255: what the
                         // scattered reads of rounds >= 2 and of the check use (32 weights per sector
                         // instead of 4; the conversion back is exact)
  double base_const;
  uint32_t n;
  uint32_t m;
  uint32_t has_large;  // some edges have more than kLargeEdge pins
  uint32_t id_base;    // global id of local edge 0 (edge shards); priorities use global ids
  const uint32_t* orig;  // null, or: resident edge e is the caller's edge orig[e] (the loader
                         // sorted the edges by first pin so that pin-0 accesses are coalesced)
  StreamParams stream;
  KeyScheme ks;
  Ctrl* ctrl;
  unsigned long long* vkey;  // n round-tagged vertex maxima (full 64-bit keys)
  uint32_t* vtop;            // n: high word of vkey, or kTopDead; the L2-resident filter array
  uint32_t* dead;            // n bits: where completion marking sets its bits (multi-GPU: the exchange area)
  const uint32_t* dead_all;  // n bits: every vertex covered so far; stable during a sweep
  uint32_t greedy;           // exact levels compare (base weight, lower id): the static priority of
                             // greedy_sorted (local_max_seq.hpp:130-139) instead of the round's stream
  uint32_t hot_vtop;         // vertex ids below this keep their filter word in L1 (ld.ca); others ld.cg
  uint32_t hot_bits;         // same for the dead bitmap
  uint32_t dead_first;       // sweeps of rounds >= 2 test the bitmap (n/8 bytes, L2-resident) before
                             // they touch vtop
  uint32_t* mbits;           // m bits: edge matched
  uint16_t* mround;          // m: round an edge matched in (valid where its mbits bit is set)
  // class 0: segmented lists
  uint32_t* seg_ids[2];      // [buffer] nseg regions of seg_cap edge ids
  uint32_t* seg_cnt[2];      // [buffer][nseg] ids in use per region
  uint32_t nseg;
  uint32_t seg_cap;
  const uint32_t* bat_pin0;  // first pin of the first edge of every 32-edge batch, one entry more than
                             // batches (first-pin sorted uniform instances; null otherwise): the first
                             // pins of edges [32 a, 32 b) lie in [bat_pin0[a], bat_pin0[b]]
  uint32_t check_claim;      // regions a warp of the check kernel claims per ticket (1..8)
  uint32_t* cand_ids;        // class 0, same regions: edges that did not lose during vertex-max
  uint32_t* cand_cnt;        // [nseg]
  // class 1: the (static) list of large edges and a state byte per entry
  const uint32_t* large_ids;
  uint8_t* large_state;
  uint32_t num_large;
  uint32_t large_chunk;      // entries of the large list a warp scans per step (power of two, 1..32)
  uint32_t* matched_cnt;     // [round] edges matched in that round
  uint32_t* deact_cnt;       // [round] edges dropped after that round (matched + deactivated)
};

// vtop[v] mirrors the high 32 bits of vkey[v] (round tag + the leading payload bits).  It is half
// the size of vkey, so it stays L2-resident where vkey would spill to HBM as random 32-byte
// sectors, and almost every decision is made on it: an edge whose high word is below vtop[v]
// cannot be the maximum at v (no atomic needed), an edge whose high word differs from vtop[v]
// after the vertex-max pass lost at v (no 64-bit compare needed).  A vertex covered by a matched
// edge keeps kTopDead there for the rest of the run: larger than every key's high word (the
// all-ones tag is reserved), so atomicMax never disturbs it, and the same load that filters the
// atomics tells the filter kernel that the edge must be dropped.
constexpr uint32_t kTopDead = 0xFFFFFFFFu;

__device__ __forceinline__ bool vertex_dead(const uint32_t* dead, uint32_t v) {
  return (__ldg(dead + (v >> 5)) >> (v & 31)) & 1u;
}
// kTopDead if v was covered in an earlier round, else 0: a stand-in for vtop[v] that only answers
// the deactivation question (rounds >= 2 of instances whose vtop does not fit in L2)
__device__ __forceinline__ uint32_t dead_word(const uint32_t* dead_all, uint32_t v) {
  return vertex_dead(dead_all, v) ? 0xFFFFFFFFu : 0u;
}

// The id the reference knows an edge by: keys, tie hashes and results always use it.
__device__ __forceinline__ uint32_t edge_local_id(const RoundParams& P, uint32_t e) {
  return P.orig ? __ldg(P.orig + e) : e;
}
__device__ __forceinline__ uint32_t edge_gid(const RoundParams& P, uint32_t e) {
  return edge_local_id(P, e) + P.id_base;
}

// matched edges record their round and set their bit in the (caller-id indexed) matched bitmap
__device__ __forceinline__ void mark_matched(const RoundParams& P, uint32_t e, uint32_t r) {
  const uint32_t id = edge_local_id(P, e);
  P.mround[id] = static_cast<uint16_t>(r);
  atomicOr(P.mbits + (id >> 5), 1u << (id & 31));
}

// completion marking (local_max_par.hpp:221): matched edges are vertex-disjoint, so the key
// store is exclusive; the bitmap copy feeds verification and the multi-GPU dead-bit exchange.
__device__ __forceinline__ void mark_dead(const RoundParams& P, uint32_t v) {
  P.vtop[v] = kTopDead;
  atomicOr(P.dead + (v >> 5), 1u << (v & 31));
}

// Gathers of the per-vertex arrays by the sweeps.  Ids below the hot limits (the highest degrees
// after the loader's renumbering) go through L1 (ld.ca; a stale filter word is only ever too small,
// and dead bits never change during a sweep); all other ids bypass it (ld.cg) so that the random
// cold accesses cannot evict the hot window.  Without renumbering the limits are 0 / everything.
__device__ __forceinline__ uint32_t ld_top(const RoundParams& P, uint32_t v) {
  return v < P.hot_vtop ? __ldca(P.vtop + v) : __ldcg(P.vtop + v);
}
__device__ __forceinline__ bool is_dead(const RoundParams& P, uint32_t v) {
  const uint32_t* w = P.dead_all + (v >> 5);
  const uint32_t bits = v < P.hot_bits ? __ldca(w) : __ldcg(w);
  return (bits >> (v & 31)) & 1u;
}

// vkey[v] = max(vkey[v], key), vtop[v] = max(vtop[v], high word), filtered by `cur` = an earlier
// (possibly stale, never too large) read of vtop[v].  Returns true if another edge deposited the
// same 64-bit key: the returning atomicMax sees it, because an edge is only skipped when a
// strictly larger high word is already present.
__device__ __forceinline__ bool deposit_key(const RoundParams& P, uint32_t v, unsigned long long key,
                                            uint32_t cur) {
  const uint32_t hi = static_cast<uint32_t>(key >> 32);
  if (cur > hi) return false;
  const unsigned long long old = atomicMax(P.vkey + v, key);
  atomicMax(P.vtop + v, hi);
  return old == key;
}

__device__ __forceinline__ bool key_wins_at(const RoundParams& P, uint32_t v, unsigned long long key) {
  if (__ldcg(P.vtop + v) != static_cast<uint32_t>(key >> 32)) return false;
  return __ldcg(P.vkey + v) == key;
}

__device__ __forceinline__ double base_of(const RoundParams& P, uint32_t e) {
  return P.base8 ? static_cast<double>(__ldg(P.base8 + e)) : (P.base ? __ldg(P.base + e) : P.base_const);
}

template <int D>
struct PinVec {
  uint32_t v[D];
};

template <int D>
__device__ __forceinline__ PinVec<D> load_pins(const uint32_t* pins, uint32_t e);
template <>
__device__ __forceinline__ PinVec<2> load_pins<2>(const uint32_t* pins, uint32_t e) {
  const uint2 q = __ldg(reinterpret_cast<const uint2*>(pins) + e);
  return {{q.x, q.y}};
}
template <>
__device__ __forceinline__ PinVec<4> load_pins<4>(const uint32_t* pins, uint32_t e) {
  const uint4 q = __ldg(reinterpret_cast<const uint4*>(pins) + e);
  return {{q.x, q.y, q.z, q.w}};
}
template <>
__device__ __forceinline__ PinVec<8> load_pins<8>(const uint32_t* pins, uint32_t e) {
  const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(pins) + 2ull * e);
  const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(pins) + 2ull * e + 1);
  return {{q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w}};
}

// Streaming (evict-first) variants for data a sweep reads exactly once: the pin rows, the id
// lists, the caller ids and the base weights must not push the per-vertex arrays out of L2.
template <int D>
__device__ __forceinline__ PinVec<D> load_pins_stream(const uint32_t* pins, uint32_t e);
template <>
__device__ __forceinline__ PinVec<2> load_pins_stream<2>(const uint32_t* pins, uint32_t e) {
  const uint2 q = __ldcs(reinterpret_cast<const uint2*>(pins) + e);
  return {{q.x, q.y}};
}
template <>
__device__ __forceinline__ PinVec<4> load_pins_stream<4>(const uint32_t* pins, uint32_t e) {
  const uint4 q = __ldcs(reinterpret_cast<const uint4*>(pins) + e);
  return {{q.x, q.y, q.z, q.w}};
}
template <>
__device__ __forceinline__ PinVec<8> load_pins_stream<8>(const uint32_t* pins, uint32_t e) {
  const uint4 q0 = __ldcs(reinterpret_cast<const uint4*>(pins) + 2ull * e);
  const uint4 q1 = __ldcs(reinterpret_cast<const uint4*>(pins) + 2ull * e + 1);
  return {{q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w}};
}
__device__ __forceinline__ uint32_t edge_gid_stream(const RoundParams& P, uint32_t e) {
  return (P.orig ? __ldcs(P.orig + e) : e) + P.id_base;
}
__device__ __forceinline__ double base_of_stream(const RoundParams& P, uint32_t e) {
  // the round-1 sweep streams every weight once, coalesced: the f64 array (always kept beside the
  // byte codes) costs it fewer instructions and registers (measured: 2.18 vs 2.52 ms on config 2)
  return P.base ? __ldcs(P.base + e) : P.base_const;
}

// Block-wide exclusive offset of `flag` plus the block total (warp ballot + scan of 8 warp sums).
// Callers must __syncthreads() before the next use of s_warp.
__device__ __forceinline__ uint32_t block_rank(bool flag, uint32_t* s_warp, uint32_t& total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ballot = __ballot_sync(0xffffffffu, flag);
  const uint32_t within = __popc(ballot & ((1u << lane) - 1u));
  if (lane == 0) s_warp[warp] = __popc(ballot);
  __syncthreads();
  uint32_t before = 0, sum = 0;
#pragma unroll
  for (int w = 0; w < kWarpsPerBlock; ++w) {
    const uint32_t c = s_warp[w];
    if (w < static_cast<int>(warp)) before += c;
    sum += c;
  }
  total = sum;
  return before + within;
}

__device__ __forceinline__ uint32_t block_sum(uint32_t x, uint32_t* s_warp) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = x;
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int w = 0; w < kWarpsPerBlock; ++w) s += s_warp[w];
  return s;
}

struct WeightStats {
  unsigned long long min_bits;  // of fl(base + lo); positive doubles order like their bit patterns
  unsigned long long max_bits;
  uint32_t non_integer;         // some fl(base + lo) is not an integer below 2^32
  uint32_t non_positive;        // some base weight is <= 0 or NaN (hypergraph.hpp:104)
};

}  // namespace hlmb
