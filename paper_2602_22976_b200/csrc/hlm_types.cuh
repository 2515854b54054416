// hlm_types.cuh -- shared device types / helpers for the sm_100a kernels of the local-max matching round (CRCW variant) plus the
// loader / result-assembly helpers.  Reference semantics: local_max_par.hpp:93-253
// (run_soft_delete + local_max_crcw) and local_max_seq.hpp:22-90; see DESIGN.md for the mapping
// of reference phases onto these kernels.
//
// Round r on the device (one "step" of the WHILE graph):
//   k_filter_vmax  -- for every edge that was active in round r-1: drop it if it matched, drop it
//                     (and count it as deactivated) if one of its pins died, otherwise append it to
//                     the round-r active list and atomicMax its round-tagged key into vkey[pin].
//                     (reference phases: deactivation :229-248, collect :163, weight refresh
//                     :126-135 and vertex argmax :137-159, fused)
//   k_check_commit -- an active edge is matched iff its key is the maximum at every pin
//                     (== agreement count :202-224); matched edges record their round and set the
//                     dead bit of their pins (completion marking :221).
//   k_advance      -- one thread: round bookkeeping, termination, round cap, tie / epoch exits.
// All memory-bound integer work: no tensor cores.
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
};

// Device-resident loop state; every kernel reads it, k_advance is its only writer besides the
// per-list counters.
struct Ctrl {
  uint32_t round;        // round being processed (1-based)
  uint32_t parity;       // list buffer holding the previous round's active list
  uint32_t count[2][2];  // [buffer][class] list lengths
  uint32_t tie_flag;
  uint32_t status;
  uint32_t max_rounds;
  uint32_t rounds_done;
  unsigned long long edges_swept;  // sum over rounds of the active-list lengths
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
  double base_const;
  uint32_t n;
  uint32_t m;
  uint32_t has_large;  // some edges have more than kLargeEdge pins
  uint32_t id_base;    // global id of local edge 0 (edge-partitioned instances); priorities use global ids
  StreamParams stream;
  KeyScheme ks;
  Ctrl* ctrl;
  unsigned long long* vkey;  // n round-tagged vertex maxima
  uint32_t* dead;            // n bits: vertex covered by a matched edge
  uint16_t* mround;          // m: 0 = not matched, else the round it matched in
  uint32_t* list[2][2];      // [class][buffer] active-edge lists
  uint8_t* mflag[2];         // [class] per list position: matched in the round just checked
  uint32_t ident0;           // class-0 list of round 1 is the identity (no array)
  uint32_t* matched_cnt;     // [round] edges matched in that round
  uint32_t* deact_cnt;       // [round] edges deactivated in that round
};

__device__ __forceinline__ bool vertex_dead(const uint32_t* dead, uint32_t v) {
  return (__ldg(dead + (v >> 5)) >> (v & 31)) & 1u;
}

__device__ __forceinline__ double base_of(const RoundParams& P, uint32_t e) {
  return P.base ? __ldg(P.base + e) : P.base_const;
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

// Block-wide exclusive offset of `flag` plus the block total (warp ballot + scan of 8 warp sums).
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
