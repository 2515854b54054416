// hlm_priority.cuh -- per-(edge, round) priorities on the device.
//
// Bit-exact restatement of the reference's WeightStream (weight_stream.hpp:26-94) for sm_100a:
// every FP64 operation uses an explicit round-to-nearest intrinsic so nvcc's default -fmad=true
// can never contract the reference's two-rounding expression `base + lo + u * width`
// (weight_stream.hpp:82) into an FMA.
//
// On top of it: the 64-bit *round-tagged priority key* the CRCW kernels feed to atomicMax.
//   key(e, r) = tag(r) << payload_bits | payload(e, r)
// payload is a monotone (order-preserving, possibly non-injective) image of the reference's
// strict order (weight, tie_hash, id) (weight_stream.hpp:105-113); tag grows with the round so a
// vertex slot never has to be cleared between rounds.  Equal payloads at one vertex are detected
// by the returning atomicMax and that round is redone on the exact three-level path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hlmb {

struct StreamParams {
  uint64_t seed;
  int32_t kind;   // 0 xorshift, 1 park_miller, 2 splitmix (weight_stream.hpp:17)
  int32_t mode;   // 0 perturb_base, 1 replace_uniform    (weight_stream.hpp:19-22)
  double lo;
  double hi;
  double width;   // hi - lo, computed once on the host exactly as weight_stream.hpp:80
};

enum KeyKind : int32_t {
  KEY_WEIGHT_BITS = 0,  // payload = bits(w) - bits(w_min)
  KEY_INT_HASH = 1,     // zero-width noise, small-integer / constant weights:
                        // payload = (uint(w) - wq_min) << hash_bits | tie_hash >> (64 - hash_bits)
};

struct KeyScheme {
  int32_t kind;
  int32_t payload_bits;  // 1..63
  int32_t hash_bits;     // KEY_INT_HASH only
  uint32_t tag_period;   // number of distinct non-zero tags = 2^(64-payload_bits) - 1 (capped)
  uint32_t precheck;     // filter atomics with a plain L2 load of the running maximum first
  uint32_t fast_default; // xorshift + perturb_base + width != 0 + KEY_WEIGHT_BITS: branch-free key code
  uint64_t wmin_bits;    // KEY_WEIGHT_BITS: bits of the smallest possible weight
  uint64_t wq_min;       // KEY_INT_HASH: smallest integer weight
};

__host__ __device__ __forceinline__ uint64_t mix_splitmix(uint64_t x) {  // weight_stream.hpp:26-31
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix_xorshift(uint64_t x) {  // weight_stream.hpp:33-39
  x *= 0x9E3779B97F4A7C15ull;
  x ^= x >> 12;
  x ^= x << 25;
  x ^= x >> 27;
  return x * 0x2545F4914F6CDD1Dull;
}

__host__ __device__ __forceinline__ uint64_t mix_park_miller(uint64_t x) {  // weight_stream.hpp:42-47
  uint64_t s = x % 2147483646ull + 1ull;
  s = (s * 16807ull) % 2147483647ull;
  s = (s * 16807ull) % 2147483647ull;
  return s;
}

__device__ __forceinline__ uint64_t stream_counter(const StreamParams& s, uint32_t e, uint32_t r) {
  return s.seed ^ (static_cast<uint64_t>(r) << 40) ^ static_cast<uint64_t>(e);  // weight_stream.hpp:91-93
}

__device__ __forceinline__ double unit_from_bits(uint64_t bits) {  // weight_stream.hpp:49-52
  return __dmul_rn(__dadd_rn(__ull2double_rn(bits >> 11), 0.5), 0x1.0p-53);
}

__device__ __forceinline__ double unit_noise(const StreamParams& s, uint32_t e, uint32_t r) {  // :64-75
  const uint64_t c = stream_counter(s, e, r);
  if (s.kind == 0) return unit_from_bits(mix_xorshift(c));
  if (s.kind == 2) return unit_from_bits(mix_splitmix(c));
  return __ddiv_rn(__ull2double_rn(mix_park_miller(c)), 2147483647.0);
}

__device__ __forceinline__ double edge_weight(const StreamParams& s, uint32_t e, uint32_t r,
                                              double base) {  // weight_stream.hpp:78-83
  if (s.mode == 1) return unit_noise(s, e, r);
  if (s.width == 0.0) return __dadd_rn(base, s.lo);
  return __dadd_rn(__dadd_rn(base, s.lo), __dmul_rn(unit_noise(s, e, r), s.width));
}

__device__ __forceinline__ uint64_t tie_hash(const StreamParams& s, uint32_t e, uint32_t r) {  // :86-88
  return mix_splitmix(stream_counter(s, e, r) ^ 0x6A09E667F3BCC909ull);
}

__device__ __forceinline__ uint32_t round_tag(const KeyScheme& k, uint32_t r) {
  return (r - 1u) % k.tag_period + 1u;
}

// Monotone 64-bit image of (weight, tie_hash, id) for round r, tagged with the round.
__device__ __forceinline__ uint64_t priority_key(const StreamParams& s, const KeyScheme& k,
                                                 uint32_t e, uint32_t r, double base, uint32_t tag) {
  uint64_t payload;
  if (k.fast_default) {
    // the reference's default stream (xorshift noise added to the base weight, non-zero width,
    // weight-bit keys) as straight-line code: same operations, no branches on the stream's fields
    const double u = unit_from_bits(mix_xorshift(stream_counter(s, e, r)));
    const double w = __dadd_rn(__dadd_rn(base, s.lo), __dmul_rn(u, s.width));
    return (static_cast<uint64_t>(tag) << k.payload_bits) | (static_cast<uint64_t>(__double_as_longlong(w)) - k.wmin_bits);
  }
  const double w = edge_weight(s, e, r, base);
  if (k.kind == KEY_WEIGHT_BITS) {
    payload = static_cast<uint64_t>(__double_as_longlong(w)) - k.wmin_bits;
  } else {
    const uint64_t wq = static_cast<uint64_t>(__double2ull_rz(w)) - k.wq_min;
    payload = (wq << k.hash_bits) | (tie_hash(s, e, r) >> (64 - k.hash_bits));
  }
  return (static_cast<uint64_t>(tag) << k.payload_bits) | payload;
}

}  // namespace hlmb
