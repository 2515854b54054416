// hlm_host_simd.h -- the two loops of the host-assisted loader (hlm_engine.cu `upload`).
//
// While the pin array crosses PCIe the host's cores look at the other two arrays of the reference's
// Hypergraph (hypergraph.hpp:19-27): the u64 edge offsets (are all differences equal?) and the f64
// base weights (are all of them integers in 0..255, so that one byte each can be shipped?).  These
// two passes over 4.3 GB are the critical path of the one-shot call on config 2, so they run as
// AVX2 code where the CPU has it (runtime dispatch) -- the scalar weight loop is compute-bound at
// ~1.7 GB/s per core, the vector form runs at the memory bandwidth.
#pragma once
#include <cstdint>

namespace hlmb {

// packed[i] = (uint8_t) w[i] for i in [b, e); true if some w[i] is not an integer in [0, 255]
// (the packed bytes are then meaningless).
bool host_pack_weights_u8(const double* w, uint8_t* packed, uint64_t b, uint64_t e);
bool host_pack_weights_u8_scalar(const double* w, uint8_t* packed, uint64_t b, uint64_t e);

// true if off[i + 1] - off[i] != d for some i in [b, e)
bool host_offsets_differ(const uint64_t* off, uint64_t d, uint64_t b, uint64_t e);
bool host_offsets_differ_scalar(const uint64_t* off, uint64_t d, uint64_t b, uint64_t e);

// sizes[i] = off[i + 1] - off[i] for i in [b, e) as 16-bit values; true if some difference does not fit (or
// the offsets decrease): the sizes are then meaningless.  Ragged instances ship these 2 bytes per edge instead
// of 8 bytes of offset and the device rebuilds the offsets with a scan.
bool host_pack_sizes_u16(const uint64_t* off, uint16_t* sizes, uint64_t b, uint64_t e);

// which implementation the dispatcher picked: "avx2" or "scalar"
const char* host_simd_level();

}  // namespace hlmb
