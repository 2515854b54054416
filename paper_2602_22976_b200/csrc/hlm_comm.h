// hlm_comm.h -- NCCL behind a function table bound at run time (dlopen of libnccl.so.2).
//
// The library has no link-time dependency on NCCL: a single-GPU user never loads it, and inside a
// process that already holds a libnccl.so.2 (e.g. torch's bundled one) dlopen returns that copy, so
// the communicator and the framework's own collectives share one NCCL.  Only the handful of calls
// the edge-partitioned round driver (hlm_shard.inc) issues are bound.  The constants below are
// NCCL's public ABI (nccl.h: ncclDataType_t, ncclRedOp_t, NCCL_UNIQUE_ID_BYTES).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace hlmb {

constexpr int kNcclUniqueIdBytes = 128;
struct NcclUniqueId {
  char internal[kNcclUniqueIdBytes];
};
using NcclComm = void*;
enum NcclType { kNcclUint32 = 3, kNcclUint64 = 5, kNcclFloat64 = 8 };
enum NcclOp { kNcclSum = 0, kNcclMax = 2 };

struct NcclApi {
  int (*GetVersion)(int*);
  int (*GetUniqueId)(NcclUniqueId*);
  int (*CommInitRank)(NcclComm*, int, NcclUniqueId, int);
  int (*CommInitAll)(NcclComm*, int, const int*);
  int (*CommDestroy)(NcclComm);
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
  int (*Broadcast)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
  int (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t);
  int (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t);
  int (*GroupStart)();
  int (*GroupEnd)();
  const char* (*GetErrorString)(int);
};

// null (with set_error) when libnccl.so.2 cannot be loaded or lacks a symbol
const NcclApi* nccl_api();

// A communicator handed across the C-ABI: one rank of `nranks` processes, bound to one device.
struct Comm {
  NcclComm nccl = nullptr;
  int rank = 0, nranks = 1, device = 0;
  bool owned = true;
};

}  // namespace hlmb
