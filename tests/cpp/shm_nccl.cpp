// shm_nccl.cpp -- TEST INFRASTRUCTURE: the twelve NCCL entry points libhlm_b200.so binds (csrc/hlm_comm.h),
// implemented over a POSIX shared-memory segment, so that several PROCESSES can run the library's multi-rank
// round driver (hlm_b200_match_sharded with nranks > 1) on ONE GPU.  NCCL itself refuses two ranks on the same
// device, and the test boxes have one.  Selected with HLM_B200_NCCL_LIB=<this .so>; never shipped, never loaded
// by the product on its own.  Collectives are blocking and go through the host: synchronise the stream, copy
// to the rank's slot, barrier, combine, copy back.  Sizes are test sizes (a slot holds 16 MB).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <vector>

namespace {

constexpr int kMaxRanks = 8;
constexpr size_t kSlotBytes = 16u << 20;
constexpr size_t kMailBytes = 4096;

struct Header {
  std::atomic<int> ready;      // ranks that have mapped the segment
  std::atomic<int> arrived;    // barrier counter
  std::atomic<int> sense;      // barrier generation
  std::atomic<int> mail_full[kMaxRanks][kMaxRanks];  // [src][dst]
};

struct FakeComm {
  int rank, nranks;
  char name[128];
  uint8_t* base;
  size_t bytes;
  int local_sense;
  Header* hdr() const { return reinterpret_cast<Header*>(base); }
  uint8_t* slot(int r) const { return base + 65536 + static_cast<size_t>(r) * kSlotBytes; }
  uint8_t* mail(int src, int dst) const {
    return base + 65536 + static_cast<size_t>(kMaxRanks) * kSlotBytes + (static_cast<size_t>(src) * kMaxRanks + dst) * kMailBytes;
  }
};

size_t elem_size(int type) {
  switch (type) {
    case 3: return 4;   // ncclUint32
    case 5: return 8;   // ncclUint64
    case 8: return 8;   // ncclFloat64
    default: return 0;
  }
}

void barrier(FakeComm* c) {
  Header* h = c->hdr();
  c->local_sense ^= 1;
  if (h->arrived.fetch_add(1) + 1 == c->nranks) {
    h->arrived.store(0);
    h->sense.store(c->local_sense);
  } else {
    while (h->sense.load() != c->local_sense) usleep(20);
  }
}

// copies ordered on the caller's stream and complete on return (a plain cudaMemcpy from pageable memory may
// return before its DMA has landed, and the library's streams do not synchronise with the legacy stream)
bool d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
}
bool h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
}

template <typename T>
void combine(T* acc, const T* other, size_t count, int op) {
  for (size_t i = 0; i < count; ++i) acc[i] = op == 0 ? static_cast<T>(acc[i] + other[i]) : (acc[i] < other[i] ? other[i] : acc[i]);
}

}  // namespace

extern "C" {

int ncclGetVersion(int* v) {
  *v = 99999;  // recognisably not NCCL
  return 0;
}

int ncclGetUniqueId(void* id) {
  std::memset(id, 0, 128);
  std::snprintf(static_cast<char*>(id), 128, "/hlm_shm_nccl_%d_%ld", static_cast<int>(getpid()), static_cast<long>(time(nullptr)));
  return 0;
}

struct UniqueId {
  char internal[128];
};

int ncclCommInitRank(void** comm, int nranks, UniqueId id, int rank) {
  if (nranks > kMaxRanks) return 5;
  FakeComm* c = new FakeComm();
  c->rank = rank;
  c->nranks = nranks;
  std::memcpy(c->name, id.internal, 128);
  c->bytes = 65536 + static_cast<size_t>(kMaxRanks) * kSlotBytes + static_cast<size_t>(kMaxRanks) * kMaxRanks * kMailBytes;
  c->local_sense = 0;
  int fd = -1;
  if (rank == 0) {
    fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, static_cast<off_t>(c->bytes)) != 0) return 2;  // zero-filled: every atomic starts at 0
  } else {
    for (int tries = 0; tries < 20000 && fd < 0; ++tries) {
      fd = shm_open(c->name, O_RDWR, 0600);
      if (fd < 0) usleep(1000);
    }
    if (fd < 0) return 2;
    off_t have = 0;
    for (int tries = 0; tries < 20000 && have < static_cast<off_t>(c->bytes); ++tries) {
      have = lseek(fd, 0, SEEK_END);
      if (have < static_cast<off_t>(c->bytes)) usleep(1000);
    }
  }
  c->base = static_cast<uint8_t*>(mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
  close(fd);
  if (c->base == MAP_FAILED) return 2;
  c->hdr()->ready.fetch_add(1);
  while (c->hdr()->ready.load() < nranks) usleep(100);
  *comm = c;
  return 0;
}

int ncclCommInitAll(void**, int, const int*) { return 5; }  // several devices in one process: not on one GPU

int ncclCommDestroy(void* comm) {
  FakeComm* c = static_cast<FakeComm*>(comm);
  if (!c) return 0;
  barrier(c);
  if (c->rank == 0) shm_unlink(c->name);
  munmap(c->base, c->bytes);
  delete c;
  return 0;
}

int ncclAllReduce(const void* send, void* recv, size_t count, int type, int op, void* comm, cudaStream_t s) {
  FakeComm* c = static_cast<FakeComm*>(comm);
  const size_t es = elem_size(type), bytes = count * es;
  if (!es || bytes > kSlotBytes) return 5;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  if (!d2h(c->slot(c->rank), send, bytes, s)) return 1;
  barrier(c);
  std::vector<uint8_t> acc(c->slot(0), c->slot(0) + bytes);
  for (int r = 1; r < c->nranks; ++r) {
    if (type == 3) combine(reinterpret_cast<uint32_t*>(acc.data()), reinterpret_cast<const uint32_t*>(c->slot(r)), count, op);
    else if (type == 5) combine(reinterpret_cast<uint64_t*>(acc.data()), reinterpret_cast<const uint64_t*>(c->slot(r)), count, op);
    else combine(reinterpret_cast<double*>(acc.data()), reinterpret_cast<const double*>(c->slot(r)), count, op);
  }
  if (!h2d(recv, acc.data(), bytes, s)) return 1;
  if (std::getenv("SHM_NCCL_TRACE") && count <= 8) {
    std::fprintf(stderr, "[shm_nccl %d] allreduce count %zu type %d op %d:", c->rank, count, type, op);
    for (size_t i = 0; i < count && type == 3; ++i)
      std::fprintf(stderr, " %u->%u", reinterpret_cast<const uint32_t*>(c->slot(c->rank))[i], reinterpret_cast<const uint32_t*>(acc.data())[i]);
    std::fprintf(stderr, "\n");
  }
  barrier(c);  // the slots are free again
  return 0;
}

int ncclBroadcast(const void* send, void* recv, size_t count, int type, int root, void* comm, cudaStream_t s) {
  FakeComm* c = static_cast<FakeComm*>(comm);
  const size_t bytes = count * elem_size(type);
  if (!bytes || bytes > kSlotBytes) return 5;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  if (c->rank == root && !d2h(c->slot(root), send, bytes, s)) return 1;
  barrier(c);
  if (!h2d(recv, c->slot(root), bytes, s)) return 1;
  barrier(c);
  return 0;
}

int ncclSend(const void* send, size_t count, int type, int peer, void* comm, cudaStream_t s) {
  FakeComm* c = static_cast<FakeComm*>(comm);
  const size_t bytes = count * elem_size(type);
  if (!bytes || bytes > kMailBytes) return 5;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  std::atomic<int>& full = c->hdr()->mail_full[c->rank][peer];
  while (full.load() != 0) usleep(20);
  if (!d2h(c->mail(c->rank, peer), send, bytes, s)) return 1;
  full.store(1);
  return 0;
}

int ncclRecv(void* recv, size_t count, int type, int peer, void* comm, cudaStream_t s) {
  FakeComm* c = static_cast<FakeComm*>(comm);
  const size_t bytes = count * elem_size(type);
  if (!bytes || bytes > kMailBytes) return 5;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  std::atomic<int>& full = c->hdr()->mail_full[peer][c->rank];
  while (full.load() != 1) usleep(20);
  if (!h2d(recv, c->mail(peer, c->rank), bytes, s)) return 1;
  full.store(0);
  return 0;
}

int ncclGroupStart() { return 0; }
int ncclGroupEnd() { return 0; }
const char* ncclGetErrorString(int rc) { return rc == 5 ? "shm transport: unsupported call or size" : "shm transport: failure"; }

}  // extern "C"
