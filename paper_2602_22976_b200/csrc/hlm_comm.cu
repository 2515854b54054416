// hlm_comm.cu -- run-time binding of NCCL and the communicator entry points of the C-ABI.
#include "hlm_comm.h"

#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "hlm_engine.h"

namespace hlmb {

static NcclApi g_api;
static bool g_api_ok = false;
static std::once_flag g_api_once;
static char g_api_err[256] = "";

static void bind_nccl() {
  // HLM_B200_NCCL_LIB: an explicit path; otherwise the soname (the copy already in the process wins)
  const char* names[] = {std::getenv("HLM_B200_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names) {
    if (!nm || !nm[0]) continue;
    h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    std::snprintf(g_api_err, sizeof(g_api_err), "libnccl.so.2 could not be loaded: %s", dlerror());
    return;
  }
  struct Sym {
    const char* name;
    void** slot;
  } syms[] = {{"ncclGetVersion", reinterpret_cast<void**>(&g_api.GetVersion)},
              {"ncclGetUniqueId", reinterpret_cast<void**>(&g_api.GetUniqueId)},
              {"ncclCommInitRank", reinterpret_cast<void**>(&g_api.CommInitRank)},
              {"ncclCommInitAll", reinterpret_cast<void**>(&g_api.CommInitAll)},
              {"ncclCommDestroy", reinterpret_cast<void**>(&g_api.CommDestroy)},
              {"ncclAllReduce", reinterpret_cast<void**>(&g_api.AllReduce)},
              {"ncclBroadcast", reinterpret_cast<void**>(&g_api.Broadcast)},
              {"ncclSend", reinterpret_cast<void**>(&g_api.Send)},
              {"ncclRecv", reinterpret_cast<void**>(&g_api.Recv)},
              {"ncclGroupStart", reinterpret_cast<void**>(&g_api.GroupStart)},
              {"ncclGroupEnd", reinterpret_cast<void**>(&g_api.GroupEnd)},
              {"ncclGetErrorString", reinterpret_cast<void**>(&g_api.GetErrorString)}};
  for (const Sym& s : syms) {
    *s.slot = dlsym(h, s.name);
    if (!*s.slot) {
      std::snprintf(g_api_err, sizeof(g_api_err), "libnccl.so.2 lacks %s", s.name);
      return;
    }
  }
  g_api_ok = true;
}

const NcclApi* nccl_api() {
  std::call_once(g_api_once, bind_nccl);
  if (!g_api_ok) {
    set_error("%s", g_api_err);
    return nullptr;
  }
  return &g_api;
}

}  // namespace hlmb

using namespace hlmb;

extern "C" {

int hlm_b200_comm_unique_id(uint8_t* id) {
  if (!id) {
    set_error("null argument");
    return HLM_B200_ERR_INPUT;
  }
  const NcclApi* api = nccl_api();
  if (!api) return HLM_B200_ERR_NCCL;
  NcclUniqueId u;
  const int rc = api->GetUniqueId(&u);
  if (rc != 0) {
    set_error("ncclGetUniqueId failed: %s", api->GetErrorString(rc));
    return HLM_B200_ERR_NCCL;
  }
  std::memcpy(id, u.internal, kNcclUniqueIdBytes);
  return HLM_B200_OK;
}

int hlm_b200_comm_create(const uint8_t* id, int rank, int nranks, int device, hlm_b200_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !id)) {
    set_error("hlm_b200_comm_create: bad rank %d of %d or null argument", rank, nranks);
    return HLM_B200_ERR_INPUT;
  }
  *out = nullptr;
  const NcclApi* api = nccl_api();
  if (!api) return HLM_B200_ERR_NCCL;
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) {
    set_error("cudaSetDevice(%d) failed: %s", device, cudaGetErrorString(ce));
    return HLM_B200_ERR_CUDA;
  }
  NcclUniqueId u;
  if (id) {
    std::memcpy(u.internal, id, kNcclUniqueIdBytes);
  } else {
    const int rc = api->GetUniqueId(&u);
    if (rc != 0) {
      set_error("ncclGetUniqueId failed: %s", api->GetErrorString(rc));
      return HLM_B200_ERR_NCCL;
    }
  }
  Comm* c = new Comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  const int rc = api->CommInitRank(&c->nccl, nranks, u, rank);
  if (rc != 0) {
    set_error("ncclCommInitRank(rank %d of %d, device %d) failed: %s", rank, nranks, device, api->GetErrorString(rc));
    delete c;
    return HLM_B200_ERR_NCCL;
  }
  *out = reinterpret_cast<hlm_b200_comm*>(c);
  return HLM_B200_OK;
}

int hlm_b200_comm_info(const hlm_b200_comm* comm, int* rank, int* nranks, int* device, int* nccl_version) {
  const Comm* c = reinterpret_cast<const Comm*>(comm);
  if (!c) {
    set_error("null communicator");
    return HLM_B200_ERR_INPUT;
  }
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  if (device) *device = c->device;
  if (nccl_version) {
    *nccl_version = 0;
    if (const NcclApi* api = nccl_api()) api->GetVersion(nccl_version);
  }
  return HLM_B200_OK;
}

void hlm_b200_comm_destroy(hlm_b200_comm* comm) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!c) return;
  if (c->nccl && c->owned) {
    if (const NcclApi* api = nccl_api()) api->CommDestroy(c->nccl);
  }
  delete c;
}

}  // extern "C"
