// ctis_comm.cu — the latency mode's collective: a NCCL communicator owned
// by libctis, so that one band-sharded MLEM iteration (partial forward -> reduce-scatter of g_hat ->
// ratio on the rank's pixel slice -> all-gather of r -> back-projection + update) is enqueued, and
// captured into ONE CUDA graph, by the library itself (ctis_api.cu: ctis_mlem_band_sharded).
//
// NCCL is resolved at run time (dlopen / dlsym): libctis loads and runs its single-GPU entry points on
// a machine without NCCL; the band-sharded entry points then return CTIS_ERR_UNSUPPORTED.  Inside a
// PyTorch process the NCCL that torch already loaded (same SONAME libnccl.so.2) is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "ctis_comm.h"
#include "ctis_nvls.h"

namespace ctis {
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*reduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
  // symmetric memory + device API (NCCL >= 2.28), for the fused exchange kernel (f-1)
  ncclResult_t (*memAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*memFree)(void*) = nullptr;
  ncclResult_t (*windowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*windowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
  ncclResult_t (*devCommCreate)(ncclComm_t, const void*, void*) = nullptr;
  ncclResult_t (*devCommDestroy)(ncclComm_t, const void*) = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    if (const char* p = std::getenv("CTIS_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not loadable: ") + (dlerror() ? dlerror() : "?");
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(sym("ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(sym("ncclCommInitRank"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(sym("ncclCommDestroy"));
    a.reduceScatter = reinterpret_cast<decltype(a.reduceScatter)>(sym("ncclReduceScatter"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(sym("ncclAllGather"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(sym("ncclAllReduce"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(sym("ncclGetErrorString"));
    a.getVersion = reinterpret_cast<decltype(a.getVersion)>(sym("ncclGetVersion"));
    a.memAlloc = reinterpret_cast<decltype(a.memAlloc)>(sym("ncclMemAlloc"));
    a.memFree = reinterpret_cast<decltype(a.memFree)>(sym("ncclMemFree"));
    a.windowRegister = reinterpret_cast<decltype(a.windowRegister)>(sym("ncclCommWindowRegister"));
    a.windowDeregister = reinterpret_cast<decltype(a.windowDeregister)>(sym("ncclCommWindowDeregister"));
    a.devCommCreate = reinterpret_cast<decltype(a.devCommCreate)>(sym("ncclDevCommCreate"));
    a.devCommDestroy = reinterpret_cast<decltype(a.devCommDestroy)>(sym("ncclDevCommDestroy"));
    a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.reduceScatter && a.allGather && a.allReduce &&
           a.errorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

std::string nccl_msg(const char* where, ncclResult_t r) {
  return std::string(where) + ": " + (api().errorString ? api().errorString(r) : "NCCL error");
}

}  // namespace

bool nccl_available(std::string* why) {
  const NcclApi& a = api();
  if (!a.ok && why) *why = a.why;
  return a.ok;
}

int nccl_version() {
  int v = 0;
  if (api().ok && api().getVersion) api().getVersion(&v);
  return v;
}

bool nccl_unique_id(unsigned char out[kNcclIdBytes], std::string* err) {
  if (!nccl_available(err)) return false;
  ncclUniqueId id;
  ncclResult_t r = api().getUniqueId(&id);
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclGetUniqueId", r);
    return false;
  }
  static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId size");
  memcpy(out, &id, kNcclIdBytes);
  return true;
}

bool nccl_comm_init(void** comm, int nranks, int rank, const unsigned char id[kNcclIdBytes], std::string* err) {
  if (!nccl_available(err)) return false;
  ncclUniqueId uid;
  memcpy(&uid, id, kNcclIdBytes);
  ncclComm_t c = nullptr;
  ncclResult_t r = api().commInitRank(&c, nranks, uid, rank);
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclCommInitRank", r);
    return false;
  }
  *comm = c;
  return true;
}

void nccl_comm_destroy(void* comm) {
  if (comm && api().ok) api().commDestroy(static_cast<ncclComm_t>(comm));
}

bool nccl_reduce_scatter_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s,
                             std::string* err) {
  ncclResult_t r = api().reduceScatter(send, recv, count, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) *err = nccl_msg("ncclReduceScatter", r);
  return r == ncclSuccess;
}

bool nccl_all_gather_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s, std::string* err) {
  ncclResult_t r = api().allGather(send, recv, count, ncclFloat32, static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) *err = nccl_msg("ncclAllGather", r);
  return r == ncclSuccess;
}

bool nccl_all_reduce_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s, std::string* err) {
  ncclResult_t r = api().allReduce(send, recv, count, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) *err = nccl_msg("ncclAllReduce", r);
  return r == ncclSuccess;
}

bool nvls_setup(void* nccl_comm, size_t bytes, int device, NvlsComm* out, std::string* err) {
  const NcclApi& a = api();
  if (!a.ok || !a.memAlloc || !a.windowRegister || !a.devCommCreate) {
    *err = "NCCL symmetric memory / device API unavailable (needs NCCL >= 2.28)";
    return false;
  }
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  NvlsComm c;
  c.bytes = (bytes + 4095) & ~size_t(4095);
  ncclResult_t r = a.memAlloc(&c.buf, c.bytes);
  if (r != ncclSuccess) {
    *err = nccl_msg("ncclMemAlloc", r);
    return false;
  }
  ncclWindow_t win = nullptr;
  r = a.windowRegister(comm, c.buf, c.bytes, &win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    a.memFree(c.buf);
    *err = nccl_msg("ncclCommWindowRegister", r);
    return false;
  }
  c.window = win;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  c.blocks = 2 * sms;
  const bool mc = !std::getenv("CTIS_NVLS_NO_MULTIMEM");  // try NVLS first; NCCL refuses it where unsupported
  std::vector<uint64_t> reqs((devcomm_requirements_bytes() + 7) / 8, 0);
  c.devcomm = ::operator new(devcomm_bytes());
  memset(c.devcomm, 0, devcomm_bytes());
  r = ncclInvalidUsage;
  if (mc) {
    devcomm_requirements(reqs.data(), c.blocks, true);
    r = a.devCommCreate(comm, reqs.data(), c.devcomm);
  }
  if (r != ncclSuccess) {  // no multimem: NVLink peer loads / stores
    devcomm_requirements(reqs.data(), c.blocks, false);
    r = a.devCommCreate(comm, reqs.data(), c.devcomm);
  }
  if (r != ncclSuccess) {
    a.windowDeregister(comm, win);
    a.memFree(c.buf);
    ::operator delete(c.devcomm);
    *err = nccl_msg("ncclDevCommCreate", r);
    return false;
  }
  c.multimem = devcomm_has_multimem(c.devcomm) && devcomm_lsa_size(c.devcomm) > 1 ? 1 : 0;
  if (std::getenv("CTIS_NVLS_NO_MULTIMEM")) c.multimem = 0;
  *out = c;
  return true;
}

void nvls_teardown(void* nccl_comm, NvlsComm* c) {
  const NcclApi& a = api();
  if (!c || !c->buf || !a.ok) return;
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  if (a.devCommDestroy && c->devcomm) a.devCommDestroy(comm, c->devcomm);
  if (a.windowDeregister && c->window) a.windowDeregister(comm, static_cast<ncclWindow_t>(c->window));
  if (a.memFree) a.memFree(c->buf);
  ::operator delete(c->devcomm);
  *c = NvlsComm();
}

}  // namespace ctis
