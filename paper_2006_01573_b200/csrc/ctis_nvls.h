// The fused NVLink exchange + ratio of the latency mode (ctis_nvls.cu) and its NCCL
// symmetric-memory state (ctis_comm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace ctis {
struct NvlsComm {
  void* buf = nullptr;      // symmetric exchange buffer (ncclMemAlloc), `bytes` long
  size_t bytes = 0;
  void* window = nullptr;   // ncclWindow_t
  void* devcomm = nullptr;  // heap copy of the ncclDevComm
  int blocks = 0;           // CTAs of the exchange kernel (one LSA barrier each)
  int multimem = 0;         // 1: NVLS multimem path, 0: NVLink peer loads / stores
};
// collective over the communicator: allocate + register the window, create the device communicator
bool nvls_setup(void* nccl_comm, size_t bytes, int device, NvlsComm* out, std::string* err);
void nvls_teardown(void* nccl_comm, NvlsComm* c);
cudaError_t launch_exchange_ratio(const NvlsComm& c, long long base, long long slice, const float* g, long long n,
                                  cudaStream_t s);
size_t devcomm_bytes();
size_t devcomm_requirements_bytes();
void devcomm_requirements(void* reqs, int barriers, bool multimem);
int devcomm_lsa_size(const void* devcomm);
bool devcomm_has_multimem(const void* devcomm);
}  // namespace ctis
