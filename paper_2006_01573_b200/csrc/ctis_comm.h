// NCCL entry points used by the latency mode (ctis_comm.cu; resolved at run time with dlopen).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <string>

namespace ctis {
constexpr int kNcclIdBytes = 128;
bool nccl_available(std::string* why);
int nccl_version();
bool nccl_unique_id(unsigned char out[kNcclIdBytes], std::string* err);
bool nccl_comm_init(void** comm, int nranks, int rank, const unsigned char id[kNcclIdBytes], std::string* err);
void nccl_comm_destroy(void* comm);
bool nccl_reduce_scatter_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s,
                             std::string* err);
bool nccl_all_gather_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s, std::string* err);
bool nccl_all_reduce_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s, std::string* err);
}  // namespace ctis
