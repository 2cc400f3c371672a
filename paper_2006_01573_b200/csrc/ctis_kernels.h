// Launchers of the element-wise kernels (ctis_kernels.cu).
#pragma once

#include <cuda_runtime.h>

namespace ctis {
cudaError_t launch_ratio(const float* g, float* ghat, float* r, long long count, bool zero_ghat, cudaStream_t s);
cudaError_t launch_sensitivity(const float* hband, float* h, int ell, int m, cudaStream_t s);
cudaError_t launch_validate(const float* x, long long count, int* flag, cudaStream_t s);
}  // namespace ctis
