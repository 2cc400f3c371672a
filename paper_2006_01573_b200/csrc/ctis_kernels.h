// Launchers of the element-wise kernels (ctis_kernels.cu).
#pragma once

#include <cuda_runtime.h>

namespace ctis {
// pdl: launch with programmatic stream serialization (the kernels call griddepcontrol.wait first)
cudaError_t launch_ratio(const float* g, float* ghat, float* r, long long count, bool zero_ghat, cudaStream_t s,
                         bool pdl = false);
// ratio (zeroing g_hat) over the pixel box rows [r0, r0 + 4*nr4) x columns [c0, c0 + nc) of every frame
// (frames of n pixels, column pitch gamma; r0 and gamma multiples of 4, buffers 16-byte aligned)
cudaError_t launch_ratio_box(const float* g, float* ghat, float* r, long long n, int gamma, int r0, int nr4, int c0,
                             int nc, int frames, cudaStream_t s, bool pdl = false);
// dst[c * pitch + r] = src[c * a + r] for r < a, c < cols (row repack to a 16-byte pitch for TMA)
cudaError_t launch_repack_rows(const float* src, float* dst, int a, int pitch, long long cols, cudaStream_t s);
// mode-split back update: f[j] <- upd(mode, f[j], z[j], invh[(j % (ell*w)) / ell]) (1: f*z*ih, 2: f*exp(z*ih)),
// z[j] <- 0, for j < count (frames of ell*w voxels)
cudaError_t launch_split_update(float* f, float* z, const float* invh, int ell, int w, long long count, int mode,
                                cudaStream_t s);
cudaError_t launch_sensitivity(const float* hband, float* h, int ell, int m, cudaStream_t s);
cudaError_t launch_validate(const float* x, long long count, int* flag, cudaStream_t s);
// SMART log-ratio (zeroing g_hat)
cudaError_t launch_log_ratio(const float* g, float* ghat, float* r, long long count, cudaStream_t s, bool pdl = false);
// ratio (zeroing g_hat) + ll[*counter] += sum_p [g log g_hat - g_hat] (fp64)
cudaError_t launch_ratio_ll(const float* g, float* ghat, float* r, long long count, double* ll, const int* counter,
                            cudaStream_t s, bool pdl = false);
// one thread: ++*counter, then the WHILE condition (continue unless max_iters or the stop rule)
cudaError_t launch_mlem_check(const double* ll, int* counter, int max_iters, double rel_tol,
                              unsigned long long cond_handle, cudaStream_t s);
}  // namespace ctis
