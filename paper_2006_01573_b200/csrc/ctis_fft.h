// The paper's Fourier (WBH) projector as a comparator arm (ctis_fft.cu).  Internal, not ABI.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <utility>
#include <vector>

namespace ctis {

struct FftState {
  int a = 0, alpha = 0, w = 0, gamma = 0;
  long long n = 0, nc = 0, ell = 0;
  cufftHandle r2c_w = 0, c2r_w = 0, r2c_1 = 0, c2r_1 = 0;
  cufftComplex* d = nullptr;     // [w][nc] spectra of the calibration images c_i
  float* real = nullptr;         // [w][n] embedded bands / back-projected bands
  cufftComplex* spec = nullptr;  // [w][nc]
  cufftComplex* acc = nullptr;   // [nc]
  float* tmp = nullptr;          // [n]
  float* inv_h = nullptr;        // [w] 1 / h_lambda
};

cudaError_t fft_create(FftState** out, int a, int alpha, int w, int gamma, int xi,
                       const std::vector<std::vector<std::pair<int64_t, float>>>& band_taps,
                       const std::vector<float>& inv_h);
void fft_destroy(FftState* st);
// g_hat[n] += H f (one frame)
cudaError_t fft_forward_accumulate(FftState* st, const float* f, float* ghat, cudaStream_t s, int64_t* cnt);
// mode 1: f <- f (.) (H^T r) (/) h; mode 0: fz = H^T r (one frame)
cudaError_t fft_back(FftState* st, const float* r, float* fz, int mode, cudaStream_t s, int64_t* cnt);

}  // namespace ctis
