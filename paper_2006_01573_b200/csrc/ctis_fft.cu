// ctis_fft.cu — the paper's own WBH projector (Fourier route) on B200, as a comparator arm of the
// tap projector under the same plan (ctis_set_option(CTIS_OPT_PROJECTOR, 1)):
//
//   embed    v_i = E f_i (zero outside the field stop)            PAPER.md P:127-133 Eq. 11, Alg. 1 l. 6
//   forward  g_hat = F^-1 sum_i d_i (.) F v_i,  d_i = F c_i        P:140-145 Eq. 13, Alg. 1 l. 7
//   back     z_i = E^T F^-1 (conj(d_i) (.) F u)                    P:180-184 Eq. 17, Eq. 15
//
// F is cuFFT's unnormalised 1-D real-to-complex DFT of length n (half spectra of beta = n/2 + 1
// points, Hermitian symmetry of P:180-190); the 1/n of F^-1 is applied in the epilogues.  Per
// projection: w batched R2C (forward) or C2R (back) transforms of length n plus one single
// transform, i.e. the 2w + 2 FFTs per iteration of Alg. 1; O(w n) complex scratch.
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include "ctis_fft.h"

namespace ctis {

namespace {

// v[i][p] = f_i[p_r + a p_c] if (p_r, p_c) = (p mod gamma, p div gamma) lies in the field stop, else 0
// (the embed map E of Eq. 11 written as a gather over the whole FPA, so no separate zero fill).
__global__ void fft_embed_kernel(const float* __restrict__ f, float* __restrict__ v, int w, int a, int alpha,
                                 int gamma, long long n, long long ell) {
  const long long total = (long long)w * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n, p = t - i * n;
    const int pr = (int)(p % gamma), pc = (int)(p / gamma);
    v[t] = (pr < a && pc < alpha) ? __ldg(f + i * ell + pr + (long long)a * pc) : 0.f;
  }
}

// acc[k] = sum_i d_i[k] * V_i[k]  (the band sum of Eq. 13 in the frequency domain)
__global__ void fft_mac_kernel(const cufftComplex* __restrict__ d, const cufftComplex* __restrict__ V,
                               cufftComplex* __restrict__ acc, int w, long long nc) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nc;
       k += (long long)gridDim.x * blockDim.x) {
    float re = 0.f, im = 0.f;
    for (int i = 0; i < w; ++i) {
      const cufftComplex x = d[(long long)i * nc + k], y = V[(long long)i * nc + k];
      re = fmaf(x.x, y.x, fmaf(-x.y, y.y, re));
      im = fmaf(x.x, y.y, fmaf(x.y, y.x, im));
    }
    acc[k] = make_float2(re, im);
  }
}

// g_hat[p] += t[p] / n
__global__ void fft_scale_add_kernel(const float* __restrict__ t, float* __restrict__ ghat, long long n, float inv_n) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x)
    ghat[p] += t[p] * inv_n;
}

// Y_i[k] = conj(d_i[k]) * U[k]  (Eq. 17)
__global__ void fft_conj_mul_kernel(const cufftComplex* __restrict__ d, const cufftComplex* __restrict__ U,
                                    cufftComplex* __restrict__ Y, int w, long long nc) {
  const long long total = (long long)w * nc;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long k = t % nc;
    const cufftComplex x = d[t], u = U[k];
    Y[t] = make_float2(fmaf(x.x, u.x, x.y * u.y), fmaf(x.x, u.y, -x.y * u.x));
  }
}

// zeta_j = y_i[E(q)] / n (Eq. 15); mode 1: f_j <- f_j * zeta_j * (1/h_i); 2: f_j <- f_j exp(zeta_j / h_i);
// mode 0: out_j = zeta_j
__global__ void fft_extract_kernel(const float* __restrict__ y, float* __restrict__ fz,
                                   const float* __restrict__ inv_h, int mode, int a, int gamma, long long n,
                                   long long ell, long long m, float inv_n) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < m; j += (long long)gridDim.x * blockDim.x) {
    const long long i = j / ell, q = j - i * ell;
    const long long qr = q % a, qc = q / a;
    const float z = y[i * n + qr + (long long)gamma * qc] * inv_n;
    const float ih = __ldg(inv_h + i);
    fz[j] = mode == 1 ? fz[j] * z * ih : mode == 2 ? fz[j] * expf(z * ih) : z;
  }
}

int blocks_for(long long work) {
  const long long b = (work + 255) / 256;
  return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

cudaError_t cufft_err(cufftResult r) { return r == CUFFT_SUCCESS ? cudaSuccess : cudaErrorUnknown; }

}  // namespace

void fft_destroy(FftState* st) {
  if (!st) return;
  for (cufftHandle h : {st->r2c_w, st->c2r_w, st->r2c_1, st->c2r_1})
    if (h) cufftDestroy(h);
  for (void* p : {(void*)st->d, (void*)st->real, (void*)st->spec, (void*)st->acc, (void*)st->tmp, (void*)st->inv_h})
    if (p) cudaFree(p);
  delete st;
}

cudaError_t fft_create(FftState** out, int a, int alpha, int w, int gamma, int xi,
                       const std::vector<std::vector<std::pair<int64_t, float>>>& band_taps,
                       const std::vector<float>& inv_h) {
  *out = nullptr;
  auto* st = new FftState();
  st->a = a;
  st->alpha = alpha;
  st->w = w;
  st->gamma = gamma;
  st->n = (long long)gamma * xi;
  st->nc = st->n / 2 + 1;
  st->ell = (long long)a * alpha;
  const size_t rbytes = sizeof(float) * (size_t)w * (size_t)st->n;
  const size_t cbytes = sizeof(cufftComplex) * (size_t)w * (size_t)st->nc;
  cudaError_t e = cudaMalloc(&st->d, cbytes);
  if (e == cudaSuccess) e = cudaMalloc(&st->real, rbytes);
  if (e == cudaSuccess) e = cudaMalloc(&st->spec, cbytes);
  if (e == cudaSuccess) e = cudaMalloc(&st->acc, sizeof(cufftComplex) * (size_t)st->nc);
  if (e == cudaSuccess) e = cudaMalloc(&st->tmp, sizeof(float) * (size_t)st->n);
  if (e == cudaSuccess) e = cudaMalloc(&st->inv_h, sizeof(float) * (size_t)w);
  if (e == cudaSuccess) e = cudaMemcpy(st->inv_h, inv_h.data(), sizeof(float) * (size_t)w, cudaMemcpyHostToDevice);
  int nn = (int)st->n;
  if (e == cudaSuccess)
    e = cufft_err(cufftPlanMany(&st->r2c_w, 1, &nn, nullptr, 1, (int)st->n, nullptr, 1, (int)st->nc, CUFFT_R2C, w));
  if (e == cudaSuccess)
    e = cufft_err(cufftPlanMany(&st->c2r_w, 1, &nn, nullptr, 1, (int)st->nc, nullptr, 1, (int)st->n, CUFFT_C2R, w));
  if (e == cudaSuccess) e = cufft_err(cufftPlan1d(&st->r2c_1, nn, CUFFT_R2C, 1));
  if (e == cudaSuccess) e = cufft_err(cufftPlan1d(&st->c2r_1, nn, CUFFT_C2R, 1));
  if (e == cudaSuccess) {
    // d_i = F c_i: the calibration images (taps scattered into n-vectors), one batched R2C
    std::vector<float> c((size_t)w * (size_t)st->n, 0.f);
    for (int i = 0; i < w; ++i)
      for (const auto& t : band_taps[i]) c[(size_t)i * st->n + (size_t)t.first] += t.second;
    e = cudaMemcpy(st->real, c.data(), rbytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cufft_err(cufftSetStream(st->r2c_w, 0));
    if (e == cudaSuccess) e = cufft_err(cufftExecR2C(st->r2c_w, st->real, st->d));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    fft_destroy(st);
    return e;
  }
  *out = st;
  return cudaSuccess;
}

cudaError_t fft_forward_accumulate(FftState* st, const float* f, float* ghat, cudaStream_t s, int64_t* cnt) {
  fft_embed_kernel<<<blocks_for((long long)st->w * st->n), 256, 0, s>>>(f, st->real, st->w, st->a, st->alpha,
                                                                       st->gamma, st->n, st->ell);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cufft_err(cufftSetStream(st->r2c_w, s));
  if (e == cudaSuccess) e = cufft_err(cufftExecR2C(st->r2c_w, st->real, st->spec));
  if (e != cudaSuccess) return e;
  fft_mac_kernel<<<blocks_for(st->nc), 256, 0, s>>>(st->d, st->spec, st->acc, st->w, st->nc);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cufft_err(cufftSetStream(st->c2r_1, s));
  if (e == cudaSuccess) e = cufft_err(cufftExecC2R(st->c2r_1, st->acc, st->tmp));
  if (e != cudaSuccess) return e;
  fft_scale_add_kernel<<<blocks_for(st->n), 256, 0, s>>>(st->tmp, ghat, st->n, 1.0f / (float)st->n);
  if (cnt) *cnt += 5;
  return cudaGetLastError();
}

cudaError_t fft_back(FftState* st, const float* r, float* fz, int mode, cudaStream_t s, int64_t* cnt) {
  cudaError_t e = cufft_err(cufftSetStream(st->r2c_1, s));
  if (e == cudaSuccess) e = cufft_err(cufftExecR2C(st->r2c_1, const_cast<float*>(r), st->acc));
  if (e != cudaSuccess) return e;
  fft_conj_mul_kernel<<<blocks_for((long long)st->w * st->nc), 256, 0, s>>>(st->d, st->acc, st->spec, st->w, st->nc);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cufft_err(cufftSetStream(st->c2r_w, s));
  if (e == cudaSuccess) e = cufft_err(cufftExecC2R(st->c2r_w, st->spec, st->real));
  if (e != cudaSuccess) return e;
  const long long m = (long long)st->w * st->ell;
  fft_extract_kernel<<<blocks_for(m), 256, 0, s>>>(st->real, fz, st->inv_h, mode, st->a, st->gamma, st->n, st->ell, m,
                                                   1.0f / (float)st->n);
  if (cnt) *cnt += 4;
  return cudaGetLastError();
}

}  // namespace ctis
