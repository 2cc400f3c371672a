// ctis_kernels.cu — element-wise kernels of the CTIS MLEM hot path (sm_100a):
//   ratio     r = g (/) g_hat, r_p = 0 where g_hat_p <= 0   (Alg. 1 line 8; R4)
//   sensitivity h = H^T 1 = h_lam on every voxel of band lam (P:39 with P:93-97)
//   validate  flag data that EM cannot take (negative, NaN, Inf)
// The projections themselves live in ctis_tables.cu (per-plan cubin with __constant__ taps).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ctis_kernels.h"

namespace ctis {

// Programmatic dependent launch (see ctis_tables.cu pdl_enter)
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... Args>
cudaError_t launch_ex(void (*kern)(Args...), int blocks, int threads, cudaStream_t s, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Ratio over `count` pixels; if zero_ghat, g_hat is reset to 0 after it is read (so the next
// forward projection can accumulate into it with red.add).  Vectorised by 4 when aligned.
__global__ void ratio_kernel(const float* __restrict__ g, float* gh, float* r,
                             long long count, int zero_ghat) {
  pdl_enter();
  const bool aligned = ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(gh) |
                         reinterpret_cast<uintptr_t>(r)) & 15u) == 0;
  const long long n4 = aligned ? (count >> 2) : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
#ifndef CTIS_RATIO_UNROLL
#define CTIS_RATIO_UNROLL 1  // measured (B200, C4, with 4 blocks per SM): 128.2 -> 127.7 us per iteration
#endif
#if CTIS_RATIO_UNROLL
  // two float4 per thread and iteration: the loads of both issued before any division
  for (; t0 + stride < n4; t0 += 2 * stride) {
    const long long i0 = t0, i1 = t0 + stride;
    const float4 gv0 = __ldg(reinterpret_cast<const float4*>(g) + i0);
    const float4 gv1 = __ldg(reinterpret_cast<const float4*>(g) + i1);
    const float4 hv0 = reinterpret_cast<const float4*>(gh)[i0];
    const float4 hv1 = reinterpret_cast<const float4*>(gh)[i1];
    float4 o0, o1;
    o0.x = hv0.x > 0.f ? __fdiv_rn(gv0.x, hv0.x) : 0.f;
    o0.y = hv0.y > 0.f ? __fdiv_rn(gv0.y, hv0.y) : 0.f;
    o0.z = hv0.z > 0.f ? __fdiv_rn(gv0.z, hv0.z) : 0.f;
    o0.w = hv0.w > 0.f ? __fdiv_rn(gv0.w, hv0.w) : 0.f;
    o1.x = hv1.x > 0.f ? __fdiv_rn(gv1.x, hv1.x) : 0.f;
    o1.y = hv1.y > 0.f ? __fdiv_rn(gv1.y, hv1.y) : 0.f;
    o1.z = hv1.z > 0.f ? __fdiv_rn(gv1.z, hv1.z) : 0.f;
    o1.w = hv1.w > 0.f ? __fdiv_rn(gv1.w, hv1.w) : 0.f;
    reinterpret_cast<float4*>(r)[i0] = o0;
    reinterpret_cast<float4*>(r)[i1] = o1;
    if (zero_ghat) {
      reinterpret_cast<float4*>(gh)[i0] = make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(gh)[i1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
#endif
  for (long long i = t0; i < n4; i += stride) {
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    const float4 hv = reinterpret_cast<const float4*>(gh)[i];
    float4 o;
    o.x = hv.x > 0.f ? __fdiv_rn(gv.x, hv.x) : 0.f;
    o.y = hv.y > 0.f ? __fdiv_rn(gv.y, hv.y) : 0.f;
    o.z = hv.z > 0.f ? __fdiv_rn(gv.z, hv.z) : 0.f;
    o.w = hv.w > 0.f ? __fdiv_rn(gv.w, hv.w) : 0.f;
    reinterpret_cast<float4*>(r)[i] = o;
    if (zero_ghat) reinterpret_cast<float4*>(gh)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (long long i = 4 * n4 + t0; i < count; i += stride) {
    const float hv = gh[i];
    r[i] = hv > 0.f ? __fdiv_rn(__ldg(g + i), hv) : 0.f;
    if (zero_ghat) gh[i] = 0.f;
  }
}

cudaError_t launch_ratio(const float* g, float* ghat, float* r, long long count, bool zero_ghat, cudaStream_t s,
                         bool pdl) {
#ifndef CTIS_RATIO_BPS
#define CTIS_RATIO_BPS 4  // blocks of 256 threads per SM (8 / 16 without the unroll: 128.2 / 128.0 us)
#endif
  const long long want = (count / 4 + 255) / 256;
  const int blocks = (int)(want < 148 * CTIS_RATIO_BPS ? (want > 0 ? want : 1) : 148 * CTIS_RATIO_BPS);
  return launch_ex(ratio_kernel, blocks, 256, s, pdl, g, ghat, r, count, zero_ghat ? 1 : 0);
}

// Ratio over the reachable pixel box of each frame: float4 i of the box is rows
// r0 + 4*(i % nr4) .. +3 of column c0 + (i / nr4) % nc of frame i / (nr4 * nc); g_hat is reset to 0.
__global__ void ratio_box_kernel(const float* __restrict__ g, float* gh, float* r, long long n, int gamma, int r0,
                                 int nr4, int c0, int nc, long long total4) {
  pdl_enter();
  // blockIdx.y = frame; 32-bit index math within the frame (per_frame = nr4 * nc < 2^31); measured against
  // one flat grid with 64-bit divisions: C3 40.9 -> 40.4, T1w75 35.6 -> 35.1 us per MLEM iteration
  const unsigned per_frame = (unsigned)nr4 * (unsigned)nc;
  const long long fbase = (long long)blockIdx.y * n + (long long)c0 * gamma + r0;
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < per_frame; k += gridDim.x * blockDim.x) {
    const unsigned col = k / (unsigned)nr4;
    const long long p = fbase + (long long)col * gamma + 4 * (k - col * (unsigned)nr4);
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g + p));
    const float4 hv = *reinterpret_cast<const float4*>(gh + p);
    float4 o;
    o.x = hv.x > 0.f ? __fdiv_rn(gv.x, hv.x) : 0.f;
    o.y = hv.y > 0.f ? __fdiv_rn(gv.y, hv.y) : 0.f;
    o.z = hv.z > 0.f ? __fdiv_rn(gv.z, hv.z) : 0.f;
    o.w = hv.w > 0.f ? __fdiv_rn(gv.w, hv.w) : 0.f;
    *reinterpret_cast<float4*>(r + p) = o;
    *reinterpret_cast<float4*>(gh + p) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

cudaError_t launch_ratio_box(const float* g, float* ghat, float* r, long long n, int gamma, int r0, int nr4, int c0,
                             int nc, int frames, cudaStream_t s, bool pdl) {
  const long long total4 = (long long)nr4 * nc * frames;
  const long long per_frame = (long long)nr4 * nc;
  const long long want = (per_frame + 255) / 256;
  const long long cap = std::max<long long>(1, 148LL * 8 / std::max(1, frames));  // ~8 blocks per SM in all
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::max<long long>(1, std::min(want, cap)), (unsigned)frames);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ratio_box_kernel, g, ghat, r, n, gamma, r0, nr4, c0, nc, total4);
}

// Row repack of f for the TMA forward (plans with a % 4 != 0): one thread per element.
__global__ void repack_rows_kernel(const float* __restrict__ src, float* __restrict__ dst, int a, int pitch,
                                   long long cols) {
  pdl_enter();
  // one warp per column (lanes stride over its a rows): no integer division per element
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long c = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); c < cols; c += wstride)
    for (int r = lane; r < a; r += 32) dst[c * pitch + r] = __ldg(src + c * a + r);
}

cudaError_t launch_repack_rows(const float* src, float* dst, int a, int pitch, long long cols, cudaStream_t s) {
  const long long want = (cols + 7) / 8;  // 8 warps (columns) per block
  const int blocks = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
  return launch_ex(repack_rows_kernel, blocks, 256, s, false, src, dst, a, pitch, cols);
}

// Update pass of mode-split back projections (ctis_api.cu enqueue_back): the epilogue's arithmetic
// (ctis_tables.cu upd_value) on the accumulated z, which is re-zeroed for the next accumulation.
__global__ void split_update_kernel(float* f, float* z, const float* __restrict__ invh, int ell, int w,
                                    long long count, int mode) {
  pdl_enter();
  // blockIdx.y = frame, blockIdx.x strides over the frame's m = ell * w voxels with 32-bit band index math
  const unsigned m = (unsigned)ell * (unsigned)w;
  const long long base = (long long)blockIdx.y * m;
  for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    const long long j = base + k;
    const float ih = __ldg(invh + k / (unsigned)ell);
    const float zz = z[j];
    z[j] = 0.f;
    f[j] = mode == 1 ? f[j] * zz * ih : mode == 2 ? f[j] * expf(zz * ih) : zz;
  }
}

cudaError_t launch_split_update(float* f, float* z, const float* invh, int ell, int w, long long count, int mode,
                                cudaStream_t s) {
  const long long m = (long long)ell * w;
  const long long frames = m > 0 ? count / m : 0;
  if (frames < 1) return cudaSuccess;
  const long long want = (m + 255) / 256;
  const long long cap = std::max<long long>(1, 148LL * 8 / frames);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::max<long long>(1, std::min(want, cap)), (unsigned)frames);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, split_update_kernel, f, z, invh, ell, w, count, mode);
}

__global__ void sensitivity_kernel(const float* __restrict__ hband, float* __restrict__ h, int ell, int m) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) h[j] = __ldg(hband + j / ell);
}

cudaError_t launch_sensitivity(const float* hband, float* h, int ell, int m, cudaStream_t s) {
  const int want = (m + 255) / 256;
  const int blocks = want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8;
  sensitivity_kernel<<<blocks, 256, 0, s>>>(hband, h, ell, m);
  return cudaGetLastError();
}

__global__ void validate_kernel(const float* __restrict__ x, long long count, int* flag) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    const float v = __ldg(x + i);
    bad |= !(v >= 0.f && v <= 3.402823466e38f);
  }
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

cudaError_t launch_validate(const float* x, long long count, int* flag, cudaStream_t s) {
  const long long want = (count + 255) / 256;
  const int blocks = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
  validate_kernel<<<blocks, 256, 0, s>>>(x, count, flag);
  return cudaGetLastError();
}

// SMART log-ratio r_p = log(g_p / g_hat_p) where both are > 0, else 0 (R17); resets g_hat.
__global__ void log_ratio_kernel(const float* __restrict__ g, float* gh, float* r, long long count) {
  pdl_enter();
  auto one = [](float gv, float hv) { return (gv > 0.f && hv > 0.f) ? logf(__fdiv_rn(gv, hv)) : 0.f; };
  const bool aligned = ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(gh) |
                         reinterpret_cast<uintptr_t>(r)) & 15u) == 0;
  const long long n4 = aligned ? (count >> 2) : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long i = t0; i < n4; i += stride) {
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    const float4 hv = reinterpret_cast<const float4*>(gh)[i];
    reinterpret_cast<float4*>(r)[i] = make_float4(one(gv.x, hv.x), one(gv.y, hv.y), one(gv.z, hv.z), one(gv.w, hv.w));
    reinterpret_cast<float4*>(gh)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (long long i = 4 * n4 + t0; i < count; i += stride) {
    r[i] = one(__ldg(g + i), gh[i]);
    gh[i] = 0.f;
  }
}

cudaError_t launch_log_ratio(const float* g, float* ghat, float* r, long long count, cudaStream_t s, bool pdl) {
  const long long want = (count / 4 + 255) / 256;
  const int blocks = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
  return launch_ex(log_ratio_kernel, blocks, 256, s, pdl, g, ghat, r, count);
}

// Ratio + Poisson log-likelihood of the current model (R15): each thread accumulates its
// terms in fp64, the block reduces them (warp shuffles, then shared memory) and adds one value to
// ll[*counter] with a double-precision atomic.
__global__ void ratio_ll_kernel(const float* __restrict__ g, float* gh, float* r, long long count, double* ll,
                                const int* __restrict__ counter) {
  pdl_enter();
  double acc = 0.0;
  auto one = [&acc](float gv, float hv) -> float {
    if (hv > 0.f)
      acc += (double)gv * (double)logf(hv) - (double)hv;
    else if (gv > 0.f)
      acc = -INFINITY;
    return hv > 0.f ? __fdiv_rn(gv, hv) : 0.f;
  };
  const bool aligned = ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(gh) |
                         reinterpret_cast<uintptr_t>(r)) & 15u) == 0;
  const long long n4 = aligned ? (count >> 2) : 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long i = t0; i < n4; i += stride) {
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    const float4 hv = reinterpret_cast<const float4*>(gh)[i];
    const float rx = one(gv.x, hv.x), ry = one(gv.y, hv.y), rz = one(gv.z, hv.z), rw = one(gv.w, hv.w);
    reinterpret_cast<float4*>(r)[i] = make_float4(rx, ry, rz, rw);
    reinterpret_cast<float4*>(gh)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (long long i = 4 * n4 + t0; i < count; i += stride) {
    r[i] = one(__ldg(g + i), gh[i]);
    gh[i] = 0.f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double part[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) part[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    double v = lane < (int)(blockDim.x >> 5) ? part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) atomicAdd(ll + *counter, v);
  }
}

cudaError_t launch_ratio_ll(const float* g, float* ghat, float* r, long long count, double* ll, const int* counter,
                            cudaStream_t s, bool pdl) {
  const long long want = (count / 4 + 255) / 256;
  const int blocks = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
  return launch_ex(ratio_ll_kernel, blocks, 256, s, pdl, g, ghat, r, count, ll, counter);
}

// Stop rule after update k = *counter + 1 (R16), evaluated on the device: sets the WHILE
// node's condition so the graph itself decides whether the next iteration runs.
__global__ void mlem_check_kernel(const double* __restrict__ ll, int* counter, int max_iters, double rel_tol,
                                  cudaGraphConditionalHandle handle) {
  const int k = *counter + 1;
  *counter = k;
  bool stop = k >= max_iters;
  if (k >= 2 && ll[k - 1] - ll[k - 2] <= rel_tol * fabs(ll[k - 1])) stop = true;
  cudaGraphSetConditional(handle, stop ? 0u : 1u);
}

cudaError_t launch_mlem_check(const double* ll, int* counter, int max_iters, double rel_tol,
                              unsigned long long cond_handle, cudaStream_t s) {
  mlem_check_kernel<<<1, 1, 0, s>>>(ll, counter, max_iters, rel_tol, (cudaGraphConditionalHandle)cond_handle);
  return cudaGetLastError();
}

}  // namespace ctis
