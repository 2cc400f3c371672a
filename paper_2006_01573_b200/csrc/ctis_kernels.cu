// ctis_kernels.cu — sm_100a kernels of the CTIS MLEM hot path (first version).
//
//   forward  g_hat = H f          (Eqs. 8-13; Alg. 1 lines 6-7)
//   ratio    r = g (/) g_hat      (Alg. 1 line 8; fused into the forward epilogue)
//   back     z = H^T r            (Eqs. 14-17; Alg. 1 lines 9-11)
//   update   f <- f (.) z (/) h   (Eq. 2; Alg. 1 line 12; fused into the back kernel)
//
// The FFT route of the paper (Eqs. 13/17) is replaced by a direct sparse-tap
// evaluation of the same circulant products: see DESIGN.md §"Path".
#include <cuda_runtime.h>
#include <math.h>

#include "ctis_internal.h"

namespace ctis {

// ---------------------------------------------------------------------------
// Forward: one CTA per 64x16 FPA tile (x frames); each thread owns 2 rows x 2
// columns of the tile: rows lane, lane+32 (a warp covers 32 contiguous FPA
// rows => coalesced f loads and g/r stores), columns 2*warp, 2*warp+1.
// The CTA walks its (piece, tile) entries and accumulates w * f in fp32 registers
// over all bands and taps; the epilogue writes g_hat, or r = g / g_hat.
template <bool kRatio>
__global__ void __launch_bounds__(kFwdThreads)
forward_gather_kernel(const float* __restrict__ f, const FwdEntry* __restrict__ ent,
                      const int* __restrict__ tile_ptr, int tiles_r, int a, int gamma, int xi,
                      int m, int n, const float* __restrict__ g, float* __restrict__ out) {
  const int tile = blockIdx.x;
  const int frame = blockIdx.y;
  const int tr = tile % tiles_r, tc = tile / tiles_r;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R0 = tr * kFwdTileR + lane;
  const int C0 = tc * kFwdTileC + 2 * warp;
  const float* fb = f + (size_t)frame * m;
  float acc00 = 0.f, acc10 = 0.f, acc01 = 0.f, acc11 = 0.f;
  const int o00 = R0 + a * C0;
  const int e0 = __ldg(tile_ptr + tile), e1 = __ldg(tile_ptr + tile + 1);
  for (int e = e0; e < e1; ++e) {
    const int4 h0 = __ldg(reinterpret_cast<const int4*>(ent + e));
    const int4 h1 = __ldg(reinterpret_cast<const int4*>(ent + e) + 1);
    const int base = h0.x;
    const float w = __int_as_float(h0.y);
    const float* src = fb + base + o00;
    if (h1.z) {  // full tile
      acc00 = fmaf(w, __ldg(src), acc00);
      acc10 = fmaf(w, __ldg(src + 32), acc10);
      acc01 = fmaf(w, __ldg(src + a), acc01);
      acc11 = fmaf(w, __ldg(src + a + 32), acc11);
    } else {
      const int rR0 = h0.z, rR1 = h0.w, rC0 = h1.x, rC1 = h1.y;
      const bool r0 = (R0 >= rR0) & (R0 < rR1), r1 = (R0 + 32 >= rR0) & (R0 + 32 < rR1);
      const bool c0 = (C0 >= rC0) & (C0 < rC1), c1 = (C0 + 1 >= rC0) & (C0 + 1 < rC1);
      if (r0 & c0) acc00 = fmaf(w, __ldg(src), acc00);
      if (r1 & c0) acc10 = fmaf(w, __ldg(src + 32), acc10);
      if (r0 & c1) acc01 = fmaf(w, __ldg(src + a), acc01);
      if (r1 & c1) acc11 = fmaf(w, __ldg(src + a + 32), acc11);
    }
  }
  const size_t gb = (size_t)frame * n;
  auto emit = [&](int R, int C, float v) {
    if (R < gamma && C < xi) {
      const int p = R + gamma * C;
      if (kRatio) {
        const float gv = __ldg(g + gb + p);
        v = v > 0.f ? __fdiv_rn(gv, v) : 0.f;
      }
      out[gb + p] = v;
    }
  };
  emit(R0, C0, acc00);
  emit(R0 + 32, C0, acc10);
  emit(R0, C0 + 1, acc01);
  emit(R0 + 32, C0 + 1, acc11);
}

cudaError_t launch_forward(const Dims& d, const DevTables& t, const float* f, const float* g,
                           float* out, int frames, bool ratio, cudaStream_t s) {
  dim3 grid(t.tiles_r * t.tiles_c, frames);
  if (ratio)
    forward_gather_kernel<true><<<grid, kFwdThreads, 0, s>>>(f, t.fwd_entries, t.fwd_tile_ptr, t.tiles_r,
                                                            d.a, d.gamma, d.xi, d.m, d.n, g, out);
  else
    forward_gather_kernel<false><<<grid, kFwdThreads, 0, s>>>(f, t.fwd_entries, t.fwd_tile_ptr, t.tiles_r,
                                                             d.a, d.gamma, d.xi, d.m, d.n, g, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Back projection (+ fused multiplicative update): one thread per voxel (r, c)
// of a 32x8 spatial tile, for kBackBands consecutive bands.  The 1-D circulant
// index (r + gamma*c + o) mod n (Eq. 7 transposed) is evaluated exactly with a
// single conditional subtract (r + gamma*c < n and o < n).
template <int kMode>
__global__ void __launch_bounds__(kBackThreads)
back_kernel(const float* __restrict__ rr, float* __restrict__ fz, const int* __restrict__ band_ptr4,
            const int* __restrict__ band_cnt, const int* __restrict__ tap_off,
            const float* __restrict__ tap_w, const float* __restrict__ inv_h, int a, int alpha,
            int w, int gamma, int n, int m, int nchunks) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * kBackTileR + lane;
  const int c = blockIdx.y * kBackTileC + warp;
  const int chunk = blockIdx.z % nchunks, frame = blockIdx.z / nchunks;
  if (r >= a || c >= alpha) return;
  const float* rb = rr + (size_t)frame * n;
  float* fb = fz + (size_t)frame * m;
  const int base = r + gamma * c;
  const int ell = a * alpha;
  const int lam0 = chunk * kBackBands;
  const int lam1 = min(w, lam0 + kBackBands);
  for (int lam = lam0; lam < lam1; ++lam) {
    const int t0 = __ldg(band_ptr4 + lam);
    const int cnt = __ldg(band_cnt + lam);
    const int t4 = t0 + (cnt & ~3);
    float acc0 = 0.f, acc1 = 0.f;
    for (int t = t0; t < t4; t += 4) {
      const int4 o = __ldg(reinterpret_cast<const int4*>(tap_off + t));
      const float4 wv = __ldg(reinterpret_cast<const float4*>(tap_w + t));
      int i0 = base + o.x, i1 = base + o.y, i2 = base + o.z, i3 = base + o.w;
      i0 -= (i0 >= n) ? n : 0;
      i1 -= (i1 >= n) ? n : 0;
      i2 -= (i2 >= n) ? n : 0;
      i3 -= (i3 >= n) ? n : 0;
      acc0 = fmaf(wv.x, __ldg(rb + i0), acc0);
      acc1 = fmaf(wv.y, __ldg(rb + i1), acc1);
      acc0 = fmaf(wv.z, __ldg(rb + i2), acc0);
      acc1 = fmaf(wv.w, __ldg(rb + i3), acc1);
    }
    for (int t = t4; t < t0 + cnt; ++t) {
      int i0 = base + __ldg(tap_off + t);
      i0 -= (i0 >= n) ? n : 0;
      acc0 = fmaf(__ldg(tap_w + t), __ldg(rb + i0), acc0);
    }
    const float z = acc0 + acc1;
    const int j = lam * ell + c * a + r;
    if (kMode == kBackUpdate) {
      fb[j] = fb[j] * z * __ldg(inv_h + lam);
    } else {
      fb[j] = z;
    }
  }
}

cudaError_t launch_back(const Dims& d, const DevTables& t, const float* r, float* fz, int frames,
                        BackMode mode, cudaStream_t s) {
  const int nchunks = (d.w + kBackBands - 1) / kBackBands;
  dim3 grid((d.a + kBackTileR - 1) / kBackTileR, (d.alpha + kBackTileC - 1) / kBackTileC, nchunks * frames);
  if (mode == kBackUpdate)
    back_kernel<kBackUpdate><<<grid, kBackThreads, 0, s>>>(r, fz, t.band_ptr4, t.band_cnt, t.tap_off, t.tap_w,
                                                           t.inv_h, d.a, d.alpha, d.w, d.gamma, d.n, d.m,
                                                           nchunks);
  else
    back_kernel<kBackOnly><<<grid, kBackThreads, 0, s>>>(r, fz, t.band_ptr4, t.band_cnt, t.tap_off, t.tap_w,
                                                         t.inv_h, d.a, d.alpha, d.w, d.gamma, d.n, d.m,
                                                         nchunks);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Sensitivity h = H^T 1: every column of C_lam E sums to h_lam (P:39 with P:93-97).
__global__ void sensitivity_kernel(const float* __restrict__ hband, float* __restrict__ h, int ell, int m) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
    h[j] = __ldg(hband + j / ell);
}

cudaError_t launch_sensitivity(const Dims& d, const DevTables& t, float* h, cudaStream_t s) {
  const int blocks = min(148 * 8, (d.m + 255) / 256);
  sensitivity_kernel<<<blocks, 256, 0, s>>>(t.h, h, d.ell, d.m);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Ratio r = g (/) g_hat (Alg. 1 line 8), r = 0 where g_hat <= 0 (R4).
__global__ void ratio_kernel(const float* __restrict__ g, const float* __restrict__ gh, float* __restrict__ r,
                             int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = __ldg(gh + i);
    r[i] = v > 0.f ? __fdiv_rn(__ldg(g + i), v) : 0.f;
  }
}

cudaError_t launch_ratio(const float* g, const float* ghat, float* r, int64_t count, cudaStream_t s) {
  const int64_t want = (count + 255) / 256;
  const int blocks = (int)(want < 148 * 16 ? want : 148 * 16);
  ratio_kernel<<<blocks, 256, 0, s>>>(g, ghat, r, count);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Data validation: flag |= 1 if any element is negative, NaN or Inf.
__global__ void validate_kernel(const float* __restrict__ x, int64_t count, int* flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = __ldg(x + i);
    bad |= !(v >= 0.f && v <= 3.402823466e38f);
  }
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

cudaError_t launch_validate(const float* x, int64_t count, int* flag, cudaStream_t s) {
  const int64_t want = (count + 255) / 256;
  const int blocks = (int)(want < 148 * 8 ? (want > 0 ? want : 1) : 148 * 8);
  validate_kernel<<<blocks, 256, 0, s>>>(x, count, flag);
  return cudaGetLastError();
}

}  // namespace ctis
