// ctis_tables.cu — the two projection kernels of the CTIS MLEM hot path, compiled to a
// standalone sm_100a cubin that libctis embeds and loads once per plan and tap page
// (cudaLibraryLoadData), so that every plan owns private __constant__ tap tables.
//
//   forward  g_hat = H f = sum_lam C_lam E f_lam        (Eqs. 8-13; Alg. 1 l. 6-7)
//   back     z = H^T r,  f <- f (.) z (/) h              (Eqs. 14-17; Eq. 2; l. 9-12)
//
// Both evaluate the circulant products directly from the sparse first columns c_lam
// ("taps"): voxel q of band lam meets FPA pixel (E(q) + o) mod n with weight w
// for every tap (o, w) of c_lam.  Writing o = o_ref + dr + gamma*dc for a per-chunk
// "mode" reference o_ref (taps of consecutive bands that drift together, e.g. one
// diffraction order) turns each tap into a small 2-D shift (dr, dc) of the field stop:
//   E(q) + o = E(q + (dr, dc)) + o_ref   (exact integer identity, so the 1-D cyclic
//   wrap of Eq. 7 is reproduced exactly by reducing the final index mod n).
//
// forward ("constellation"): a CTA owns a 32 x 16 tile of u = q + (dr, dc) space and ALL
//   modes of a chunk of bands.  Per band it stages one shared-memory window of f_lam
//   (cp.async, zero outside the field stop) that every mode reads, accumulates
//   acc[mode] += w * f_lam[u - (dr, dc)] in registers, and finally adds acc[mode] to
//   g_hat[(E(u) + o_ref) mod n] with red.global.add.f32 (chunks of bands overlap there).
// back: a CTA owns a 32 x 32 voxel tile and a chunk of 16 bands; per mode it stages one
//   shared-memory window of r (1-D modular addressing, exact wrap) that every band of the
//   chunk reads, accumulates z[band] for 2 voxels per thread in registers, and fuses the
//   multiplicative update f <- f * z * (1/h_lam) into the epilogue.
// Tap metadata (window offsets, weights) is read from __constant__ through the uniform
// datapath (LDCU + FFMA R,R,UR,R): the only per-FMA shared-memory traffic is the operand.
#include <stdint.h>

#include "ctis_internal.h"

using namespace ctis;

__constant__ uint32_t c_tab[kPageWords];

namespace {

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ int tabi(uint32_t i) { return (int)c_tab[i]; }
__device__ __forceinline__ float tabf(uint32_t i) { return __uint_as_float(c_tab[i]); }

// Window loaders.  A window is WR x WC floats (WR <= 64, WR % 4 == 0 on the 16-byte path),
// stored column by column with pitch WR.  Lanes 0-15 copy 16 four-float chunks of one window
// column, lanes 16-31 the next column, so a warp covers two columns per pass (32-bit math only).

// f_lam window: element (i, j) = f_lam[(row0 + i) + a*(col0 + j)], zero outside the field stop.
template <int NWARPS, bool VEC>
__device__ __forceinline__ void load_f_window(float* buf, const float* fl, const TabArgs& A, int row0, int col0,
                                              int WR, int WC) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (VEC) {
    const int i = (lane & 15) * 4, rr = row0 + i;
    const bool rok = (i < WR) & (rr >= 0) & (rr < A.a);
    for (int j = 2 * warp + (lane >> 4); j < WC; j += 2 * NWARPS) {
      const int cc = col0 + j;
      const bool ok = rok & (cc >= 0) & (cc < A.alpha);
      if (i < WR) cp_async16(buf + i + WR * j, ok ? fl + rr + A.a * cc : fl, ok);
    }
  } else {
    for (int j = warp; j < WC; j += NWARPS) {
      const int cc = col0 + j;
      const bool cok = (cc >= 0) & (cc < A.alpha);
      for (int i = lane; i < WR; i += 32) {
        const int rr = row0 + i;
        const bool ok = cok & (rr >= 0) & (rr < A.a);
        cp_async4(buf + i + WR * j, ok ? fl + rr + A.a * cc : fl, ok);
      }
    }
  }
}

// r window: element (i, j) = r[(B + i + gamma*j) mod n]  (0 <= B < n).
template <int NWARPS, bool VEC>
__device__ __forceinline__ void load_r_window(float* buf, const float* r, const TabArgs& A, unsigned B, int WR,
                                              int WC) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned n = (unsigned)A.n;
  if (VEC) {
    const int i = (lane & 15) * 4;
    if (i >= WR) return;
    const int j0 = 2 * warp + (lane >> 4);
    unsigned cb = B + (unsigned)A.gamma * (unsigned)j0;
    while (cb >= n) cb -= n;
    const unsigned step = (unsigned)A.gamma * (2u * NWARPS);
    for (int j = j0; j < WC; j += 2 * NWARPS) {
      unsigned idx = cb + (unsigned)i;
      while (idx >= n) idx -= n;
      cp_async16(buf + i + WR * j, r + idx, true);
      cb += step;
      while (cb >= n) cb -= n;
    }
  } else {
    for (int j = warp; j < WC; j += NWARPS) {
      unsigned cb = B + (unsigned)((unsigned long long)A.gamma * (unsigned)j % n);
      while (cb >= n) cb -= n;
      for (int i = lane; i < WR; i += 32) {
        unsigned idx = cb + (unsigned)i;
        while (idx >= n) idx -= n;
        cp_async4(buf + i + WR * j, r + idx, true);
      }
    }
  }
}

__device__ __forceinline__ float lds(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

template <int MAXM, bool VEC>
__device__ __forceinline__ void forward_body(const TabArgs& A) {
  extern __shared__ __align__(16) float smem[];
  const uint32_t D = c_tab[1 + blockIdx.y];
  const int lam0 = tabi(D + 0), nb = tabi(D + 1), nm = tabi(D + 2);
  const int u_r0 = tabi(D + 3), u_c0 = tabi(D + 4), tiles_r = tabi(D + 5), tiles_c = tabi(D + 6);
  const int tile = blockIdx.x;
  if (tile >= tiles_r * tiles_c) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int U_r = u_r0 + (tile % tiles_r) * kFwdTR, U_c = u_c0 + (tile / tiles_r) * kFwdTC;
  const float* f = A.src + (long long)blockIdx.z * A.src_frame;
  const uint32_t BI = D + kDescHeader + nm, TP = BI + 4 * nb;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);

  float acc[MAXM];
#pragma unroll
  for (int c = 0; c < MAXM; ++c) acc[c] = 0.f;

  auto issue = [&](int b) {
    if (b < nb) {
      const uint32_t bi = BI + 4 * b;
      load_f_window<kFwdThreads / 32, VEC>(smem + (b % kStages) * kFwdWinFloats, f + (long long)(lam0 + b) * A.ell, A,
                                           U_r + tabi(bi + 0), U_c + tabi(bi + 1), tabi(bi + 2), tabi(bi + 3));
    }
    cp_commit();  // one (possibly empty) group per band keeps the group arithmetic uniform
  };
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) issue(s);
  for (int b = 0; b < nb; ++b) {
    issue(b + kStages - 1);
    cp_wait<kStages - 1>();
    __syncthreads();
    // byte address of this thread's u in the window; tap entries hold byte offsets (absent: w = 0)
    const unsigned base = sbase + 4u * ((b % kStages) * kFwdWinFloats + lane + tabi(BI + 4 * b + 2) * warp);
    // pointer arithmetic (not an unsigned index) lets ptxas fold 8*c into LDCU.64 c[0x3][UR+imm]
    const uint2* ent = reinterpret_cast<const uint2*>(c_tab + TP) + b * MAXM;
#pragma unroll
    for (int c = 0; c < MAXM; ++c) {
      const uint2 e = ent[c];
      acc[c] = fmaf(__uint_as_float(e.y), lds(base + e.x), acc[c]);
    }
    __syncthreads();
  }
  float* g = A.dst + (long long)blockIdx.z * A.dst_frame;
  const long long ub = (long long)(U_r + lane) + (long long)A.gamma * (U_c + warp);
#pragma unroll
  for (int c = 0; c < MAXM; ++c) {
    if (c < nm && acc[c] != 0.f) {
      long long P = (ub + tabi(D + kDescHeader + c)) % A.n;
      if (P < 0) P += A.n;
      atomicAdd(g + P, acc[c]);
    }
  }
}

template <int NB, bool VEC>
__device__ __forceinline__ void back_body(const TabArgs& A) {
  extern __shared__ __align__(16) float smem[];
  const uint32_t D = c_tab[1 + blockIdx.y];
  const int lam0 = tabi(D + 0), nb = tabi(D + 1), nm = tabi(D + 2);
  const int tiles_r = tabi(D + 3), tiles_c = tabi(D + 4);
  const int tile = blockIdx.x;
  if (tile >= tiles_r * tiles_c) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q_r0 = (tile % tiles_r) * kBackTR, q_c0 = (tile / tiles_r) * kBackTC;
  const float* r = A.src + (long long)blockIdx.z * A.src_frame;
  const uint32_t MI = D + kDescHeader, TP = MI + 4 * nm, IH = TP + 2 * nm * NB;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned tile1d = (unsigned)(q_r0 + A.gamma * q_c0);  // < n

  float acc0[NB], acc1[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) acc0[b] = acc1[b] = 0.f;

  auto origin = [&](int c) {
    unsigned B = tile1d + c_tab[MI + 4 * c];
    while (B >= (unsigned)A.n) B -= (unsigned)A.n;
    return B;
  };
  auto issue = [&](int c) {
    if (c < nm)
      load_r_window<kBackThreads / 32, VEC>(smem + (c % kStages) * kBackWinFloats, r, A, origin(c),
                                            tabi(MI + 4 * c + 1), tabi(MI + 4 * c + 2));
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) issue(s);
  for (int c = 0; c < nm; ++c) {
    issue(c + kStages - 1);
    cp_wait<kStages - 1>();
    __syncthreads();
    const int WR = tabi(MI + 4 * c + 1);
    const unsigned b0a = sbase + 4u * ((c % kStages) * kBackWinFloats + lane + WR * warp);
    const unsigned b1a = b0a + 4u * WR * (kBackThreads / 32);
    const uint2* ent = reinterpret_cast<const uint2*>(c_tab + TP) + c * NB;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint2 e = ent[b];
      const float w = __uint_as_float(e.y);
      acc0[b] = fmaf(w, lds(b0a + e.x), acc0[b]);
      acc1[b] = fmaf(w, lds(b1a + e.x), acc1[b]);
    }
    __syncthreads();
  }
  float* f = A.dst + (long long)blockIdx.z * A.dst_frame;
  const int qr = q_r0 + lane, qc0 = q_c0 + warp, qc1 = qc0 + kBackThreads / 32;
  if (qr >= A.a) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b < nb) {
      const long long lb = (long long)(lam0 + b) * A.ell + qr;
      const float ih = tabf(IH + b);
      if (qc0 < A.alpha) {
        float* p = f + lb + (long long)A.a * qc0;
        *p = A.mode ? (*p) * acc0[b] * ih : acc0[b];
      }
      if (qc1 < A.alpha) {
        float* p = f + lb + (long long)A.a * qc1;
        *p = A.mode ? (*p) * acc1[b] * ih : acc1[b];
      }
    }
  }
}

}  // namespace

#define CTIS_FWD(M, V, NAME) \
  extern "C" __global__ void __launch_bounds__(kFwdThreads, 1) NAME(const TabArgs A) { forward_body<M, V>(A); }
CTIS_FWD(8, true, ctis_fwd_m8_v)
CTIS_FWD(8, false, ctis_fwd_m8_s)
CTIS_FWD(16, true, ctis_fwd_m16_v)
CTIS_FWD(16, false, ctis_fwd_m16_s)
CTIS_FWD(24, true, ctis_fwd_m24_v)
CTIS_FWD(24, false, ctis_fwd_m24_s)
CTIS_FWD(32, true, ctis_fwd_m32_v)
CTIS_FWD(32, false, ctis_fwd_m32_s)
CTIS_FWD(40, true, ctis_fwd_m40_v)
CTIS_FWD(40, false, ctis_fwd_m40_s)
CTIS_FWD(48, true, ctis_fwd_m48_v)
CTIS_FWD(48, false, ctis_fwd_m48_s)
CTIS_FWD(56, true, ctis_fwd_m56_v)
CTIS_FWD(56, false, ctis_fwd_m56_s)
CTIS_FWD(64, true, ctis_fwd_m64_v)
CTIS_FWD(64, false, ctis_fwd_m64_s)
CTIS_FWD(72, true, ctis_fwd_m72_v)
CTIS_FWD(72, false, ctis_fwd_m72_s)
CTIS_FWD(80, true, ctis_fwd_m80_v)
CTIS_FWD(80, false, ctis_fwd_m80_s)
CTIS_FWD(88, true, ctis_fwd_m88_v)
CTIS_FWD(88, false, ctis_fwd_m88_s)
CTIS_FWD(96, true, ctis_fwd_m96_v)
CTIS_FWD(96, false, ctis_fwd_m96_s)

#define CTIS_BACK(NB, V, NAME) \
  extern "C" __global__ void __launch_bounds__(kBackThreads, 2) NAME(const TabArgs A) { back_body<NB, V>(A); }
CTIS_BACK(4, true, ctis_back_b4_v)
CTIS_BACK(4, false, ctis_back_b4_s)
CTIS_BACK(8, true, ctis_back_b8_v)
CTIS_BACK(8, false, ctis_back_b8_s)
CTIS_BACK(12, true, ctis_back_b12_v)
CTIS_BACK(12, false, ctis_back_b12_s)
CTIS_BACK(16, true, ctis_back_b16_v)
CTIS_BACK(16, false, ctis_back_b16_s)
