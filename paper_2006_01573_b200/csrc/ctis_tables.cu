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
//   modes of a chunk of bands.  Per band it stages one shared-memory window of f_lam that
//   every mode reads, accumulates acc[mode] += w * f_lam[u - (dr, dc)] in registers, and
//   finally adds acc[mode] to g_hat[(E(u) + o_ref) mod n] with red.global.add.f32.
// back: a CTA owns a 32 x 32 voxel tile and a chunk of NB bands; per mode it stages one
//   shared-memory window of r (exact 1-D modular addressing) that every band of the chunk
//   reads, accumulates z[band] for 2 voxels per thread in registers, and fuses the
//   multiplicative update f <- f * z * (1/h_lam) into the epilogue.
// Windows are moved by TMA (cp.async.bulk.tensor, one elected thread, mbarrier completion,
// zero fill outside the field stop) through a kStages-deep ring; geometries whose strides are
// not 16-byte multiples (and r windows that wrap around the FPA) use a cp.async element loader.
// Tap metadata (byte offsets into the window, weights) is read from __constant__ through the
// uniform datapath (LDCU; LDS [R+UR]; FFMA R,R,UR,R): no per-tap address arithmetic.
#include <cuda.h>
#include <stdint.h>

#include <utility>

#include "ctis_internal.h"

using namespace ctis;

// 16-byte aligned so that tap entries (uint2 at even word offsets) load as one LDCU.64
__constant__ __align__(16) uint32_t c_tab[kPageWords];
// Tap entries are 16-byte pairs (off0, off1, w0, w1) at word offsets that are multiples of 4.
__device__ __forceinline__ const uint4* tab4(uint32_t word4) {
  return reinterpret_cast<const uint4*>(c_tab) + (word4 >> 2);
}

namespace {

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool valid, bool cg = false) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (cg) {  // experiment: L1-bypassing synchronous load
    float v = 0.f;
    if (valid) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(gmem) : "memory");
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(s), "f"(v) : "memory");
    return;
  }
  const int sz = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ int tabi(uint32_t i) { return (int)c_tab[i]; }

// Back-projection epilogue (TabArgs::mode): 0 z = H^T r; 1 MLEM f <- f * z / h (Eq. 2, Alg. 1 l. 12);
// 2 SMART f <- f * exp(z / h) with r the log-ratio (R17); 3 z += partial H^T r (red.add: mode-split
// plans, the update runs as a separate pass)
__device__ __forceinline__ float upd_value(int mode, float f, float z, float ih) {
  return mode == 1 ? f * z * ih : mode == 2 ? f * expf(z * ih) : z;
}
__device__ __forceinline__ float tabf(uint32_t i) { return __uint_as_float(c_tab[i]); }

__device__ __forceinline__ float lds(unsigned addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// ---- mbarrier / TMA helpers -----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// non-blocking probe of an mbarrier phase (true once the phase with this parity has completed)
__device__ __forceinline__ bool mbar_test(unsigned bar, unsigned parity) {
  unsigned r;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(r)
      : "r"(bar), "r"(parity)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ unsigned atom_add_shared(unsigned addr, unsigned v) {
  unsigned old;
  asm volatile("atom.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_shared_u32(unsigned addr, unsigned v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_shared_u32(unsigned addr) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
// slot release counter: release orders this warp's reads of the slot before the increment, acquire
// makes every earlier release (the other warps' reads) visible to the warp that completes the count
__device__ __forceinline__ unsigned atom_add_acqrel_shared(unsigned addr, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tma_3d(unsigned dst, const CUtensorMap* tm, int c0, int c1, int c2, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_4d(unsigned dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                       unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

// ---- element loaders (cp.async, 4 bytes) ----------------------------------------------------
// f_lam window: element (i, j) = f_lam[(row0 + i) + a*(col0 + j)], zero outside the field stop.
template <int NWARPS>
__device__ __forceinline__ void load_f_window(float* buf, const float* fl, const TabArgs& A, int row0, int col0,
                                              int WR, int WC) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < WC; j += NWARPS) {
    const int cc = col0 + j;
    const bool cok = (cc >= 0) & (cc < A.alpha);
    for (int i = lane; i < WR; i += 32) {
      const int rr = row0 + i;
      const bool ok = cok & (rr >= 0) & (rr < A.a);
      cp_async4(buf + i + WR * j, ok ? fl + rr + A.a * cc : fl, ok, A.dbg & 4);
    }
  }
}

// r window: element (i, j) = r[(B + i + gamma*j) mod n]  (0 <= B < n).
template <int NWARPS>
__device__ __forceinline__ void load_r_window(float* buf, const float* r, const TabArgs& A, unsigned B, int WR,
                                              int WC) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned n = (unsigned)A.n;
  for (int j = warp; j < WC; j += NWARPS) {
    unsigned cb = B + (unsigned)((unsigned long long)A.gamma * (unsigned)j % n);
    while (cb >= n) cb -= n;
    for (int i = lane; i < WR; i += 32) {
      unsigned idx = cb + (unsigned)i;
      while (idx >= n) idx -= n;
      cp_async4(buf + i + WR * j, r + idx, true, A.dbg & 4);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Forward.  TMA: f viewed as a 4-D tensor {a, alpha, w, frames}; the window box {WRbox, WCbox, 1, 1}
// starts at (U_r + row0_rel, U_c + col0_rel, lam, frame); out-of-bounds elements are zero.
// G groups of 16 warps share every window; group GRP owns modes [GRP*MAXM, (GRP+1)*MAXM) of the
// pass.  GRP is a template parameter (dispatched on a warp-uniform branch) so that the tap-table
// pointer stays uniform and the entries load through LDCU.64 rather than per-thread LDC.
template <int G, int MAXM, bool TMA, int GRP, bool PAIR>
__device__ __forceinline__ void forward_group(const TabArgs& A, const CUtensorMap* tm) {
  extern __shared__ __align__(128) float smem[];
  constexpr int S = kFwdStages;
  constexpr int NWARPS = G * kFwdThreads / 32;
  const uint32_t D = c_tab[1 + blockIdx.y];
  const int lam0 = tabi(D + 0), nb = tabi(D + 1), nm = tabi(D + 2);
  const int u_r0 = tabi(D + 3), u_c0 = tabi(D + 4), tiles_r = tabi(D + 5), tiles_c = tabi(D + 6);
  const int tile = blockIdx.x;
  if (tile >= tiles_r * tiles_c) return;
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 15;
  constexpr int grp = GRP;
  const int U_r = u_r0 + (tile % tiles_r) * kFwdTR, U_c = u_c0 + (tile / tiles_r) * kFwdTC;
  const float* f = A.src + (long long)blockIdx.z * A.src_frame;
  const uint32_t BI = D + kDescHeader + ((nm + 3) & ~3), TP = BI + 4 * nb;  // TP % 4 == 0
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned full = sbase + S * A.slot_floats * 4u;  // S "full" mbarriers, then S release counters
  const unsigned empty = full + 8 * S;
  constexpr int MP = MAXM / 2;  // mode pairs: one FFMA2 (fp32x2) per pair

  float2 acc[MP];
#pragma unroll
  for (int k = 0; k < MP; ++k) acc[k] = make_float2(0.f, 0.f);
  // one band: acc[mode] += w * window[u - shift(mode)]; entries hold byte offsets (absent: w = 0).
  // Pointer arithmetic lets ptxas fold the entry offset into LDCU.64 c[0x3][UR+imm]; the weight
  // pair feeds FFMA2 R, R.F32x2, UR.F32x2, R.F32x2 straight from the uniform registers.
  auto compute = [&](unsigned base, int b) {
    if (PAIR) {
      const uint4* ent = tab4(TP) + (b * G + grp) * MP;
#pragma unroll
      for (int k = 0; k < MP; ++k) {
        const uint4 e = ent[k];
        const float2 x = make_float2(lds(base + e.x), lds(base + e.y));
        acc[k] = __ffma2_rn(make_float2(__uint_as_float(e.z), __uint_as_float(e.w)), x, acc[k]);
      }
    } else {  // plain FFMA, 8-byte (offset, weight) entries
      const uint2* ent = reinterpret_cast<const uint2*>(tab4(TP)) + (b * G + grp) * MAXM;
#pragma unroll
      for (int k = 0; k < MP; ++k) {
        const uint2 e0 = ent[2 * k], e1 = ent[2 * k + 1];
        acc[k].x = fmaf(__uint_as_float(e0.y), lds(base + e0.x), acc[k].x);
        acc[k].y = fmaf(__uint_as_float(e1.y), lds(base + e1.x), acc[k].y);
      }
    }
  };

  if (TMA) {
    // Full/empty mbarrier ring: thread 0 produces TMA boxes, every warp consumes and releases;
    // warps only wait for data, never for each other.
    auto issue = [&](int b) {
      const int slot = b % S;
      const uint32_t bi = BI + 4 * b;
      mbar_expect_tx(full + 8 * slot, A.box_bytes);
      tma_4d(sbase + 4u * slot * A.slot_floats, tm, U_r + tabi(bi + 0), U_c + tabi(bi + 1), lam0 + b,
             (int)blockIdx.z, full + 8 * slot);
    };
    // Batched refills: S = 2K slots; every K bands one CTA barrier (all warps are done with the
    // previous K bands), then thread 0 issues the next K boxes.  The tap loop itself has no
    // spinning producer and no atomics, so its control flow stays warp-uniform; it handles two
    // bands per trip (K is even) to amortise the per-trip bookkeeping over 2*MAXM taps.
    constexpr int K = S / 2;
    static_assert(K % 2 == 0, "two bands per trip");
    if (threadIdx.x == 0) {
      for (int s = 0; s < S; ++s) mbar_init(full + 8 * s, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (!(A.dbg & 1))
        for (int b = 0; b < S && b < nb; ++b) issue(b);
    }
    __syncthreads();
    const unsigned tbase = sbase + 4u * (lane + A.box_r * warp);
    const unsigned slot_bytes = 4u * A.slot_floats;
    int slot = 0;
    unsigned phase = 0;
    int b = 0;
    for (; b + 1 < nb; b += 2) {
      if (b >= K && b % K == 0) {
        __syncthreads();
        if (threadIdx.x == 0 && !(A.dbg & 1)) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (b + K + k < nb) issue(b + K + k);
        }
      }
      if (!(A.dbg & 1)) {
        mbar_wait(full + 8 * slot, phase);
        mbar_wait(full + 8 * (slot + 1), phase);
      }
      compute(tbase + slot * slot_bytes, b);
      compute(tbase + (slot + 1) * slot_bytes, b + 1);
      slot += 2;
      if (slot == S) {
        slot = 0;
        phase ^= 1u;
      }
    }
    if (b < nb) {  // odd band count: last band alone (its box was issued by the last refill)
      if (b >= K && b % K == 0) {
        __syncthreads();
        if (threadIdx.x == 0 && !(A.dbg & 1) && b + K < nb) issue(b + K);
      }
      if (!(A.dbg & 1)) mbar_wait(full + 8 * slot, phase);
      compute(tbase + slot * slot_bytes, b);
    }
  } else {
    auto issue = [&](int b) {
      if (b < nb) {
        const uint32_t bi = BI + 4 * b;
        load_f_window<NWARPS>(smem + (b % S) * A.slot_floats, f + (long long)(lam0 + b) * A.ell, A,
                              U_r + tabi(bi + 0), U_c + tabi(bi + 1), tabi(bi + 2), tabi(bi + 3));
      }
      cp_commit();  // one (possibly empty) group per band keeps the group arithmetic uniform
    };
#pragma unroll
    for (int s = 0; s < S - 1; ++s) issue(s);
    for (int b = 0; b < nb; ++b) {
      issue(b + S - 1);
      cp_wait<S - 1>();
      __syncwarp();  // the loader's per-lane trip counts diverge: reconverge before the aligned barrier
      __syncthreads();
      // a band without taps in this pass has an empty window (WC = 0): nothing was loaded into its
      // slot, so it must not be read (stale shared memory may hold NaN/Inf, and 0 * NaN != 0)
      if (tabi(BI + 4 * b + 3) != 0) compute(sbase + 4u * ((b % S) * A.slot_floats + lane + tabi(BI + 4 * b + 2) * warp), b);
      __syncthreads();  // every thread is done with this slot before it is refilled
    }
  }
  // flush: g_hat[(E(u) + o_ref) mod n] += acc.  E(u) = u_r + gamma*u_c can be negative (u reaches
  // kModeSpanMax outside the field stop); the host-chosen bias (a multiple of n) makes it >= 0, and
  // the sum stays far below 2^32 (n < 2^30 is enforced at plan creation).
  float* g = A.dst + (long long)blockIdx.z * A.dst_frame;
  const unsigned n = (unsigned)A.n;
  const int ue = (U_r + lane) + A.gamma * (U_c + warp);
  if (A.dbg & 2) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < MP; ++k) t += acc[k].x + acc[k].y;
    if (t == -1.f) g[0] = t;
    return;
  }
  unsigned ub = (unsigned)ue + A.bias;  // reduce E(u) mod n once per thread ...
  for (int k = 0; k < A.nsub; ++k) ub = min(ub, ub - n);
#pragma unroll
  for (int c = 0; c < MAXM; ++c) {
    const float v = (c & 1) ? acc[c >> 1].y : acc[c >> 1].x;
    if (grp * MAXM + c < nm && v != 0.f) {
      unsigned P = ub + c_tab[D + kDescHeader + grp * MAXM + c];  // ... then once per mode: < 2n
      P = min(P, P - n);
      atomicAdd(g + P, v);
    }
  }
}

template <int G, int MAXM, bool TMA, bool PAIR>
__device__ __forceinline__ void forward_body(const TabArgs& A, const CUtensorMap* tm) {
  if (G == 2 && threadIdx.x >= kFwdThreads)
    forward_group<G, MAXM, TMA, (G == 2 ? 1 : 0), PAIR>(A, tm);
  else
    forward_group<G, MAXM, TMA, 0, PAIR>(A, tm);
}

// ------------------------------------------------------------------------------------------------
// Back.  TMA: r viewed as a 3-D tensor {gamma, xi, frames}; a window whose 1-D origin B = (R0, C0)
// on the FPA fits without carry/wrap (R0 + WRbox <= gamma, C0 + WCbox <= xi) is one box load; any
// other window (cyclic wrap of Eq. 7) is loaded element by element with exact modular indices.
template <int NB, bool TMA, bool PAIR>
__device__ __forceinline__ void back_body(const TabArgs& A, const CUtensorMap* tm) {
  extern __shared__ __align__(128) float smem[];
  constexpr int S = kBackStages;
  constexpr int NWARPS = kBackThreads / 32;
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
  const unsigned full = sbase + S * A.slot_floats * 4u;
  const unsigned empty = full + 8 * S;

  // Window origin on the FPA: B = (tile1d + Bm) mod n as (R0, C0), from the host-split
  // Bm = Bm_r + gamma*Bm_c with one carry and one wrap (no division).
  auto origin_rc = [&](int c, int& R0, int& C0) {
    R0 = q_r0 + tabi(MI + 4 * c + 0);
    C0 = q_c0 + tabi(MI + 4 * c + 1);
    if (R0 >= A.gamma) {
      R0 -= A.gamma;
      C0 += 1;
    }
    if (C0 >= A.xi) C0 -= A.xi;
  };
  constexpr int BP = NB / 2;  // band pairs: one FFMA2 (fp32x2) per pair and voxel
  float2 acc0[BP], acc1[BP];
#pragma unroll
  for (int k = 0; k < BP; ++k) acc0[k] = acc1[k] = make_float2(0.f, 0.f);
  // one mode: z[band] += w * window[q + shift(mode, band)] for 2 voxels (columns warp, warp+16)
  auto compute = [&](unsigned b0a, unsigned b1a, int c) {
    if (PAIR) {
      const uint4* ent = tab4(TP) + c * BP;
#pragma unroll
      for (int k = 0; k < BP; ++k) {
        const uint4 e = ent[k];
        const float2 w = make_float2(__uint_as_float(e.z), __uint_as_float(e.w));
        acc0[k] = __ffma2_rn(w, make_float2(lds(b0a + e.x), lds(b0a + e.y)), acc0[k]);
        acc1[k] = __ffma2_rn(w, make_float2(lds(b1a + e.x), lds(b1a + e.y)), acc1[k]);
      }
    } else {  // plain FFMA, 8-byte (offset, weight) entries
      const uint2* ent = reinterpret_cast<const uint2*>(tab4(TP)) + c * NB;
#pragma unroll
      for (int k = 0; k < BP; ++k) {
        const uint2 e0 = ent[2 * k], e1 = ent[2 * k + 1];
        const float w0 = __uint_as_float(e0.y), w1 = __uint_as_float(e1.y);
        acc0[k].x = fmaf(w0, lds(b0a + e0.x), acc0[k].x);
        acc1[k].x = fmaf(w0, lds(b1a + e0.x), acc1[k].x);
        acc0[k].y = fmaf(w1, lds(b0a + e1.x), acc0[k].y);
        acc1[k].y = fmaf(w1, lds(b1a + e1.x), acc1[k].y);
      }
    }
  };

  // TMA is usable when every window of this tile is a plain FPA box (no carry / wrap of Eq. 7)
  bool boxes = TMA;
  if (TMA) {
    for (int c = 0; c < nm && boxes; ++c) {
      int R0, C0;
      origin_rc(c, R0, C0);
      boxes = (R0 + A.box_r <= A.gamma) && (C0 + A.box_c <= A.xi);
    }
  }
  if (TMA && boxes) {
    auto issue = [&](int c) {
      const int slot = c % S;
      int R0, C0;
      origin_rc(c, R0, C0);
      mbar_expect_tx(full + 8 * slot, A.box_bytes);
      tma_3d(sbase + 4u * slot * A.slot_floats, tm, R0, C0, (int)blockIdx.z, full + 8 * slot);
    };
    constexpr int K = S / 2;  // batched refills and two modes per trip, as in the forward kernel
    static_assert(K % 2 == 0, "two modes per trip");
    if (threadIdx.x == 0) {
      for (int s = 0; s < S; ++s) mbar_init(full + 8 * s, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (!(A.dbg & 1))
        for (int c = 0; c < S && c < nm; ++c) issue(c);
    }
    __syncthreads();
    const unsigned t0 = sbase + 4u * (lane + A.box_r * warp), t1 = t0 + 4u * A.box_r * NWARPS;
    const unsigned slot_bytes = 4u * A.slot_floats;
    int slot = 0;
    unsigned phase = 0;
    int c = 0;
    for (; c + 1 < nm; c += 2) {
      if (c >= K && c % K == 0) {
        __syncthreads();
        if (threadIdx.x == 0 && !(A.dbg & 1)) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (c + K + k < nm) issue(c + K + k);
        }
      }
      if (!(A.dbg & 1)) {
        mbar_wait(full + 8 * slot, phase);
        mbar_wait(full + 8 * (slot + 1), phase);
      }
      compute(t0 + slot * slot_bytes, t1 + slot * slot_bytes, c);
      compute(t0 + (slot + 1) * slot_bytes, t1 + (slot + 1) * slot_bytes, c + 1);
      slot += 2;
      if (slot == S) {
        slot = 0;
        phase ^= 1u;
      }
    }
    if (c < nm) {
      if (c >= K && c % K == 0) {
        __syncthreads();
        if (threadIdx.x == 0 && !(A.dbg & 1) && c + K < nm) issue(c + K);
      }
      if (!(A.dbg & 1)) mbar_wait(full + 8 * slot, phase);
      compute(t0 + slot * slot_bytes, t1 + slot * slot_bytes, c);
    }
  } else {
    // element loads with exact modular indices (wrapped windows, unaligned geometries)
    const int fixed_r = TMA ? A.box_r : 0, fixed_c = TMA ? A.box_c : 0;
    auto issue = [&](int c) {
      if (c < nm) {
        int R0, C0;
        origin_rc(c, R0, C0);
        const unsigned B = (unsigned)R0 + (unsigned)A.gamma * (unsigned)C0;
        load_r_window<NWARPS>(smem + (c % S) * A.slot_floats, r, A, B, TMA ? fixed_r : tabi(MI + 4 * c + 2),
                              TMA ? fixed_c : tabi(MI + 4 * c + 3));
      }
      cp_commit();
    };
#pragma unroll
    for (int s = 0; s < S - 1; ++s) issue(s);
    for (int c = 0; c < nm; ++c) {
      issue(c + S - 1);
      cp_wait<S - 1>();
      __syncwarp();  // reconverge after the loader's divergent loops (aligned barrier next)
      __syncthreads();
      const int WR = TMA ? fixed_r : tabi(MI + 4 * c + 2);
      const unsigned b0a = sbase + 4u * ((c % S) * A.slot_floats + lane + WR * warp);
      compute(b0a, b0a + 4u * WR * NWARPS, c);
      __syncthreads();
    }
  }
  float* f = A.dst + (long long)blockIdx.z * A.dst_frame;
  const int qr = q_r0 + lane, qc0 = q_c0 + warp, qc1 = qc0 + NWARPS;
  if (qr >= A.a) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b < nb) {
      const long long lb = (long long)(lam0 + b) * A.ell + qr;
      const float ih = tabf(IH + b);
      const float z0 = (b & 1) ? acc0[b >> 1].y : acc0[b >> 1].x;
      const float z1 = (b & 1) ? acc1[b >> 1].y : acc1[b >> 1].x;
      if (qc0 < A.alpha) {
        float* p = f + lb + (long long)A.a * qc0;
        *p = upd_value(A.mode, *p, z0, ih);
      }
      if (qc1 < A.alpha) {
        float* p = f + lb + (long long)A.a * qc1;
        *p = upd_value(A.mode, *p, z1, ih);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Persistent TMA kernels.  grid = min(items, 2 x SMs); CTA i processes work items i, i + grid, ...
// (item = (frame, chunk, tile), decoded from the page header) and consumes ONE continuous stream of
// windows across its items (forward: one window per band; back: one per mode), so the TMA ring, the
// tap loop and the per-item flush of one item overlap the first windows of the next (a CTA that
// processed only ~15 windows spent most of its time filling the pipeline: tools/tapbench.cu).
// The producer (thread 0) runs only at refill points (one CTA barrier per K = S/2 windows) and is
// loop-free, so the tap loop's control flow stays warp-uniform (tap tables stay on LDCU).

// item -> (frame z, chunk k, tile within the chunk); chunk found by an unrolled binary search over
// the page's cumulative item counts (words kItemBase..kItemBase+nch).
__device__ __forceinline__ void decode_item(int it, int per_frame, int nch, int& z, int& k, int& tile) {
  z = it / per_frame;
  const int r = it - z * per_frame;
  int lo = 0;
#pragma unroll
  for (int step = 32; step >= 1; step >>= 1)
    if (lo + step < nch && tabi(kItemBase + lo + step) <= r) lo += step;
  k = lo;
  tile = r - tabi(kItemBase + lo);
}

// Forward, two u positions per thread (columns warp and warp + 8 of a 32 x 16 tile; 256 threads):
// every tap entry read through the uniform datapath (LDCU.64) feeds four shared-memory loads and two
// FFMA2, halving the table and loop-control instructions per tap of forward_persistent (the kernel
// is issue-bound, not shared-memory-bound, with one position per thread: ncu r01c).  The flush is
// branch-free (predicated red.global.add per mode and position).
__device__ __forceinline__ void red_nz(float* p, float v) {
  asm volatile(
      "{\n.reg .pred q;\n"
      "setp.ne.f32 q, %1, 0f00000000;\n"
      "@q red.global.add.f32 [%0], %1;\n}\n" ::"l"(p),
      "f"(v)
      : "memory");
}

// Grid-wide barrier for persistent launches (every CTA resident: cooperative launch).  The word is
// zero-initialised once; CTA 0 adds 2^31 - (G - 1), the others 1, so the top bit flips exactly when
// all G CTAs have arrived and the low bits return to their old value (self-resetting across launches).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    __threadfence();  // this CTA's g_hat reductions are performed before its arrival
    const unsigned old = atomicAdd(bar, inc);
    unsigned cur;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
      if ((old ^ cur) & 0x80000000u) break;
      __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// r = g (/) g_hat in place over [0, count) (mode 1; reading R4) or the SMART log-ratio (mode 2; R17),
// grid-stride with float4 (both buffers 16-byte aligned, count of any size).
__device__ __forceinline__ float ratio_one(int mode, float g, float h) {
  if (mode == 2) return (g > 0.f && h > 0.f) ? logf(__fdiv_rn(g, h)) : 0.f;
  return h > 0.f ? __fdiv_rn(g, h) : 0.f;
}
__device__ __forceinline__ void ratio_pass(const TabArgs& A) {
  const long long n4 = A.ratio_count >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const float4* g4 = reinterpret_cast<const float4*>(A.meas);
  float4* h4 = reinterpret_cast<float4*>(A.dst);
  // U float4 of g and g_hat in flight per thread (the persistent grid has ~4x fewer threads than a
  // standalone element-wise launch: memory-level parallelism comes from the unroll)
  constexpr int U = 4;
  long long i = t0;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 gv[U], hv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gv[u] = __ldg(g4 + i + u * stride);
      hv[u] = __ldcg(h4 + i + u * stride);  // L2: the reductions of every CTA landed there
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      h4[i + u * stride] = make_float4(ratio_one(A.ratio_mode, gv[u].x, hv[u].x), ratio_one(A.ratio_mode, gv[u].y, hv[u].y),
                                       ratio_one(A.ratio_mode, gv[u].z, hv[u].z), ratio_one(A.ratio_mode, gv[u].w, hv[u].w));
  }
  for (; i < n4; i += stride) {
    const float4 gv = __ldg(g4 + i);
    const float4 hv = __ldcg(h4 + i);
    h4[i] = make_float4(ratio_one(A.ratio_mode, gv.x, hv.x), ratio_one(A.ratio_mode, gv.y, hv.y),
                        ratio_one(A.ratio_mode, gv.z, hv.z), ratio_one(A.ratio_mode, gv.w, hv.w));
  }
  for (long long i = 4 * n4 + t0; i < A.ratio_count; i += stride)
    A.dst[i] = ratio_one(A.ratio_mode, __ldg(A.meas + i), __ldcg(A.dst + i));
}

// zero the next iteration's g_hat accumulator (back kernel prologue; nobody reads it meanwhile)
__device__ __forceinline__ void zero_pass(const TabArgs& A) {
  const long long n4 = A.zero_count >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  float4* z4 = reinterpret_cast<float4*>(A.zero_buf);
  for (long long i = t0; i < n4; i += stride) z4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (long long i = 4 * n4 + t0; i < A.zero_count; i += stride) A.zero_buf[i] = 0.f;
}

#ifndef CTIS_FWD_PROBE
#define CTIS_FWD_PROBE 1
#endif
template <int MAXM, int S, bool EARLY, int PROBE = CTIS_FWD_PROBE>
__device__ __forceinline__ void forward_persistent2(const TabArgs& A, const CUtensorMap* tm) {
  extern __shared__ __align__(128) float smem[];
#ifndef CTIS_FWD_K
#define CTIS_FWD_K (S * 3 / 4)  // 8-slot ring: refill every 6 windows (C5 22.77 -> 22.54 us per frame-iteration; K = 2: 23.63)
#endif
  constexpr int K = CTIS_FWD_K, MP = MAXM / 2;  // refill every K windows
  constexpr int NW = kFwd2Threads / 32;  // 8 warps; warp w owns columns w and w + NW
  static_assert(2 * NW == kFwdTC, "two columns per warp");
  const int nch = tabi(0);
  const int per_frame = tabi(kItemBase + nch);
  const int items = per_frame * A.frames;
  if ((int)blockIdx.x >= items) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned slot_bytes = 4u * A.slot_floats;
  const unsigned full = sbase + S * slot_bytes;

  int p_item = blockIdx.x, p_band = 0, p_nb = 0, p_z = 0, p_Ur = 0, p_Uc = 0, p_lam0 = 0;
  uint32_t p_BI = 0;
  unsigned p_w = 0;
  auto p_load_item = [&]() {
    int k, tile;
    decode_item(p_item, per_frame, nch, p_z, k, tile);
    const uint32_t D = c_tab[1 + k];
    const int tiles_r = tabi(D + 5), nm = tabi(D + 2);
    p_lam0 = tabi(D + 0);
    p_nb = tabi(D + 1);
    p_Ur = tabi(D + 3) + (tile % tiles_r) * kFwdTR;
    p_Uc = tabi(D + 4) + (tile / tiles_r) * kFwdTC;
    p_BI = D + kDescHeader + ((nm + 3) & ~3);
    p_band = 0;
  };
  unsigned p_slot = 0;
  auto issue_one = [&]() {
    if (p_item >= items) return;
    const uint32_t bi = p_BI + 4 * p_band;
    mbar_expect_tx(full + 8 * p_slot, A.box_bytes);
    tma_4d(sbase + p_slot * slot_bytes, tm, p_Ur + tabi(bi + 0), p_Uc + tabi(bi + 1), p_lam0 + p_band, p_z,
           full + 8 * p_slot);
    ++p_w;
    if (++p_slot == S) p_slot = 0;
    if (++p_band == p_nb) {
      p_item += gridDim.x;
      if (p_item < items) p_load_item();
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(full + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    p_load_item();
    if (!(A.dbg & 1)) {
#pragma unroll 1
      for (int s = 0; s < S; ++s) issue_one();
    }
  }
  __syncthreads();

  unsigned c_slot = 0, c_phase = 0;  // consumer position in the ring
  const unsigned tb0 = sbase + 4u * (lane + A.box_r * warp);
  const unsigned tb1 = tb0 + 4u * A.box_r * NW;
  const unsigned n = (unsigned)A.n;
  unsigned w = 0, next_refill = K;
  bool ready = false;  // the current window's full barrier was already seen complete (early probe)
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int z, k, tile;
    decode_item(it, per_frame, nch, z, k, tile);
    const uint32_t D = c_tab[1 + k];
    const int nb = tabi(D + 1), nm = tabi(D + 2), tiles_r = tabi(D + 5);
    const int U_r = tabi(D + 3) + (tile % tiles_r) * kFwdTR, U_c = tabi(D + 4) + (tile / tiles_r) * kFwdTC;
    const uint32_t TP = D + kDescHeader + ((nm + 3) & ~3) + 4 * nb;
    float2 a0[MP], a1[MP];
#pragma unroll
    for (int q = 0; q < MP; ++q) a0[q] = a1[q] = make_float2(0.f, 0.f);
    auto compute = [&](unsigned off, int b) {
      const uint4* ent = tab4(TP) + b * MP;
#pragma unroll
      for (int q = 0; q < MP; ++q) {
        const uint4 e = ent[q];
        const float2 wv = make_float2(__uint_as_float(e.z), __uint_as_float(e.w));
        a0[q] = __ffma2_rn(wv, make_float2(lds(tb0 + off + e.x), lds(tb0 + off + e.y)), a0[q]);
        a1[q] = __ffma2_rn(wv, make_float2(lds(tb1 + off + e.x), lds(tb1 + off + e.y)), a1[q]);
      }
    };
#pragma unroll 1
    for (int b = 0; b < nb; ++b, ++w) {
      if (w >= next_refill) {
        if (!(A.dbg & 16)) __syncthreads();  // every warp has consumed the windows before w: slots free
        // (CTIS_DEBUG & 16: profiling only — no refill barrier, results invalid; measures its cost)
        if (threadIdx.x == 0 && !(A.dbg & 1)) {
#pragma unroll 1
          for (int q = 0; q < S; ++q)  // catch up fully: refill points can land one window late
            if (p_w < w + S) issue_one();
        }
        next_refill = w + K;
      }
      if (!(A.dbg & 1) && !ready) mbar_wait(full + 8 * c_slot, c_phase);
      const unsigned n_slot = c_slot + 1 == S ? 0u : c_slot + 1, n_phase = c_slot + 1 == S ? c_phase ^ 1u : c_phase;
      // PROBE 1: probe the next window's barrier before the tap loop; PROBE 2: after it (the probe has
      // acquire semantics, so shared loads issued after it wait for it); PROBE 0: plain waits only
      bool ready_next = false;
      if (EARLY && PROBE == 1) ready_next = mbar_test(full + 8 * n_slot, n_phase);
      compute(c_slot * slot_bytes, b);
      if (EARLY && PROBE == 2) ready_next = mbar_test(full + 8 * n_slot, n_phase);
      c_slot = n_slot;
      c_phase = n_phase;
      ready = ready_next;
    }
    // flush this item: g_hat[(E(u) + o_ref) mod n] += acc for both positions (see forward_group)
    float* g = A.dst + (long long)z * A.dst_frame;
    if (A.dbg & 2) {  // profiling: no flush (keep the accumulators live)
      float t = 0.f;
#pragma unroll
      for (int q = 0; q < MP; ++q) t += a0[q].x + a0[q].y + a1[q].x + a1[q].y;
      if (t == -1.f) g[0] = t;
      continue;
    }
    if (A.nowrap && !(A.dbg & 1)) {  // (CTIS_DEBUG & 1 computes on stale windows: keep the modular path)
      // no tap wraps: every nonzero accumulator's pixel E(u) + o_ref is the exact FPA index in [0, n)
      // (E(q) + o of each contributing tap), so no modular reduction; zero accumulators (positions u
      // outside every band's live range) are never stored, so their out-of-range addresses are unused
      const float* gz = g;
      const long long e0 = (long long)(U_r + lane) + (long long)A.gamma * (U_c + warp);
      const long long e1 = e0 + (long long)A.gamma * NW;
#pragma unroll
      for (int c = 0; c < MAXM; ++c) {
        if (c < nm) {
          const unsigned o = c_tab[D + kDescHeader + c];
          red_nz(const_cast<float*>(gz) + (e0 + o), (c & 1) ? a0[c >> 1].y : a0[c >> 1].x);
          red_nz(const_cast<float*>(gz) + (e1 + o), (c & 1) ? a1[c >> 1].y : a1[c >> 1].x);
        }
      }
      continue;
    }
    unsigned ub0 = (unsigned)((U_r + lane) + A.gamma * (U_c + warp)) + A.bias;
    for (int q = 0; q < A.nsub; ++q) ub0 = min(ub0, ub0 - n);
    unsigned ub1 = ub0 + (unsigned)(((unsigned long long)A.gamma * NW) % n);  // E(u + NW columns) mod n
    ub1 = min(ub1, ub1 - n);
#pragma unroll
    for (int c = 0; c < MAXM; ++c) {
      if (c < nm) {
        const unsigned o = c_tab[D + kDescHeader + c];
        unsigned P0 = ub0 + o, P1 = ub1 + o;
        P0 = min(P0, P0 - n);
        P1 = min(P1, P1 - n);
        red_nz(g + P0, (c & 1) ? a0[c >> 1].y : a0[c >> 1].x);
        red_nz(g + P1, (c & 1) ? a1[c >> 1].y : a1[c >> 1].x);
      }
    }
  }
  if (A.ratio_mode) {  // fused ratio (Alg. 1 line 8) once every CTA's reductions have landed
    grid_sync(A.gbar);
    ratio_pass(A);
#ifdef CTIS_ZERO_IN_FWD
    if (A.zero_count) zero_pass(A);
#endif
  }
}

// Programmatic dependent launch: let the next kernel of the MLEM chain be scheduled as soon as this
// grid's CTAs are all resident, and wait for the previous kernel's results (its memory is visible
// after griddepcontrol.wait) — hides the kernel-boundary launch latency inside the CUDA graph.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// CTIS_DEBUG & 8: fill the window ring with NaN before the kernel runs, so that any read of shared
// memory the kernel did not write this launch poisons the result (tests/test_gpu_parity.py)
__device__ __forceinline__ void nan_fill_smem(int nf) {
  extern __shared__ __align__(128) float smem[];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) smem[i] = __int_as_float(0x7fc00000);
  __syncwarp();
  __syncthreads();
}

// Back with four voxels per thread (columns warp + 8k of the 32 x 32 tile, 256 threads): every tap
// entry read through the uniform datapath feeds eight shared-memory loads (cf. forward_persistent2).
// POS voxels per thread: columns warp + 8k (k < POS) of a 32 x 8*POS tile (POS = 2 for small problems,
// where 32 x 32 tiles would leave SMs idle)
#ifndef CTIS_BACK_REFILL
#define CTIS_BACK_REFILL 0
#endif
template <int NB, int POS, bool REFILL = CTIS_BACK_REFILL>
__device__ __forceinline__ void back_persistent4(const TabArgs& A, const CUtensorMap* tm) {
  constexpr int TC = 8 * POS;
  extern __shared__ __align__(128) float smem[];
#ifndef CTIS_BACK_K
#define CTIS_BACK_K 6  // measured (B200): K = 2/3/4/6/7 -> C4 back 60.6/59.8/59.8/58.2/59.7 us, C3 29.1/25.1/25.1/23.0 us
#endif
  constexpr int S = kBackStages, K = CTIS_BACK_K, BP = NB / 2;  // refill every K windows
  constexpr int NWARPS = kBack4Threads / 32;  // 8: voxel columns warp + 8k, k < 4
  const int nch = tabi(0);
  const int per_frame = tabi(kItemBase + nch);
  const int items = per_frame * A.frames;
#ifndef CTIS_ZERO_AT_END
  if (A.zero_count) zero_pass(A);
#endif
  if ((int)blockIdx.x >= items) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned slot_bytes = 4u * A.slot_floats;
  const unsigned full = sbase + S * slot_bytes;

  // window origin of mode c of the tile at (q_r0, q_c0): host-split Bm = Bm_r + gamma*Bm_c, one carry
  // and one wrap (the plan only selects this kernel when no window of the page wraps)
  auto origin_rc = [&](uint32_t MI, int c, int q_r0, int q_c0, int& R0, int& C0) {
    R0 = q_r0 + tabi(MI + 4 * c + 0);
    C0 = q_c0 + tabi(MI + 4 * c + 1);
    if (R0 >= A.gamma) {
      R0 -= A.gamma;
      C0 += 1;
    }
    if (C0 >= A.xi) C0 -= A.xi;
  };
  int p_item = blockIdx.x, p_mode = 0, p_nm = 0, p_z = 0, p_qr = 0, p_qc = 0;
  uint32_t p_MI = 0;
  unsigned p_w = 0;
  auto p_load_item = [&]() {
    int k, tile;
    decode_item(p_item, per_frame, nch, p_z, k, tile);
    const uint32_t D = c_tab[1 + k];
    const int tiles_r = tabi(D + 3);
    p_nm = tabi(D + 2);
    p_qr = (tile % tiles_r) * kBackTR;
    p_qc = (tile / tiles_r) * TC;
    p_MI = D + kDescHeader;
    p_mode = 0;
  };
  auto issue_one = [&]() {
    if (p_item >= items) return;
    const unsigned slot = p_w & (S - 1);
    int R0, C0;
    origin_rc(p_MI, p_mode, p_qr, p_qc, R0, C0);
    mbar_expect_tx(full + 8 * slot, A.box_bytes);
    tma_3d(sbase + slot * slot_bytes, tm, R0, C0, p_z, full + 8 * slot);
    ++p_w;
    if (++p_mode == p_nm) {
      p_item += gridDim.x;
      if (p_item < items) p_load_item();
    }
  };
  // REFILL: window w + S is loaded into slot w % S by the last warp to finish window w (release
  // counters cnt[S], producer state in shared memory); no CTA-wide refill barrier
  const unsigned cnt = full + 8 * S, pst = cnt + 4 * S;
  auto save_state = [&]() {
    st_shared_u32(pst + 0, (unsigned)p_item);
    st_shared_u32(pst + 4, (unsigned)p_mode);
    st_shared_u32(pst + 8, (unsigned)p_nm);
    st_shared_u32(pst + 12, (unsigned)p_z);
    st_shared_u32(pst + 16, (unsigned)p_qr);
    st_shared_u32(pst + 20, (unsigned)p_qc);
    st_shared_u32(pst + 24, p_MI);
    st_shared_u32(pst + 28, p_w);
  };
  auto load_state = [&]() {
    p_item = (int)ld_shared_u32(pst + 0);
    p_mode = (int)ld_shared_u32(pst + 4);
    p_nm = (int)ld_shared_u32(pst + 8);
    p_z = (int)ld_shared_u32(pst + 12);
    p_qr = (int)ld_shared_u32(pst + 16);
    p_qc = (int)ld_shared_u32(pst + 20);
    p_MI = ld_shared_u32(pst + 24);
    p_w = ld_shared_u32(pst + 28);
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) mbar_init(full + 8 * q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    p_load_item();
#pragma unroll
    for (int q = 0; q < S; ++q) issue_one();
    if (REFILL) {
      for (int q = 0; q < S; ++q) st_shared_u32(cnt + 4 * q, 0u);
      save_state();
    }
  }
  __syncthreads();
  // after consuming window wi: the warp that completes slot wi % S's count issues window wi + S
  auto release = [&](unsigned wi) {
    __syncwarp();
    if (lane == 0) {
      const unsigned old = atom_add_acqrel_shared(cnt + 4 * (wi & (S - 1)), 1u);
      if (old % NWARPS == NWARPS - 1) {
        fence_proxy_async();
        load_state();
        if (p_item < items) {
          issue_one();
          save_state();
        }
      }
    }
  };

  const unsigned t0 = sbase + 4u * (lane + A.box_r * warp), cstep = 4u * A.box_r * NWARPS;
  unsigned w = 0, next_refill = K;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int z, k, tile;
    decode_item(it, per_frame, nch, z, k, tile);
    const uint32_t D = c_tab[1 + k];
    const int lam0 = tabi(D + 0), nb = tabi(D + 1), nm = tabi(D + 2), tiles_r = tabi(D + 3);
    const int q_r0 = (tile % tiles_r) * kBackTR, q_c0 = (tile / tiles_r) * TC;
    const uint32_t MI = D + kDescHeader, TP = MI + 4 * nm, IH = TP + 2 * nm * NB;
    float2 acc[POS][BP];
#pragma unroll
    for (int k4 = 0; k4 < POS; ++k4)
#pragma unroll
      for (int q = 0; q < BP; ++q) acc[k4][q] = make_float2(0.f, 0.f);
    auto compute = [&](unsigned ba, int c) {
      const uint4* ent = tab4(TP) + c * BP;
#pragma unroll
      for (int q = 0; q < BP; ++q) {
        const uint4 e = ent[q];
        const float2 wv = make_float2(__uint_as_float(e.z), __uint_as_float(e.w));
#pragma unroll
        for (int k4 = 0; k4 < POS; ++k4) {
          const unsigned bk = ba + k4 * cstep;
          acc[k4][q] = __ffma2_rn(wv, make_float2(lds(bk + e.x), lds(bk + e.y)), acc[k4][q]);
        }
      }
    };
    for (int c = 0; c < nm;) {
      if (!REFILL && w >= next_refill) {
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll 1
          for (int q = 0; q < S; ++q)  // catch up fully: refill points can land one window late
            if (p_w < w + S) issue_one();
        }
        next_refill = w + K;
      }
      const unsigned s0 = w & (S - 1);
      mbar_wait(full + 8 * s0, (w / S) & 1u);
      compute(t0 + s0 * slot_bytes, c);
      if (REFILL) release(w);
      if (c + 1 < nm) {
        const unsigned s1 = (w + 1) & (S - 1);
        mbar_wait(full + 8 * s1, ((w + 1) / S) & 1u);
        compute(t0 + s1 * slot_bytes, c + 1);
        if (REFILL) release(w + 1);
        w += 2;
        c += 2;
      } else {
        w += 1;
        c += 1;
      }
    }
    // epilogue of this item: f <- f * z * (1/h_lam) (or z).  Loads of f for groups of EG bands are
    // issued together (ld.global.nc: each element is read and then written by this thread only), then
    // the stores: one L2 round trip per group instead of one per band (the compiler cannot move a
    // band's loads above the previous band's stores to the same array)
    float* f = A.dst + (long long)z * A.dst_frame;
    const int qr = q_r0 + lane;
#ifndef CTIS_BACK_EG
#define CTIS_BACK_EG 6  // epilogue: bands whose f loads are issued together
#endif
    constexpr int EG = NB < CTIS_BACK_EG ? NB : CTIS_BACK_EG;
    if (A.mode == 3) {  // mode-split plans: add this mode subset's partial z (ctis_api.cu enqueue_back)
      if (qr < A.a) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
          if (b < nb) {
            const long long lb = (long long)(lam0 + b) * A.ell + qr;
#pragma unroll
            for (int k4 = 0; k4 < POS; ++k4) {
              const int qc = q_c0 + warp + NWARPS * k4;
              if (qc < A.alpha) red_nz(f + lb + (long long)A.a * qc, (b & 1) ? acc[k4][b >> 1].y : acc[k4][b >> 1].x);
            }
          }
      }
      continue;
    }
    if (qr < A.a) {
#pragma unroll
      for (int b0 = 0; b0 < NB; b0 += EG) {
        float old[EG][POS];
#pragma unroll
        for (int bb = 0; bb < EG; ++bb) {
          const int b = b0 + bb;
#pragma unroll
          for (int k4 = 0; k4 < POS; ++k4) {
            const int qc = q_c0 + warp + NWARPS * k4;
            old[bb][k4] = 1.f;
            if (b < NB && b < nb && A.mode && qc < A.alpha)
              old[bb][k4] = __ldg(f + (long long)(lam0 + b) * A.ell + qr + (long long)A.a * qc);
          }
        }
#pragma unroll
        for (int bb = 0; bb < EG; ++bb) {
          const int b = b0 + bb;
          if (b < NB && b < nb) {
            const long long lb = (long long)(lam0 + b) * A.ell + qr;
            const float ih = tabf(IH + b);
#pragma unroll
            for (int k4 = 0; k4 < POS; ++k4) {
              const int qc = q_c0 + warp + NWARPS * k4;
              const float zz = (b & 1) ? acc[k4][b >> 1].y : acc[k4][b >> 1].x;
              if (qc < A.alpha) f[lb + (long long)A.a * qc] = upd_value(A.mode, old[bb][k4], zz, ih);
            }
          }
        }
      }
    }
  }
#ifdef CTIS_ZERO_AT_END
  if (A.zero_count) zero_pass(A);  // CTAs that finish early fill the tail with the zeroing
#endif
}

// ------------------------------------------------------------------------------------------------
// Strip forward (ctis_internal.h, "Strip forward").  The same u-space accumulation as
// forward_persistent2 — acc[mode](u) += w * f_lam[u - (dr, dc)], flushed to g_hat[E(u) + o_ref]
// (Eqs. 11-13) — but a warp owns a strip group of <= kStripMG modes whose column shift dc is the same
// in every band of the chunk, and each thread owns kStripP consecutive rows of one u column.  Per band
// the thread loads one strip of window rows into registers (<= kStripNQ float4) and every mode of the
// group reads its kStripP operands from that strip at its own row offset o: the offset is a run-time
// value, so each (mode slot, o) pair is its own straight-line block (FFMA2 for even o) selected by a
// warp-uniform switch.  Warp specialisation: the last warp's lane 0 produces the TMA windows into a
// A.stages-deep ring (full / empty mbarriers), the consumer warps release a slot as soon as their strip
// is in registers.
#include "ctis_strip_dispatch.inc"
#ifndef CTIS_STRIP_PIN
#define CTIS_STRIP_PIN 1  // ring depth and slot size pinned in registers in the consumer loop (C4 MLEM 134.6 -> 134.0 us)
#endif
#ifndef CTIS_STRIP_PROBE
#define CTIS_STRIP_PROBE 1  // test the next window's mbarrier inside the dispatch (hides the probe latency)
#endif

// one lane of the (converged) warp; elect.sync also orders the warp's earlier shared loads before the
// elected lane's release (it synchronises the warp like __syncwarp)
__device__ __forceinline__ bool elect_one() {
  unsigned p;
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n"
      : "=r"(p)
      :
      : "memory");
  return p != 0;
}

// g_hat tile reduction by the async proxy: out[(r0 + i) + gamma*(c0 + j) (+ n*z)] += tile[j][i] for the
// 32 x 16 box at shared address src (TMA, add).  Measured on B200 (tools/tma_red_test.cu): the box must
// start inside the tensor on a 16-byte boundary of the inner dimension, else the instruction faults.
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* tm, unsigned src, int r0, int c0, int z) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
      "r"(r0), "r"(c0), "r"(z), "r"(src)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int MG>
__device__ __forceinline__ void forward_strip_consume(const TabArgs& A, const CUtensorMap* tg, int warp, int lane,
                                                      int per_frame, int nch, int items, unsigned sbase,
                                                      unsigned slot_bytes, unsigned full, unsigned stage);

template <int MG>
__device__ __forceinline__ void forward_strip(const TabArgs& A, const CUtensorMap* tm, const CUtensorMap* tg) {
  extern __shared__ __align__(1024) float smem[];
  const unsigned S = (unsigned)A.stages;
  static_assert(MG == kStripMG, "descriptor layout assumes kStripMG slots per group");
  const int nch = tabi(0);
  const int per_frame = tabi(kItemBase + nch);
  const int items = per_frame * A.frames;
  if ((int)blockIdx.x >= items) return;
  // warp index made visibly warp-uniform (keeps the tap entries on the uniform datapath)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int nwc = (int)(blockDim.x >> 5) - 1;  // consumer warps; warp nwc is the TMA producer
  const unsigned smem0 = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned slot_bytes = 4u * A.slot_floats;
  // [full S][empty S] mbarriers | ring: S slots from byte 128 | staging: 1024-byte aligned, kStripStage
  // floats per consumer warp.  Every address is uniform (no per-band rematerialisation from blockDim).
  const unsigned full = smem0, empty = smem0 + 8 * kStripStagesMax;
  const unsigned sbase = smem0 + 128;
  const unsigned stage0 = (sbase + S * slot_bytes + 1023u) & ~1023u;
  static_assert(16 * kStripStagesMax <= 128, "mbarriers fit below the ring");
  if (threadIdx.x == 0) {
    for (unsigned s = 0; s < S; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, (unsigned)nwc);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == nwc) {  // ---- producer: one TMA box per (item, band), in the consumers' order
    if (lane == 0 && !(A.dbg & 1)) {
      unsigned slot = 0, phase = 0, w = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        int z, k, tile;
        decode_item(it, per_frame, nch, z, k, tile);
        const uint32_t D = c_tab[1 + k];
        const int lam0 = tabi(D + 0), nb = tabi(D + 1), nhg = tabi(D + 2), tiles_r = tabi(D + 5);
        const int U_r = tabi(D + 3) + (tile % tiles_r) * kFwdTR, U_c = tabi(D + 4) + (tile / tiles_r) * kFwdTC;
        const uint32_t BI = D + kDescHeader + 2 * MG * nhg;
#pragma unroll 1
        for (int b = 0; b < nb; ++b, ++w) {
          if (w >= S) mbar_wait(empty + 8 * slot, phase ^ 1u);  // consumers released the slot
          mbar_expect_tx(full + 8 * slot, A.box_bytes);
          tma_4d(sbase + slot * slot_bytes, tm, U_r + tabi(BI + 4 * b), U_c + tabi(BI + 4 * b + 1), lam0 + b, z,
                 full + 8 * slot);
          if (++slot == S) {
            slot = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else {
    forward_strip_consume<MG>(A, tg, warp, lane, per_frame, nch, items, sbase, slot_bytes, full,
                              stage0 + 4u * kStripStage * warp);
  }
  if (A.ratio_mode) {  // fused ratio (CTIS_OPT_FUSED_RATIO): one CTA per SM, cooperative launch
    grid_sync(A.gbar);
    ratio_pass(A);
  }
}

template <int MG>
__device__ __forceinline__ void forward_strip_consume(const TabArgs& A, const CUtensorMap* tg, int warp, int lane,
                                                      int per_frame, int nch, int items, unsigned sbase,
                                                      unsigned slot_bytes, unsigned full, unsigned stage) {
  const unsigned S = (unsigned)A.stages;
  constexpr int NV = 4 * kStripNQ;
  // ---- consumers: lane = rs + 2*col owns rows 16*rs .. 16*rs+15 of u column col of the 32 x 16 tile
  const int rs = lane & 1, col = lane >> 1;
  unsigned tb = sbase + 4u * (kStripP * rs + A.box_r * col);
  // opaque copies: ptxas would otherwise re-derive these addresses (S2R, LDC) in every band iteration
  asm volatile("mov.b32 %0, %0;" : "+r"(tb));
  asm volatile("mov.b32 %0, %0;" : "+r"(full));
#if CTIS_STRIP_PIN
  asm volatile("mov.b32 %0, %0;" : "+r"(slot_bytes));  // kept in registers, not re-read from the
  unsigned S_ = S;                                      // parameter bank every band
  asm volatile("mov.b32 %0, %0;" : "+r"(S_));
#define STRIP_S S_
#else
#define STRIP_S S
#endif
  // async-proxy flush: the whole plan is 2-D translations (every nonzero accumulator's pixel is inside
  // the FPA box) — otherwise (cyclic wrap of Eq. 7) red.global.add with exact modular indices
  const bool tma_flush = A.tma_flush && !(A.dbg & 1);
  float v[NV];
  unsigned phase = 0, tslot = tb;  // tslot: this thread's strip base in the current slot
  // ring position as the full-barrier address (the empty barrier of a slot sits 8 * kStripStagesMax bytes
  // above its full barrier): one add and compare per band, and the release reads an address register
  // that is not rewritten before the next band (C4 forward 60.7 -> 60.0 us, with the 32-bit entry index)
  unsigned fslot = full;
  const unsigned fend = full + 8u * STRIP_S;
  unsigned notma = A.dbg & 1;  // profiling switch, pinned in a register (not re-read every band)
  asm volatile("mov.b32 %0, %0;" : "+r"(notma));
  bool staged = false;  // bulk reductions of this warp's staging tiles may still be reading them
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int z, k, tile;
    decode_item(it, per_frame, nch, z, k, tile);
    const uint32_t D = c_tab[1 + k];
    const int nb = tabi(D + 1), nhg = tabi(D + 2), tiles_r = tabi(D + 5);
    const int U_r = tabi(D + 3) + (tile % tiles_r) * kFwdTR, U_c = tabi(D + 4) + (tile / tiles_r) * kFwdTC;
    const bool act = warp < nhg;
    // entry index in uint4 units (32-bit: no 64-bit pointer arithmetic per band)
    uint32_t ei = (D + kDescHeader + 2 * MG * nhg + 4 * nb) / 4 + 2 * warp;
    const uint32_t estep = 2u * nhg;
    const uint4* c4 = reinterpret_cast<const uint4*>(c_tab);
    float acc[MG][kStripP];
#pragma unroll
    for (int m = 0; m < MG; ++m)
#pragma unroll
      for (int i = 0; i < kStripP; ++i) acc[m][i] = 0.f;
    // tap entries are software-pipelined one band ahead (constant-cache latency overlaps a band's FMAs)
    uint4 e0 = make_uint4(0u, 0u, 0u, 0u), e1 = e0;
    if (act) {
      e0 = c4[ei];
      e1 = c4[ei + 1];
    }
    unsigned ready = 0;  // CTIS_STRIP_PROBE: the previous band's dispatch found this band's window landed
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      const uint4 c0 = e0, c1 = e1;
      if (act && b + 1 < nb) {
        ei += estep;
        e0 = c4[ei];
        e1 = c4[ei + 1];
      }
      const unsigned fcur = fslot;
      if (!notma && !ready) mbar_wait(fcur, phase);
      if (act) strip_load(v, tslot + c0.x);
      if (elect_one()) mbar_arrive(fcur + 8u * kStripStagesMax);
      tslot += slot_bytes;
      fslot += 8u;
      if (fslot == fend) {
        fslot = full;
        phase ^= 1u;
        tslot = tb;
      }
      if (act) {
        // row offset per slot (kStripNO: no tap in this band, the skip target)
#if CTIS_STRIP_PROBE
        // the next window's mbarrier is tested at the dispatch's entry and its result read at the exit, so
        // the probe's latency hides behind the FMA blocks (every band: after an item's last band the next
        // slot is the next item's first window; ONE dispatch copy — a second copy for the last band measured
        // slower, instruction-cache pressure).  C4 forward 63.6 -> 61.2 us, MLEM 133.1 -> 131.6 us/iteration.
        strip_dispatch4p(acc[0], acc[1], acc[2], acc[3], v, __uint_as_float(c0.z), __uint_as_float(c0.w),
                         __uint_as_float(c1.x), __uint_as_float(c1.y), c0.y & 0xffu, (c0.y >> 8) & 0xffu,
                         (c0.y >> 16) & 0xffu, c0.y >> 24, fslot, phase, ready);
#else
        strip_dispatch4(acc[0], acc[1], acc[2], acc[3], v, __uint_as_float(c0.z), __uint_as_float(c0.w),
                        __uint_as_float(c1.x), __uint_as_float(c1.y), c0.y & 0xffu, (c0.y >> 8) & 0xffu,
                        (c0.y >> 16) & 0xffu, c0.y >> 24);
#endif
      }
    }
    if (!act) continue;
    float* g = A.dst + (long long)z * A.dst_frame;
    if (A.dbg & 2) {  // profiling: no flush (keep the accumulators live)
      float t = 0.f;
#pragma unroll
      for (int m = 0; m < MG; ++m)
#pragma unroll
        for (int i = 0; i < kStripP; ++i) t += acc[m][i];
      if (t == -1.f) g[0] = t;
      continue;
    }
    // Flush: each mode's 32 x 16 accumulator tile -> staging (TMA 128-byte swizzle: 16-byte chunk c of u
    // column j lives at chunk c ^ (j & 7) of the column's 128-byte line) -> g_hat[E(u) + o_ref] +=.
    // A tile whose 2-D FPA box lies inside the FPA (no-wrap plans) is ONE bulk tensor reduce-add drained
    // by the async proxy while the warp moves on; any other tile (FPA edge, cyclic wrap of Eq. 7) is
    // read back lane = row and added element by element with exact modular indices (red.global.add).
    if (staged) {  // the previous item's bulk reductions must have read the staging tiles
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
      staged = false;
    }
    unsigned live = 0;  // modes whose tile holds a nonzero accumulator (dead tiles: u outside the mode's range)
#pragma unroll
    for (int m = 0; m < MG; ++m) {
      const unsigned tile_s = stage + 2048u * m + 128u * col;
      bool nz = false;
#pragma unroll
      for (int i = 0; i < kStripP; ++i) nz |= acc[m][i] != 0.f;
      live |= __any_sync(0xffffffffu, nz) ? 1u << m : 0u;
#pragma unroll
      for (int j = 0; j < kStripP / 4; ++j)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(tile_s + 16u * ((4 * rs + j) ^ (col & 7))),
                     "f"(acc[m][4 * j]), "f"(acc[m][4 * j + 1]), "f"(acc[m][4 * j + 2]), "f"(acc[m][4 * j + 3])
                     : "memory");
    }
    fence_proxy_async();
    __syncwarp();
    const long long n = A.n;
#pragma unroll 1
    for (int m = 0; m < MG; ++m) {
      const unsigned o = c_tab[D + kDescHeader + MG * warp + m];
      if (o == 0xffffffffu || !((live >> m) & 1u)) continue;
      const unsigned orc = c_tab[D + kDescHeader + MG * nhg + MG * warp + m];  // o_ref as (row, column)
      const int r0 = U_r + (int)(orc & 0xffffu), c0 = U_c + (int)(orc >> 16);
      const unsigned tile_s = stage + 2048u * m;
      if (tma_flush && r0 >= 0 && (r0 & 3) == 0 && c0 >= 0 && r0 + kFwdTR <= A.gamma && c0 + kFwdTC <= A.xi) {
        if (lane == 0) tma_reduce_add_3d(tg, tile_s, r0, c0, z);
        staged = true;
        continue;
      }
      const long long e_lane = (long long)(U_r + lane) + (long long)A.gamma * U_c + o;
#pragma unroll 4
      for (int cc = 0; cc < kFwdTC; ++cc) {
        const float val = lds(tile_s + 128u * cc + 16u * ((lane >> 2) ^ (cc & 7)) + 4u * (lane & 3));
        long long e = e_lane + (long long)A.gamma * cc;
        if (!A.nowrap || (A.dbg & 1)) {  // no-wrap plans: every nonzero accumulator's index is in [0, n)
          e %= n;
          if (e < 0) e += n;
        }
        red_nz(g + e, val);
      }
    }
    if (staged && lane == 0) bulk_commit();
    __syncwarp();  // the element path's staging reads are done before the next item's writes
  }
  if (lane == 0) bulk_wait0();  // every bulk reduction of this warp has completed (and read its staging)
  __syncwarp();
}

#undef STRIP_S
}  // namespace

// Element-loader forward (plans whose geometry rules out TMA boxes: a % 4 != 0)
#define CTIS_FWD(M, MINB)                                                                                  \
  extern "C" __global__ void __launch_bounds__(kFwdThreads, MINB)                                          \
      ctis_fwd_g1_m##M##_s(const TabArgs A, const __grid_constant__ CUtensorMap tm) {                      \
    if (A.frames == 0) return;                                                                             \
    pdl_enter();                                                                                           \
    if (A.dbg & 8) nan_fill_smem(kFwdStages * A.slot_floats);                                             \
    forward_body<1, M, false, true>(A, &tm);                                                               \
  }
CTIS_FWD(2, 2)
CTIS_FWD(4, 2)
CTIS_FWD(6, 2)
CTIS_FWD(8, 2)
CTIS_FWD(10, 2)
CTIS_FWD(12, 2)
CTIS_FWD(14, 2)
CTIS_FWD(16, 2)
CTIS_FWD(18, 2)
CTIS_FWD(20, 2)
CTIS_FWD(22, 2)
CTIS_FWD(24, 2)
CTIS_FWD(26, 2)
CTIS_FWD(28, 2)
CTIS_FWD(30, 2)
CTIS_FWD(32, 2)
CTIS_FWD(40, 1)
CTIS_FWD(48, 1)
CTIS_FWD(56, 1)
CTIS_FWD(64, 1)
CTIS_FWD(72, 1)
CTIS_FWD(80, 1)
CTIS_FWD(88, 1)
CTIS_FWD(96, 1)

#define CTIS_FWD2(OCC, S, M)                                                                               \
  extern "C" __global__ void __launch_bounds__(kFwd2Threads, OCC)                                          \
      ctis_fwd_g##OCC##_m##M##_t(const TabArgs A, const __grid_constant__ CUtensorMap tm) {                \
    if (A.frames == 0) return;                                                                             \
    pdl_enter();                                                                                           \
    if (A.dbg & 8) nan_fill_smem(S * A.slot_floats);                                                           \
    forward_persistent2<M, S, true>(A, &tm);                                                                     \
  }
CTIS_FWD2(2, 8, 2)
CTIS_FWD2(2, 8, 4)
CTIS_FWD2(2, 8, 6)
CTIS_FWD2(2, 8, 8)
CTIS_FWD2(2, 8, 10)
CTIS_FWD2(2, 8, 12)
CTIS_FWD2(2, 8, 14)
CTIS_FWD2(2, 8, 16)
CTIS_FWD2(2, 8, 18)
CTIS_FWD2(2, 8, 20)
CTIS_FWD2(2, 8, 22)
CTIS_FWD2(2, 8, 24)
CTIS_FWD2(2, 8, 26)
CTIS_FWD2(2, 8, 28)
CTIS_FWD2(2, 8, 30)
CTIS_FWD2(2, 8, 32)
CTIS_FWD2(2, 8, 36)
CTIS_FWD2(2, 8, 40)

#ifndef CTIS_BACK2_MINB
#define CTIS_BACK2_MINB 2  // resident CTAs per SM the 32 x 16-tile back kernels are compiled for
#endif
#ifndef CTIS_BACK4_MINB
#define CTIS_BACK4_MINB 2  // resident CTAs per SM the 32 x 32-tile back kernels are compiled for
#endif
#define CTIS_BACK4(NB, POS, NAME)                                                                          \
  extern "C" __global__ void __launch_bounds__(kBack4Threads, POS == 2 ? CTIS_BACK2_MINB : CTIS_BACK4_MINB) \
      NAME(const TabArgs A, const __grid_constant__ CUtensorMap tm) {                                      \
    if (A.frames == 0) return;                                                                             \
    pdl_enter();                                                                                           \
    if (A.dbg & 8) nan_fill_smem(kBackStages * A.slot_floats);                                             \
    back_persistent4<NB, POS>(A, &tm);                                                                     \
  }
CTIS_BACK4(2, 4, ctis_back4_b2_t)
CTIS_BACK4(4, 4, ctis_back4_b4_t)
CTIS_BACK4(8, 4, ctis_back4_b8_t)
CTIS_BACK4(10, 4, ctis_back4_b10_t)
CTIS_BACK4(12, 4, ctis_back4_b12_t)
CTIS_BACK4(16, 4, ctis_back4_b16_t)
CTIS_BACK4(2, 2, ctis_back2_b2_t)
CTIS_BACK4(4, 2, ctis_back2_b4_t)
CTIS_BACK4(8, 2, ctis_back2_b8_t)
CTIS_BACK4(10, 2, ctis_back2_b10_t)
CTIS_BACK4(12, 2, ctis_back2_b12_t)
CTIS_BACK4(16, 2, ctis_back2_b16_t)

// Element-loader back projection (wrapped r windows or gamma % 4 != 0)
#define CTIS_BACK(NB)                                                                                      \
  extern "C" __global__ void __launch_bounds__(kBackThreads, 2)                                            \
      ctis_back_b##NB##_s(const TabArgs A, const __grid_constant__ CUtensorMap tm) {                       \
    if (A.frames == 0) return;                                                                             \
    pdl_enter();                                                                                           \
    if (A.dbg & 8) nan_fill_smem(kBackStages * A.slot_floats);                                             \
    back_body<NB, false, true>(A, &tm);                                                                    \
  }
CTIS_BACK(2)
CTIS_BACK(4)
CTIS_BACK(8)
CTIS_BACK(10)
CTIS_BACK(12)
CTIS_BACK(16)

// Strip forward (TMA plans with column-sharing modes): kStripWarpsMax consumer warps + 1 producer
extern "C" __global__ void __launch_bounds__(32 * (kStripWarpsMax + 1), 1)
    ctis_fwd_strip_t(const TabArgs A, const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tg) {
  if (A.frames == 0) return;
  pdl_enter();
  if (A.dbg & 8) nan_fill_smem(32 + A.stages * A.slot_floats);
  forward_strip<kStripMG>(A, &tm, &tg);
}
