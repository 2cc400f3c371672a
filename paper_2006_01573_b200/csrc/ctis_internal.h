// Internal declarations shared by the plan builder (ctis_api.cu) and the kernels
// (ctis_kernels.cu).  Not part of the public ABI (include/ctis.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ctis {

// ---------------------------------------------------------------------------
// Forward projection tiles (output-stationary gather over the FPA).
// A tap (o, w) of band lam is a 1-D cyclic shift by o on the column-major
// flattened FPA (Eq. 7).  On the 2-D FPA that shift is, for
// each voxel (r, c), either (r+dr, c+dc), (r+dr-gamma, c+dc+1) [carry into the
// next column] and, modulo xi, a wrap past the last column.  So every tap is
// exactly <= 4 rectangle "pieces" of the field stop, each a pure 2-D
// translation.  The builder clips each piece against the forward tiles and
// stores one FwdEntry per (tile, piece):
//   FPA pixel (R, C) of the clip rectangle receives w * f[base + R + a*C].
constexpr int kFwdTileR = 64;   // FPA rows per forward tile (gamma direction, contiguous)
constexpr int kFwdTileC = 16;   // FPA columns per forward tile
constexpr int kFwdThreads = 256;

struct FwdEntry {
  int base;            // lam*l - sr - a*sc, so that f index = base + R + a*C
  float w;             // tap weight
  int R0, R1, C0, C1;  // clip rectangle on the FPA, half-open, inside the tile
  int full;            // rectangle covers the whole tile: no per-pixel test
  int pad;
};
static_assert(sizeof(FwdEntry) == 32, "FwdEntry must stay 32 bytes");

// ---------------------------------------------------------------------------
// Back projection (voxel-stationary gather from r).
// z_lam[r, c] = sum_t w_t * r[(r + gamma*c + o_t) mod n]   (Eqs. 14-15)
constexpr int kBackTileR = 32;  // voxel rows per CTA (one warp lane each)
constexpr int kBackTileC = 8;   // voxel columns per CTA (one warp each)
constexpr int kBackBands = 4;   // bands per CTA
constexpr int kBackThreads = kBackTileR * kBackTileC;

struct DevTables {
  // forward
  const FwdEntry* fwd_entries;
  const int* fwd_tile_ptr;     // tiles+1
  int tiles_r, tiles_c;
  // back: taps per band, offsets/weights padded to a multiple of 4 per band
  const int* band_ptr4;        // w+1, start of band lam in the padded arrays (multiple of 4)
  const int* band_cnt;         // w, real tap count of band lam
  const int* tap_off;          // padded, int32 offsets in [0, n)
  const float* tap_w;          // padded
  const float* inv_h;          // w, 1/h_lam (float32)
  const float* h;              // w, h_lam (float32)
};

struct Dims {
  int a, alpha, w, gamma, xi;
  int n, ell, m;
};

// Kernel launchers (ctis_kernels.cu).  All return the cudaGetLastError() of the launch.
cudaError_t launch_forward(const Dims& d, const DevTables& t, const float* f, const float* g,
                           float* out, int frames, bool ratio, cudaStream_t s);
enum BackMode { kBackOnly = 0, kBackUpdate = 1 };
cudaError_t launch_back(const Dims& d, const DevTables& t, const float* r, float* fz, int frames,
                        BackMode mode, cudaStream_t s);
cudaError_t launch_sensitivity(const Dims& d, const DevTables& t, float* h, cudaStream_t s);
cudaError_t launch_ratio(const float* g, const float* ghat, float* r, int64_t count, cudaStream_t s);
cudaError_t launch_validate(const float* x, int64_t count, int* flag, cudaStream_t s);

}  // namespace ctis
