// Internal declarations shared by the plan builder (ctis_api.cu), the per-plan
// table kernels (ctis_tables.cu -> embedded cubin) and the element-wise kernels
// (ctis_kernels.cu).  Not part of the public ABI (include/ctis.h is).
#pragma once

#include <stdint.h>

namespace ctis {

// ---------------------------------------------------------------------------
// Tap tables live in __constant__ memory ("pages" of 64 KB).  Every plan loads
// its own instance of the table-kernel cubin per page (cudaLibraryLoadData), so
// each page is private to the plan.  Kernels read taps through the uniform
// datapath (LDCU -> FFMA R, R, UR, R): tap metadata costs no L1/SMEM bandwidth.
constexpr int kPageWords = 16384;  // 64 KB of uint32

// Page layout (uint32 words; descriptors and tap entries start at multiples of 4 words):
//   [0]       number of chunks in the page (<= 63)
//   [1 + k]   word offset of chunk k's descriptor
//   [kItemBase + k]  work items (tiles) of chunks 0..k-1 (prefix sums); [kItemBase + nch] = total
//
// Forward chunk descriptor (Eq. 12 evaluated per "mode"):
//   [D+0] lam0   [D+1] nb   [D+2] nm   [D+3] u_r0   [D+4] u_c0   [D+5] tiles_r   [D+6] tiles_c  [D+7] G*MAXM
//   [D+8 ..]            o_ref[c]                     (nm words rounded up to a multiple of 4, in [0, n))
//   [BI = D+8+nm4 ..]   per band b: row0_rel, col0_rel, WR, WC   (window rows/cols relative to the tile)
//   [TP = BI+4*nb ..]   per band b and mode pair (2k, 2k+1) of the pass (G*MAXM modes): one 16-byte
//                       entry (off_2k, off_2k+1, w_2k, w_2k+1) at TP + 4*(b*G*MAXM/2 + k); group g
//                       owns pairs [g*MAXM/2, (g+1)*MAXM/2); w = 0 -> no tap
// Back chunk descriptor (Eqs. 14-15):
//   [D+0] lam0   [D+1] nb   [D+2] nm   [D+3] tiles_r   [D+4] tiles_c   [D+5] NB   [D+6..7] 0
//   [MI = D+8 ..]       per mode c: Bm_r, Bm_c, WR, WC  (window origin term Bm = Bm_r + gamma*Bm_c in [0, n))
//   [TP = MI+4*nm ..]   per mode c and band pair (2k, 2k+1): 16-byte entry (off_2k, off_2k+1,
//                       w_2k, w_2k+1) at TP + 4*(c*NB/2 + k)
//   [IH = TP+2*nm*NB ..] inv_h[b]
enum : int { kDescHeader = 8, kItemBase = 64, kPageHeaderWords = 128 };

// Forward kernel geometry: one u-space position per thread, 32 rows x 16 columns per CTA; a CTA
// has G in {1, 2} groups of kFwdThreads threads that share each window and split the modes.
constexpr int kFwdTR = 32;
constexpr int kFwdTC = 16;
constexpr int kFwdThreads = kFwdTR * kFwdTC;   // per group
constexpr int kFwd2Threads = kFwdThreads / 2;  // two u positions per thread (forward_persistent2)
constexpr int kFwdBands = 16;           // default max bands per forward chunk (chunks are balanced)
// Back kernel geometry: 32 x 32 voxel tile, 2 voxels per thread, NB in {2, 4, 8, 12, 16} bands
// per chunk (kernel template; the plan picks the one that fills the 148 SMs best).
constexpr int kBackTR = 32;
constexpr int kBackTC = 32;
constexpr int kBackThreads = 512;
constexpr int kBack4Threads = 256;  // back_persistent4: four voxels per thread
constexpr int kBackBandsMax = 16;

// Mode shifts are bounded by the plan's span (|dr|, |dc| <= span from the mode reference; default
// kModeSpanDefault, at most kModeSpanMax), so an element-loader window never exceeds
// (32 + 2*span) x (16 + 2*span) floats (forward) or (32 + 2*span) x (32 + 2*span) (back).
constexpr int kModeSpanDefault = 12;
constexpr int kModeSpanMax = 32;
// TMA forward plans: longer chunks with a wider mode span (fewer chunks -> fewer flush atomics)
constexpr int kFwdBandsTma = 25;
constexpr int kModeSpanTma = 16;
constexpr int kFwdStages = 8;           // window pipeline depth (TMA boxes / cp.async groups in flight),
#ifndef CTIS_BACK_STAGES
#define CTIS_BACK_STAGES 8
#endif
constexpr int kBackStages = CTIS_BACK_STAGES;  // back ring depth (refilled every CTIS_BACK_K windows)
constexpr int kFwdWinFloats = 2560;     // element-loader slot: 10 KB per stage (>= 56 x 40)
constexpr int kTmaWinFloats = 8192;     // TMA box cap (32 KB)
constexpr int kBackWinFloats = 3584;    // 14 KB per stage (>= 60 x 56)

// Strip forward (forward_strip, TMA plans whose modes share column drifts — every diffraction order
// (p, q) of a band chunk drifts by (p, q) * d'(lambda), so the orders of one q column move together):
// a warp owns a 32 x 16 u-tile as 32 strips of kStripP consecutive rows (lane = rs + 2*column) and a
// "strip group" of <= kStripMG modes with identical column shifts.  Per band it loads ONE register
// strip of <= 4*kStripNQ window rows and every mode of the group reads its 16 rows from it at its own
// row offset o in [0, kStripNO): one shared-memory word feeds ~2.4 FMAs instead of one.
//
// Strip chunk descriptor (forward pages with kind = strip):
//   [D+0] lam0 [D+1] nb [D+2] nhg (strip groups = consumer warps used) [D+3] u_r0 [D+4] u_c0
//   [D+5] tiles_r [D+6] tiles_c [D+7] 0
//   [D+8 ..]          o_ref[g*kStripMG + k] (0xffffffff: empty slot)     (4*nhg words)
//   [D+8+4*nhg ..]    the same references as ref_row | ref_col << 16     (4*nhg words)
//   [BI ..]           per band: row0_rel, col0_rel, 0, 0
//   [TP = BI+4*nb ..] per band b and group g: 8 words at TP + 8*(b*nhg + g):
//                     [0] strip byte offset into the window (thread base excluded), [1] row offset o_k
//                     of slot k in byte k (kStripNO: no tap), [2..5] w_k, [6..7] 0
constexpr int kStripP = 16;   // rows per thread strip
constexpr int kStripMG = 4;   // modes per strip group (accumulators: kStripMG x kStripP per thread)
constexpr int kStripNQ = 10;  // max float4 loads per strip (40 window rows)
constexpr int kStripNO = 4 * kStripNQ - kStripP + 1;  // row offsets 0..24 (one code block per offset)
constexpr int kStripWarpsMax = 14;  // consumer warps per CTA (+ 1 TMA producer warp): <= 136 registers
constexpr int kStripStagesMax = 8;  // ring depth: as many window slots as shared memory holds (<= 8)
constexpr int kStripStage = kStripMG * 512;  // flush staging floats per warp (kStripMG tiles of 16 x 32)

// Per-launch parameters of the table kernels.
struct TabArgs {
  const float* src;    // forward: f; back: r
  float* dst;          // forward: g_hat (accumulated with red.add); back: f (updated) or z
  long long src_frame; // elements between frames in src
  long long dst_frame; // elements between frames in dst
  int a, alpha, gamma, xi, n, ell;
  int mode;            // back: 0 = write z, 1 = MLEM update of f in place, 2 = SMART update
  unsigned bias;       // forward: multiple of n with E(u) + bias >= 0 for every u of the u-space
  int nsub;            // forward: E(u) + bias + o_ref < (nsub + 1) * n
  int slot_floats;     // floats per pipeline slot (multiple of 32)
  int box_r, box_c;    // TMA box (window) rows x columns; the window pitch is box_r
  unsigned box_bytes;  // 4 * box_r * box_c
  int dbg;             // profiling switches (CTIS_DEBUG env): 1 = no TMA (compute on stale windows), 2 = no flush
  int frames;          // persistent kernels: frames in the launch (items = frames x page items)
  int nowrap;          // every tap is a plain 2-D translation inside the FPA (no carry / wrap of Eq. 7)
  // fused ratio (persistent TMA forward, last page of the projection): after a grid-wide barrier,
  // dst[i] <- ratio(meas[i], dst[i]) for i < ratio_count (1: g / g_hat, 0 where g_hat <= 0 — Alg. 1
  // line 8, reading R4; 2: SMART log-ratio, reading R17; 0: none)
  int ratio_mode;
  const float* meas;   // g
  long long ratio_count;
  unsigned* gbar;      // grid barrier word (zero-initialised once, self-resetting)
  // back kernel: zero zero_count floats at zero_buf (the next iteration's g_hat accumulator)
  float* zero_buf;
  long long zero_count;
  // strip forward: flush accumulator tiles with TMA bulk reduce-add through the g_hat tensor map
  // (nowrap plans with 16-byte FPA column strides); otherwise red.global.add with modular indices
  int tma_flush;
  int stages;          // strip forward: window ring depth (<= kStripStagesMax)
};

}  // namespace ctis
