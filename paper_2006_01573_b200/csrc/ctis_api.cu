// ctis_api.cu — the C ABI of libctis (include/ctis.h): plan builder (tap validation,
// mode clustering, __constant__ tap pages), stream-ordered entry points, CUDA-graph
// replay of the MLEM iterations.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ctis.h"
#include "ctis_comm.h"
#include "ctis_nvls.h"
#include "ctis_internal.h"
#include "ctis_fft.h"
#include "ctis_kernels.h"
// the projection-kernel cubin, embedded by build/ctis_tables_blob.S (.incbin)
extern "C" const unsigned char ctis_tables_cubin[], ctis_tables_cubin_end[];

using namespace ctis;

namespace {

thread_local std::string g_last_error;

ctis_status fail(ctis_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

ctis_status cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return e == cudaErrorMemoryAllocation ? CTIS_ERR_OUT_OF_MEMORY : CTIS_ERR_CUDA;
}

#define CTIS_CUDA(call, where)                            \
  do {                                                    \
    cudaError_t e__ = (call);                             \
    if (e__ != cudaSuccess) return cuda_fail(e__, where); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

struct GraphKey {
  const void* g;
  void* f;
  void* ws;
  int64_t frames;
  int iters;
  int solver;  // 0 MLEM, 1 SMART
  bool operator<(const GraphKey& o) const {
    return std::tie(g, f, ws, frames, iters, solver) < std::tie(o.g, o.f, o.ws, o.frames, o.iters, o.solver);
  }
};

// Monitored MLEM graphs (conditional WHILE node) are keyed by every buffer and parameter they bake in.
struct MonKey {
  const void* g;
  void* f;
  void* ws;
  void* ll;
  void* cnt;
  int max_iters;
  double tol;
  bool operator<(const MonKey& o) const {
    return std::tie(g, f, ws, ll, cnt, max_iters, tol) < std::tie(o.g, o.f, o.ws, o.ll, o.cnt, o.max_iters, o.tol);
  }
};

// One 64 KB __constant__ page of tap tables and the library instance that owns it.
struct Page {
  bool forward = true;
  bool pair = false;
  int nchunks = 0;
  int max_tiles = 0;
  int max_modes = 0;
  int total_items = 0;  // tiles summed over the page's chunks (persistent kernels)
  int back_tc = 32;     // back pages: tile columns (kernel family)
  bool strip = false;   // forward pages: strip kernel (ctis_fwd_strip_t)
  int strip_warps = 0;  // strip pages: consumer warps (max strip groups over the page's chunks)
  std::vector<uint32_t> words;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
};

constexpr int kPageHeader = kPageHeaderWords;  // nchunks, descriptor offsets, item prefix sums

}  // namespace

struct ctis_plan_s {
  int device = 0;
  int a = 0, alpha = 0, w = 0, gamma = 0, xi = 0, n = 0, ell = 0, m = 0;
  int64_t band_begin = 0, band_end = 0, total_taps = 0;
  int64_t ex_lo = 0, ex_hi = 0;  // FPA index range any tap of any band reaches (latency-mode exchange)
  // Reachable FPA box of a no-wrap plan (every tap a 2-D translation): pixel rows [rb_r0, rb_r0 + 4*rb_nr4)
  // x columns [rb_c0, rb_c0 + rb_nc) hold every pixel E(q) + o of every voxel and tap; outside it g_hat
  // is identically 0, r is 0 (reading R4) and no back projection reads r, so the MLEM ratio pass only
  // runs over the box (rb_nr4 = 0: the whole FPA)
  int rb_r0 = 0, rb_nr4 = 0, rb_c0 = 0, rb_nc = 0;
  bool shard = false, validate = true, use_graph = true;
  bool tma_f = false, tma_b = false;
  int back_nb = kBackBandsMax;
  int back_tc = kBackTC;  // back tile columns: 32, or 16 for small TMA plans (ctis_back2_*)
  int fbox_r = 0, fbox_c = 0, bbox_r = 0, bbox_c = 0;
  int fwd_g = 1, fwd_m = 8;
  bool fwd_strip = false;  // forward pages use the strip kernel (ctis_tables.cu forward_strip)
  // TMA forward with a field stop whose rows are not a multiple of 4 floats (a % 4 != 0, e.g. the paper's
  // own 89 x 80): f is repacked into d_fpad with a 16-byte row pitch f_pitch = round4(a) before
  // each forward launch (the TMA view keeps dims a x alpha, so the pad rows are never read)
  int f_pitch = 0;
  float* d_fpad = nullptr;
  size_t fpad_cap = 0;  // floats
  // Mode-split back projection for latency-bound small plans (too few tile x band-chunk work items to fill
  // the SMs): every chunk's modes are cut into back_split descriptors that add their partial z into d_z
  // (red.add, TabArgs::mode 3); one update pass then applies Eq. 2's multiplicative step and re-zeroes d_z
  int back_split = 1;
  float* d_z = nullptr;
  size_t z_cap = 0;         // floats
  float* d_invh = nullptr;  // 1/h_lambda (fp32, the epilogue's values) for the update pass
  int sms = 148;
  bool pair = false;  // FFMA2 on tap pairs (16-byte entries) or plain FFMA (8-byte entries)
  bool nowrap = false;  // no tap carries across FPA columns or wraps past n (2-D translations only)
  std::vector<Page> fwd, back;
  float* d_hband = nullptr;
  int* d_flag = nullptr;
  float* d_g = nullptr;  // host-buffer path
  float* d_f = nullptr;
  void* d_ws = nullptr;
  int64_t host_frames = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, int64_t> graph_launches;  // kernels inside each cached graph
  std::map<MonKey, cudaGraphExec_t> mon_graphs;
  std::map<GraphKey, cudaGraphExec_t> shard_graphs;  // band-sharded iterations (key.frames = comm id)
  int projector = 0;                 // CTIS_OPT_PROJECTOR: 0 taps (default), 1 the paper's FFT route
  ctis::FftState* fft = nullptr;     // created when the FFT projector is selected
  std::vector<std::vector<std::pair<int64_t, float>>> band_taps;  // (offset, weight) per local band
  std::vector<float> inv_h;          // 1 / h_lambda per local band
  int64_t last_launches = 0;
  bool fused_ratio = false;    // CTIS_OPT_FUSED_RATIO (measured slower: DESIGN.md)
  int exchange = 0;            // CTIS_OPT_EXCHANGE: 0 NCCL collectives, 1 fused NVLink kernel
  // Throughput layout for many-frame launches: the single-frame layout shortens forward chunks and back
  // band chunks until one frame fills the SMs; with enough frames the longer chunks (fewer flushes, NB = 12
  // bands per r window) win.  A second plan over the same taps, used by batched calls (nullptr if the
  // layouts coincide).
  bool throughput = false;     // this plan IS a throughput layout
  ctis_plan_s* tput = nullptr;
  unsigned* d_gbar = nullptr;  // grid barrier word of the cooperative forward launches
  std::mutex mu;

  ~ctis_plan_s() {
    delete tput;
    DeviceGuard dg(device);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : mon_graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : shard_graphs) cudaGraphExecDestroy(kv.second);
    ctis::fft_destroy(fft);
    if (side) cudaStreamDestroy(side);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    for (auto* pages : {&fwd, &back})
      for (Page& p : *pages)
        if (p.lib) cudaLibraryUnload(p.lib);
    for (void* p : {(void*)d_hband, (void*)d_flag, (void*)d_g, (void*)d_f, d_ws, (void*)d_gbar, (void*)d_fpad, (void*)d_z, (void*)d_invh})
      if (p) cudaFree(p);
  }
};

struct ctis_comm_s {
  void* nccl = nullptr;
  int nranks = 1, rank = 0, device = 0;
  ctis::NvlsComm nvls;  // symmetric exchange window + device communicator (CTIS_OPT_EXCHANGE = 1)
  ~ctis_comm_s() {
    ctis::nvls_teardown(nccl, &nvls);
    ctis::nccl_comm_destroy(nccl);
  }
};

namespace {

// ------------------------------------------------------------------------------------------------
// Mode clustering.  Within a chunk of consecutive bands, taps that drift together from band to
// band (the same diffraction order at slightly different dispersion) are grouped into a "mode"
// with a reference offset o_ref; every tap is then o = o_ref + dr + gamma*dc with a small 2-D
// shift (dr, dc).  Any assignment is exact (the identity is integer arithmetic); clustering only
// decides how much shared-memory window each kernel stages.
struct TapXY {
  int dr, dc;  // o = dr + gamma * dc, 0 <= dr < gamma
  float w;
};
struct ModeTap {
  int b, dr, dc;
  float w;
};
struct Mode {
  int ref_dr, ref_dc;
  int lo_dr, lo_dc, hi_dr, hi_dc;  // last matched position below / above the reference band
  std::vector<ModeTap> taps;
  std::vector<char> has;
};

constexpr int kModeTrack = 3;   // max band-to-band move of a mode (pixels, Chebyshev)

// span: max |shift| of a tap from its mode reference (pixels, Chebyshev)
std::vector<Mode> cluster_modes(const std::vector<std::vector<TapXY>>& bands, int span = kModeSpanDefault) {
  const int nb = (int)bands.size();
  const int bref = (nb - 1) / 2;
  std::vector<Mode> modes;
  auto add_mode = [&](int b, const TapXY& t) {
    Mode md;
    md.ref_dr = md.lo_dr = md.hi_dr = t.dr;
    md.ref_dc = md.lo_dc = md.hi_dc = t.dc;
    md.has.assign(nb, 0);
    md.has[b] = 1;
    md.taps.push_back(ModeTap{b, t.dr, t.dc, t.w});
    modes.push_back(std::move(md));
  };
  for (const TapXY& t : bands[bref]) add_mode(bref, t);
  std::vector<int> order;
  for (int d = 1; d < nb; ++d) {
    if (bref + d < nb) order.push_back(bref + d);
    if (bref - d >= 0) order.push_back(bref - d);
  }
  for (int b : order) {
    const bool up = b > bref;
    for (const TapXY& t : bands[b]) {
      int best = -1, bestd = INT_MAX;
      for (int i = 0; i < (int)modes.size(); ++i) {
        Mode& md = modes[i];
        if (md.has[b]) continue;
        const int ldr = up ? md.hi_dr : md.lo_dr, ldc = up ? md.hi_dc : md.lo_dc;
        const int d = std::max(std::abs(t.dr - ldr), std::abs(t.dc - ldc));
        const int s = std::max(std::abs(t.dr - md.ref_dr), std::abs(t.dc - md.ref_dc));
        if (d <= kModeTrack && s <= span && d < bestd) {
          best = i;
          bestd = d;
        }
      }
      if (best < 0) {
        add_mode(b, t);
        continue;
      }
      Mode& md = modes[best];
      md.has[b] = 1;
      md.taps.push_back(ModeTap{b, t.dr, t.dc, t.w});
      if (up) {
        md.hi_dr = t.dr;
        md.hi_dc = t.dc;
      } else {
        md.lo_dr = t.dr;
        md.lo_dc = t.dc;
      }
    }
  }
  return modes;
}

inline int round4(int x) { return (x + 3) & ~3; }
inline uint32_t fbits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return u;
}

// Per-band (forward) or per-mode (back) shift ranges.
struct Span {
  int rmin = INT_MAX, rmax = INT_MIN, cmin = INT_MAX, cmax = INT_MIN;
  void add(int dr, int dc) {
    rmin = std::min(rmin, dr);
    rmax = std::max(rmax, dr);
    cmin = std::min(cmin, dc);
    cmax = std::max(cmax, dc);
  }
  bool empty() const { return rmin == INT_MAX; }
};

std::vector<Span> band_spans(int nb, const std::vector<const Mode*>& ms) {
  std::vector<Span> sp(nb);
  for (const Mode* md : ms)
    for (const ModeTap& t : md->taps) sp[t.b].add(t.dr - md->ref_dr, t.dc - md->ref_dc);
  return sp;
}

Span mode_span(const Mode& md) {
  Span s;
  for (const ModeTap& t : md.taps) s.add(t.dr - md.ref_dr, t.dc - md.ref_dc);
  return s;
}

// Forward chunk descriptor for bands [b0, b0+nb) (local) and the given modes.  box_r > 0 selects
// the TMA layout (every window is a box_r x box_c box with pitch box_r); box_r == 0 the element
// loader layout (exact per-band window, pitch = its own row count).
bool forward_desc(const ctis_plan_s& P, int b0, int nb, const std::vector<const Mode*>& ms, int maxm, int box_r,
                  int box_c, std::vector<uint32_t>& out, int& tiles) {
  const int nm = (int)ms.size();
  const std::vector<Span> sp = band_spans(nb, ms);
  Span all;
  for (const Span& x : sp)
    if (!x.empty()) {
      all.add(x.rmin, x.cmin);
      all.add(x.rmax, x.cmax);
    }
  if (all.empty()) return true;  // no taps: nothing to emit
  const int tiles_r = (P.a + all.rmax - all.rmin + kFwdTR - 1) / kFwdTR;
  const int tiles_c = (P.alpha + all.cmax - all.cmin + kFwdTC - 1) / kFwdTC;
  const int nm2 = (nm + 3) & ~3;  // keeps the tap-pair entries 16-byte aligned
  out.assign(kDescHeader + nm2 + 4 * nb + 2 * nb * maxm, 0u);
  out[0] = (uint32_t)b0;
  out[1] = (uint32_t)nb;
  out[2] = (uint32_t)nm;
  out[3] = (uint32_t)all.rmin;
  out[4] = (uint32_t)all.cmin;
  out[5] = (uint32_t)tiles_r;
  out[6] = (uint32_t)tiles_c;
  out[7] = (uint32_t)maxm;
  for (int c = 0; c < nm; ++c) out[kDescHeader + c] = (uint32_t)(ms[c]->ref_dr + P.gamma * ms[c]->ref_dc);
  const int BI = kDescHeader + nm2, TP = BI + 4 * nb;
  std::vector<int> WRs(nb, 1), lead(nb, 0);
  for (int b = 0; b < nb; ++b) {
    if (sp[b].empty()) {  // band without taps in this pass: never read, but the TMA box origin
      // must still be 16-byte aligned (row origin all.rmin + 32k - lead = multiple of 4)
      out[BI + 4 * b + 0] = (uint32_t)(-(int)((((long long)all.rmin % 4) + 4) % 4));
      out[BI + 4 * b + 1] = 0u;
      out[BI + 4 * b + 2] = (uint32_t)std::max(box_r, 1);
      out[BI + 4 * b + 3] = box_r ? (uint32_t)box_c : 0u;
      continue;
    }
    // TMA: the innermost box coordinate must be a multiple of 4 floats (16 bytes); the tile row
    // origin is all.rmin + 32*k, so start the window `lead` rows early.
    lead[b] = box_r ? (int)((((long long)all.rmin - sp[b].rmax) % 4 + 4) % 4) : 0;
    const int WR = box_r ? box_r : kFwdTR + sp[b].rmax - sp[b].rmin;
    const int WC = box_r ? box_c : kFwdTC + sp[b].cmax - sp[b].cmin;
    if (WR * WC > (box_r ? kTmaWinFloats : kFwdWinFloats) ||
        (box_r && kFwdTR + sp[b].rmax - sp[b].rmin + lead[b] > box_r))
      return false;
    WRs[b] = WR;
    out[BI + 4 * b + 0] = (uint32_t)(-sp[b].rmax - lead[b]);
    out[BI + 4 * b + 1] = (uint32_t)(-sp[b].cmax);
    out[BI + 4 * b + 2] = (uint32_t)WR;
    out[BI + 4 * b + 3] = (uint32_t)WC;
  }
  for (int c = 0; c < nm; ++c)
    for (const ModeTap& t : ms[c]->taps) {
      const int dr = t.dr - ms[c]->ref_dr, dc = t.dc - ms[c]->ref_dc;
      const int off = (sp[t.b].rmax + lead[t.b] - dr) + WRs[t.b] * (sp[t.b].cmax - dc);
      // pair layout: (off_{2k}, off_{2k+1}, w_{2k}, w_{2k+1}) of modes 2k, 2k+1 in band b (FFMA2);
      // plain layout: (off_c, w_c) per mode
      const int wi = P.pair ? TP + 4 * (t.b * (maxm / 2) + c / 2) + (c & 1) : TP + 2 * (t.b * maxm + c);
      out[wi] = (uint32_t)(4 * off);
      out[wi + (P.pair ? 2 : 1)] = fbits(t.w);
    }
  tiles = tiles_r * tiles_c;
  return true;
}

// Back chunk descriptor for bands [b0, b0+nb) (local) and all modes of the chunk (same layouts).
bool back_desc(const ctis_plan_s& P, int b0, int nb, int NB, const std::vector<Mode>& ms,
               const std::vector<float>& invh, int box_r, int box_c, std::vector<uint32_t>& out, int& tiles) {
  const int nm = (int)ms.size();
  out.assign(kDescHeader + 4 * nm + 2 * nm * NB + ((nb + 3) & ~3), 0u);  // length % 4 == 0
  const int tiles_r = (P.a + kBackTR - 1) / kBackTR, tiles_c = (P.alpha + P.back_tc - 1) / P.back_tc;
  out[0] = (uint32_t)b0;
  out[1] = (uint32_t)nb;
  out[2] = (uint32_t)nm;
  out[3] = (uint32_t)tiles_r;
  out[4] = (uint32_t)tiles_c;
  out[5] = (uint32_t)NB;
  const int MI = kDescHeader, TP = MI + 4 * nm, IH = TP + 2 * nm * NB;
  for (int c = 0; c < nm; ++c) {
    const Mode& md = ms[c];
    const Span sp = mode_span(md);
    const long long oref = (long long)md.ref_dr + (long long)P.gamma * md.ref_dc;
    const long long B0 = oref + sp.rmin + (long long)P.gamma * sp.cmin;
    // TMA: the window's FPA row origin (B mod gamma; gamma % 4 == 0 and tile origins are multiples
    // of 32) must be a multiple of 4, so start `lead` rows early.
    const int lead = box_r ? (int)(((B0 % 4) + 4) % 4) : 0;
    long long Bm = (B0 - lead) % P.n;
    if (Bm < 0) Bm += P.n;
    const int WR = box_r ? box_r : kBackTR + sp.rmax - sp.rmin;
    const int WC = box_r ? box_c : kBackTC + sp.cmax - sp.cmin;
    if (WR * WC > kBackWinFloats || (box_r && kBackTR + sp.rmax - sp.rmin + lead > box_r)) return false;
    out[MI + 4 * c + 0] = (uint32_t)(Bm % P.gamma);
    out[MI + 4 * c + 1] = (uint32_t)(Bm / P.gamma);
    out[MI + 4 * c + 2] = (uint32_t)WR;
    out[MI + 4 * c + 3] = (uint32_t)WC;
    for (const ModeTap& t : md.taps) {
      const int dr = t.dr - md.ref_dr, dc = t.dc - md.ref_dc;
      // pair layout (off_{2k}, off_{2k+1}, w_{2k}, w_{2k+1}) of bands 2k, 2k+1 (FFMA2); plain (off, w)
      const int wi = P.pair ? TP + 4 * (c * (NB / 2) + t.b / 2) + (t.b & 1) : TP + 2 * (c * NB + t.b);
      out[wi] = (uint32_t)(4 * ((dr - sp.rmin + lead) + WR * (dc - sp.cmin)));
      out[wi + (P.pair ? 2 : 1)] = fbits(t.w);
    }
  }
  for (int b = 0; b < nb; ++b) out[IH + b] = fbits(invh[b0 + b]);
  tiles = tiles_r * tiles_c;
  return true;
}

// Append descriptors to pages (<= 64 KB and <= 63 chunks each).
void pack_pages(std::vector<Page>& pages, bool forward, const std::vector<std::vector<uint32_t>>& descs,
                const std::vector<int>& tiles, const std::vector<int>& modes) {
  Page cur;
  auto flush = [&]() {
    if (cur.nchunks) pages.push_back(std::move(cur));
    cur = Page();
  };
  for (size_t i = 0; i < descs.size(); ++i) {
    if (cur.nchunks == 0) {
      cur.forward = forward;
      cur.words.assign(kPageHeader, 0u);
    }
    if (cur.nchunks == kItemBase - 1 || cur.words.size() + descs[i].size() > (size_t)kPageWords) {
      flush();
      cur.forward = forward;
      cur.words.assign(kPageHeader, 0u);
    }
    cur.words[1 + cur.nchunks] = (uint32_t)cur.words.size();
    cur.words[kItemBase + cur.nchunks + 1] = cur.words[kItemBase + cur.nchunks] + (uint32_t)tiles[i];
    cur.total_items += tiles[i];
    cur.words.insert(cur.words.end(), descs[i].begin(), descs[i].end());
    cur.nchunks++;
    cur.words[0] = (uint32_t)cur.nchunks;
    cur.max_tiles = std::max(cur.max_tiles, tiles[i]);
    cur.max_modes = std::max(cur.max_modes, modes[i]);
  }
  flush();
}

// ------------------------------------------------------------------------------------------------
// Strip forward layout (ctis_internal.h "Strip forward").  Modes of a chunk whose column shift
// dc (relative to the mode reference) is identical in every band form a column group; a column
// group is cut into strip groups of <= kStripMG modes, sorted along their drift, such that in
// every band the row offsets of the group's taps span at most kStripNO - 1 rows of one strip.
struct StripGroup {
  std::vector<const Mode*> ms;
};

// per band, per mode: row / column of the window that position 0 of the u strip reads
struct StripPass {
  int b0 = 0, nb = 0;
  std::vector<StripGroup> groups;
};

std::vector<StripGroup> strip_groups(int nb, const std::vector<Mode>& modes) {
  const int bref = (nb - 1) / 2;
  // column signature: dc relative to the reference per band (INT_MIN where the mode has no tap)
  std::map<std::vector<int>, std::vector<const Mode*>> cols;
  for (const Mode& md : modes) {
    std::vector<int> sig(nb, INT_MIN);
    for (const ModeTap& t : md.taps) sig[t.b] = t.dc - md.ref_dc;
    cols[sig].push_back(&md);
  }
  std::vector<StripGroup> out;
  for (auto& kv : cols) {
    std::vector<const Mode*> ms = kv.second;
    // order along the drift: sum_b (b - bref) * dr_rel (modes of one diffraction-order column
    // line up by order index p)
    auto key = [&](const Mode* md) {
      long long k = 0;
      for (const ModeTap& t : md->taps) k += (long long)(t.b - bref) * (t.dr - md->ref_dr);
      return k;
    };
    std::stable_sort(ms.begin(), ms.end(), [&](const Mode* x, const Mode* y) { return key(x) < key(y); });
    // greedy cut: extend the current group while every band's row-offset range (incl. 4-row
    // alignment of the strip start) stays within kStripNO - 1
    std::vector<int> lo(nb, INT_MAX), hi(nb, INT_MIN);
    StripGroup cur;
    auto fits = [&](const Mode* md) {
      if ((int)cur.ms.size() >= kStripMG) return false;
      for (const ModeTap& t : md->taps) {
        const int d = t.dr - md->ref_dr;
        const int l = std::min(lo[t.b], d), h = std::max(hi[t.b], d);
        if (h - l + 3 > kStripNO - 1) return false;
      }
      return true;
    };
    for (const Mode* md : ms) {
      if (!fits(md)) {
        out.push_back(cur);
        cur = StripGroup();
        std::fill(lo.begin(), lo.end(), INT_MAX);
        std::fill(hi.begin(), hi.end(), INT_MIN);
      }
      cur.ms.push_back(md);
      for (const ModeTap& t : md->taps) {
        const int d = t.dr - md->ref_dr;
        lo[t.b] = std::min(lo[t.b], d);
        hi[t.b] = std::max(hi[t.b], d);
      }
    }
    if (!cur.ms.empty()) out.push_back(cur);
  }
  return out;
}

// Strip chunk descriptor for one pass (bands [b0, b0+nb), its strip groups); box_r / box_c are the
// plan's TMA box.  need_r / need_c report the box this pass needs (first call with box_r = 0).
bool strip_desc(const ctis_plan_s& P, const StripPass& ps, int box_r, std::vector<uint32_t>& out, int& tiles,
                int& need_r, int& need_c) {
  const int nb = ps.nb, nhg = (int)ps.groups.size();
  std::vector<const Mode*> all_ms;
  for (const StripGroup& g : ps.groups) all_ms.insert(all_ms.end(), g.ms.begin(), g.ms.end());
  const std::vector<Span> sp = band_spans(nb, all_ms);
  Span all;
  for (const Span& x : sp)
    if (!x.empty()) {
      all.add(x.rmin, x.cmin);
      all.add(x.rmax, x.cmax);
    }
  out.clear();
  tiles = 0;
  need_r = need_c = 0;
  if (all.empty()) return true;
  // u-tile row origins u_r0 + 32k are multiples of 4 and so are the mode reference rows
  // (build_strip_forward): every flush box starts on a 16-byte FPA row boundary (TMA reduce)
  all.rmin = (int)std::floor(all.rmin / 4.0) * 4;
  const int tiles_r = (P.a + all.rmax - all.rmin + kFwdTR - 1) / kFwdTR;
  const int tiles_c = (P.alpha + all.cmax - all.cmin + kFwdTC - 1) / kFwdTC;
  const int BI = kDescHeader + 2 * kStripMG * nhg, TP = BI + 4 * nb;
  out.assign(TP + 8 * nb * nhg, 0u);
  out[0] = (uint32_t)ps.b0;
  out[1] = (uint32_t)nb;
  out[2] = (uint32_t)nhg;
  out[3] = (uint32_t)all.rmin;
  out[4] = (uint32_t)all.cmin;
  out[5] = (uint32_t)tiles_r;
  out[6] = (uint32_t)tiles_c;
  for (int g = 0; g < nhg; ++g)
    for (int k = 0; k < kStripMG; ++k) {
      const Mode* md = k < (int)ps.groups[g].ms.size() ? ps.groups[g].ms[k] : nullptr;
      out[kDescHeader + kStripMG * g + k] = md ? (uint32_t)(md->ref_dr + P.gamma * md->ref_dc) : 0xffffffffu;
      // the same reference as (row, column) for the TMA flush box (no division in the kernel)
      out[kDescHeader + kStripMG * (nhg + g) + k] = md ? (uint32_t)md->ref_dr | ((uint32_t)md->ref_dc << 16) : 0u;
    }
  for (int b = 0; b < nb; ++b) {
    // TMA box row origin all.rmin + 32k + row0_rel must be a multiple of 4 (see forward_desc)
    const int rmax = sp[b].empty() ? 0 : sp[b].rmax, cmax = sp[b].empty() ? 0 : sp[b].cmax;
    const int lead = (int)((((long long)all.rmin - rmax) % 4 + 4) % 4);
    out[BI + 4 * b + 0] = (uint32_t)(-rmax - lead);
    out[BI + 4 * b + 1] = (uint32_t)(-cmax);
    if (!sp[b].empty()) need_c = std::max(need_c, kFwdTC + sp[b].cmax - sp[b].cmin);
    for (int g = 0; g < nhg; ++g) {
      const int e = TP + 8 * (b * nhg + g);
      out[e + 1] = 0x01010101u * (uint32_t)kStripNO;  // every slot skips
      int rlo = INT_MAX, rhi = INT_MIN, ccol = INT_MIN;
      int R[kStripMG];
      float W[kStripMG];
      for (int k = 0; k < kStripMG; ++k) R[k] = INT_MIN, W[k] = 0.f;
      for (int k = 0; k < (int)ps.groups[g].ms.size(); ++k) {
        const Mode* md = ps.groups[g].ms[k];
        for (const ModeTap& t : md->taps) {
          if (t.b != b) continue;
          const int c = cmax - (t.dc - md->ref_dc);
          if (ccol != INT_MIN && c != ccol) return false;  // column groups share dc by construction
          ccol = c;
          R[k] = rmax + lead - (t.dr - md->ref_dr);
          W[k] = t.w;
          rlo = std::min(rlo, R[k]);
          rhi = std::max(rhi, R[k]);
        }
      }
      if (ccol == INT_MIN) continue;  // no tap of this group in band b: nq = 0, every slot skipped
      const int lo4 = rlo & ~3;
      const int nq = (rhi - lo4 + kStripP + 3) / 4;
      if (nq > kStripNQ) return false;
      // the kernel always loads kStripNQ float4 per strip; rows past the group's range may run into the
      // next window column or past the slot (into the next slot or the staging area): never used
      need_r = std::max(need_r, kStripP + lo4 + 4 * nq);
      if (box_r) {
        out[e + 0] = (uint32_t)(4LL * (lo4 + (long long)box_r * ccol));
        uint32_t opack = 0;
        for (int k = 0; k < kStripMG; ++k) {
          const uint32_t o = R[k] == INT_MIN ? (uint32_t)kStripNO : (uint32_t)(R[k] - lo4);
          if (o > (uint32_t)kStripNO || (o == (uint32_t)kStripNO && R[k] != INT_MIN)) return false;
          opack |= o << (8 * k);
          out[e + 2 + k] = fbits(W[k]);
        }
        out[e + 1] = opack;
      }
    }
  }
  tiles = tiles_r * tiles_c;
  return true;
}

// Strip layout of the whole forward (false: the plan keeps the classic forward kernels).
bool build_strip_forward(ctis_plan_s& P, const std::vector<std::pair<int, int>>& chunks,
                         const std::vector<std::vector<Mode>>& chunk_modes) {
  const char* env = std::getenv("CTIS_FWD_STRIP");
  const int want = env ? std::atoi(env) : -1;  // 0 never, 1 whenever possible, -1 when it pays
  if (want == 0 || !P.tma_f) return false;
  if (P.gamma >= 65536 || P.xi >= 65536) return false;  // flush references are packed as 16-bit (row, column)
  // Mode references with rows rounded down to a multiple of 4 (o = o_ref + dr + gamma*dc holds for any
  // reference; the shifts grow by <= 3 rows): flush boxes then start on 16-byte FPA row boundaries.
  std::vector<std::vector<Mode>> smodes = chunk_modes;  // outlives every StripGroup pointer below
  for (auto& ms : smodes)
    for (Mode& md : ms) md.ref_dr &= ~3;
  std::vector<StripPass> passes;
  size_t nmodes = 0, ngroups = 0;
  for (size_t k = 0; k < chunks.size(); ++k) {
    std::vector<StripGroup> gs = strip_groups(chunks[k].second, smodes[k]);
    nmodes += smodes[k].size();
    ngroups += gs.size();
    const int np = (int)((gs.size() + kStripWarpsMax - 1) / kStripWarpsMax);
    for (int i = 0; i < np; ++i) {
      StripPass ps;
      ps.b0 = chunks[k].first;
      ps.nb = chunks[k].second;
      // balanced passes: groups i, i + np, ... (neighbouring columns in different passes)
      for (size_t g = (size_t)i; g < gs.size(); g += (size_t)np) ps.groups.push_back(gs[g]);
      passes.push_back(std::move(ps));
    }
  }
  if (ngroups == 0) return false;
  if (want < 0) {
    // measured on B200 (tools/gpu_strip.sh): the strip kernel wins where every chunk fits one pass of
    // <= kStripWarpsMax groups and chunks are long (C4: 62 vs 82 us); with several passes per chunk
    // (C3's streak taps: 17 groups) or short chunks (C2: 1-band chunks) the classic kernel is faster
    if ((double)nmodes < 2.0 * (double)ngroups) return false;  // too little strip reuse
    if (passes.size() != chunks.size()) return false;
    for (auto [b0, nb] : chunks)
      if (nb < 12) return false;
  }
  int box_r = 0, box_c = 1;
  for (const StripPass& ps : passes) {
    std::vector<uint32_t> d;
    int t = 0, nr = 0, nc = 0;
    if (!strip_desc(P, ps, 0, d, t, nr, nc)) return false;
    box_r = std::max(box_r, nr);
    box_c = std::max(box_c, nc);
  }
  box_r = std::max(box_r, 8);
  while (box_r % 8 != 4) ++box_r;  // pitch / 4 odd: conflict-free float4 strip loads across columns
  if (box_r > 256 || box_c > 256 || (long long)box_r * box_c > kTmaWinFloats) return false;
  {  // shared memory: barriers + >= 3 window slots + 1 KB alignment slack + staging of the widest pass
    size_t wm = 0;
    for (const StripPass& ps : passes) wm = std::max(wm, ps.groups.size());
    const size_t slot_b = (size_t)((box_r * box_c + 31) / 32 * 32) * sizeof(float);
    if (128 + 3 * slot_b + 2048 + wm * kStripStage * sizeof(float) > 227 * 1024) return false;
  }
  std::vector<std::vector<uint32_t>> descs;
  std::vector<int> tiles, warps;
  for (const StripPass& ps : passes) {
    std::vector<uint32_t> d;
    int t = 0, nr = 0, nc = 0;
    if (!strip_desc(P, ps, box_r, d, t, nr, nc)) return false;
    if (d.empty()) continue;
    if (d.size() + kPageHeader > (size_t)kPageWords) return false;
    descs.push_back(std::move(d));
    tiles.push_back(t);
    warps.push_back((int)ps.groups.size());
  }
  P.fwd.clear();
  pack_pages(P.fwd, true, descs, tiles, warps);
  for (Page& pg : P.fwd) {
    pg.strip = true;
    pg.strip_warps = pg.max_modes;
  }
  P.fbox_r = box_r;
  P.fbox_c = box_c;
  P.fwd_strip = true;
  return true;
}

// Byte offset and size of the ".nv.constant3" section (the c_tab bank) in the embedded cubin.
bool constant_bank_section(const unsigned char* img, size_t len, size_t& off, size_t& size) {
  if (len < 64 || std::memcmp(img, "\x7f" "ELF", 4) != 0 || img[4] != 2) return false;  // ELF64 only
  uint64_t shoff;
  uint16_t shentsize, shnum, shstrndx;
  std::memcpy(&shoff, img + 0x28, 8);
  std::memcpy(&shentsize, img + 0x3a, 2);
  std::memcpy(&shnum, img + 0x3c, 2);
  std::memcpy(&shstrndx, img + 0x3e, 2);
  if (shoff + (uint64_t)shnum * shentsize > len || shstrndx >= shnum) return false;
  auto sec = [&](int i, uint32_t& name, uint32_t& type, uint64_t& o, uint64_t& sz) {
    const unsigned char* h = img + shoff + (uint64_t)i * shentsize;
    std::memcpy(&name, h + 0, 4);
    std::memcpy(&type, h + 4, 4);
    std::memcpy(&o, h + 0x18, 8);
    std::memcpy(&sz, h + 0x20, 8);
  };
  uint32_t n0, t0;
  uint64_t stro, strsz;
  sec(shstrndx, n0, t0, stro, strsz);
  for (int i = 0; i < shnum; ++i) {
    uint32_t nm, ty;
    uint64_t o, sz;
    sec(i, nm, ty, o, sz);
    if (nm >= strsz || stro + nm >= len) continue;
    const char* name = reinterpret_cast<const char*>(img + stro + nm);
    if (ty == 1 /* PROGBITS */ && std::strcmp(name, ".nv.constant3") == 0 && o + sz <= len) {
      off = (size_t)o;
      size = (size_t)sz;
      return true;
    }
  }
  return false;
}

// Load one instance of the table-kernel cubin whose c_tab bank is initialised with this page:
// the words are patched into the image's .nv.constant3 section before cudaLibraryLoadData, so the
// driver itself initialises the bank at module load (lazy or eager).  Writing the bank afterwards
// with cudaMemcpy was not reliably seen by the first launches of a fresh plan (stale constant data
// under lazy module loading: tests/test_gpu_parity.py::test_mlem_random_wrapping flaked after a C4 run).
ctis_status load_page(Page& pg, bool vec) {
  const size_t bytes = (size_t)(ctis_tables_cubin_end - ctis_tables_cubin);
  size_t off = 0, size = 0;
  if (!constant_bank_section(ctis_tables_cubin, bytes, off, size) || size < (size_t)kPageWords * 4)
    return fail(CTIS_ERR_CUDA, "embedded cubin: no .nv.constant3 bank for the tap page");
  if (pg.words.size() > (size_t)kPageWords) return fail(CTIS_ERR_INVALID_ARGUMENT, "tap page overflow");
  std::vector<uint64_t> img((bytes + 7) / 8, 0);
  std::memcpy(img.data(), ctis_tables_cubin, bytes);
  unsigned char* bank = reinterpret_cast<unsigned char*>(img.data()) + off;
  std::memset(bank, 0, (size_t)kPageWords * 4);
  std::memcpy(bank, pg.words.data(), pg.words.size() * 4);
  CTIS_CUDA(cudaLibraryLoadData(&pg.lib, img.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
            "cudaLibraryLoadData (tap page)");
  std::string name;
  if (pg.forward && pg.strip) {
    name = "ctis_fwd_strip_t";
  } else if (pg.forward) {
    name = "ctis_fwd_g" + std::to_string(pg.max_modes / 1000) + "_m" + std::to_string(pg.max_modes % 1000) +
           (vec ? "_t" : "_s");
  } else {
    name = std::string(vec ? (pg.back_tc == 16 ? "ctis_back2_b" : "ctis_back4_b") : "ctis_back_b") +
           std::to_string(pg.max_modes) + (vec ? "_t" : "_s");
  }
  CTIS_CUDA(cudaLibraryGetKernel(&pg.kern, pg.lib, name.c_str()), "cudaLibraryGetKernel");
  int dev = 0;
  CTIS_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  // deep window pipelines need more than the default 48 KB of dynamic shared memory
  const int smem_max = 227 * 1024;  // permission only: launches request what their ring needs
  CTIS_CUDA(cudaKernelSetAttributeForDevice(pg.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max, dev),
            "cudaKernelSetAttributeForDevice");
  return CTIS_OK;
}

// Split w bands into the fewest chunks of <= maxb bands, balanced (sizes differ by at most 1).
std::vector<std::pair<int, int>> balanced_chunks(int w, int maxb) {
  const int nch = (w + maxb - 1) / maxb;
  std::vector<std::pair<int, int>> out;
  int b0 = 0;
  for (int k = 0; k < nch; ++k) {
    const int nb = w / nch + (k < w % nch ? 1 : 0);
    out.emplace_back(b0, nb);
    b0 += nb;
  }
  return out;
}

// Back-kernel band template: minimise (waves over 2 CTAs/SM) x (NB + window cost in band units).
int choose_back_nb(const ctis_plan_s& P) {
  if (const char* e = std::getenv("CTIS_BACK_NB")) {  // experiments: 4, 8, 12 or 16
    const int v = std::atoi(e);
    if (v == 2 || v == 4 || v == 8 || v == 10 || v == 12 || v == 16) return v;
  }
  if (P.throughput) {  // many frames fill the SMs anyway: minimise chunks x (NB + window cost), NB <= 12
    int best = 12;
    long long bestc = LLONG_MAX;
    for (int NB : {12, 10, 8, 4, 2}) {  // 10: w = 50 (C3/C5) splits into 5 full chunks, no padded band slots
      const long long c = (long long)((P.w + NB - 1) / NB) * (NB + 5);
      if (c < bestc) {
        bestc = c;
        best = NB;
      }
    }
    return best;
  }
  const long long tiles = (long long)((P.a + kBackTR - 1) / kBackTR) * ((P.alpha + P.back_tc - 1) / P.back_tc);
  const long long slots = 148LL * 2;
  int best = kBackBandsMax;
  double bestc = 1e300;
  for (int NB : {16, 12, 10, 8, 4, 2}) {
    const long long nch = (P.w + NB - 1) / NB;
    const long long ctas = tiles * nch;
    const double waves = std::ceil((double)ctas / (double)slots);
    const double c = waves * (NB + 5.0);
    if (c < bestc - 1e-9) {
      bestc = c;
      best = NB;
    }
  }
  return best;
}

ctis_status build_tables(ctis_plan_s& P, const std::vector<std::vector<TapXY>>& bands, const std::vector<float>& invh) {
  // TMA needs 16-byte global strides: a % 4 == 0 for f, gamma % 4 == 0 for r.
  P.pair = true;  // FFMA2 on tap pairs (plain FFMA measured no faster on B200)
  // TMA forward: f rows need a 16-byte pitch — a % 4 == 0, or a repacked copy (f_pitch; CTIS_FWD_REPACK=0
  // keeps the element-loader forward for such plans)
  P.f_pitch = (P.a + 3) / 4 * 4;
  {
    const char* e = std::getenv("CTIS_FWD_REPACK");
    P.tma_f = (P.a % 4 == 0) || !(e && std::atoi(e) == 0);
  }
  P.nowrap = true;
  for (const auto& b : bands)
    for (const TapXY& t : b)
      if (t.dr > P.gamma - P.a || t.dc > P.xi - P.alpha) P.nowrap = false;
  P.tma_b = (P.gamma % 4 == 0);
  // ---- forward: chunks of <= kFwdBands bands, modes split into passes of <= 96; one kernel template
  //      (G groups x MAXM modes, MAXM even: modes are paired for FFMA2) and one TMA box per plan
  {
    std::vector<std::vector<Mode>> chunk_modes;
    // TMA plans may use longer chunks with a wider mode span (fewer chunks -> fewer flush atomics):
    // CTIS_FWD_BANDS / CTIS_FWD_SPAN override the defaults (experiments)
    int fbands = kFwdBands, fspan = kModeSpanDefault;
    if (P.tma_f) {
      fbands = kFwdBandsTma;  // measured at C4: 16/12 -> 85.3 us, 25/16 -> 82.2 us (C3: 23.0 -> 19.0 us)
      fspan = kModeSpanTma;
      // small problems: shorter chunks until the persistent grid (2 CTAs per SM) has enough work
      // items (tiles x mode passes x chunks) to keep every SM busy
      size_t tmax = 1;
      for (const auto& b : bands) tmax = std::max(tmax, b.size());
      const long long tiles = (long long)((P.a + 2 * fspan + kFwdTR - 1) / kFwdTR) *
                              ((P.alpha + 2 * fspan + kFwdTC - 1) / kFwdTC);
      const long long passes = ((long long)tmax + 31) / 32;
      while (!P.throughput && fbands > 1 && tiles * passes * ((P.w + fbands - 1) / fbands) < 2LL * P.sms)
        fbands = fbands / 2;
      if (const char* e = std::getenv("CTIS_FWD_BANDS")) fbands = std::max(1, std::atoi(e));
      if (const char* e = std::getenv("CTIS_FWD_SPAN")) fspan = std::max(1, std::min(kModeSpanMax, std::atoi(e)));
    }
    std::vector<std::pair<int, int>> chunks = balanced_chunks(P.w, fbands);
    int nm_max = 1;
    for (auto [b0, nb] : chunks) {
      std::vector<std::vector<TapXY>> cb(bands.begin() + b0, bands.begin() + b0 + nb);
      chunk_modes.push_back(cluster_modes(cb, fspan));
      nm_max = std::max(nm_max, (int)chunk_modes.back().size());
    }
    // <= 64 modes: two 16-warp groups split the modes (MAXM per group, multiple of 4, <= 32, keeps
    // the 1024-thread CTA within 64 registers); otherwise one group with up to 96 modes per pass.
    // <= 64 modes: each pass holds half of them (MAXM even, <= 32) and runs as two independent
    // 512-thread CTAs per SM, one per pass (G = 1, default: a CTA's prologue, first-window latency
    // and flush overlap the other CTA's tap loop; measured 78 vs 95 us at C4), or as one 1024-thread
    // CTA with two mode groups sharing each window (G = 2; CTIS_FWD_GROUPS=2).
    // TMA plans: forward_persistent2 (two u positions per thread, 2 CTAs of 256 threads per SM), passes
    // of <= 32 modes (CTIS_FWD_MAXM overrides the cap; templates: even MAXM <= 32, 36, 40).
    // Element-loader plans: forward_body, 512 threads, up to 96 modes per pass.
    int maxm;
    if (P.tma_f) {
      const char* cap_env = std::getenv("CTIS_FWD_MAXM");
      const int cap = cap_env ? std::max(2, std::min(40, std::atoi(cap_env))) : 32;
      const int npass = (nm_max + cap - 1) / cap;
      int mm = std::max(2, ((nm_max + npass - 1) / npass + 1) / 2 * 2);
      if (mm > 32) mm = mm <= 36 ? 36 : 40;
      P.fwd_g = 2;
      P.fwd_m = mm;
      maxm = mm;
    } else {
      P.fwd_g = 1;
      P.fwd_m = nm_max <= 64 ? std::max(2, ((nm_max + 1) / 2 + 1) / 2 * 2)
                             : std::max(40, std::min(96, (nm_max + 7) / 8 * 8));
      // modes per pass: <= 64 modes run as two passes of MAXM (two independent CTAs per SM)
      maxm = P.fwd_m;
    }
    std::vector<std::vector<const Mode*>> passes;
    std::vector<int> pass_chunk;
    for (size_t k = 0; k < chunk_modes.size(); ++k)
      for (size_t s0 = 0; s0 < chunk_modes[k].size(); s0 += (size_t)maxm) {
        std::vector<const Mode*> pass;
        for (size_t c = s0; c < std::min(chunk_modes[k].size(), s0 + (size_t)maxm); ++c) pass.push_back(&chunk_modes[k][c]);
        passes.push_back(std::move(pass));
        pass_chunk.push_back((int)k);
      }
    int box_r = 0, box_c = 0;
    if (P.tma_f) {
      for (size_t i = 0; i < passes.size(); ++i)
        for (const Span& x : band_spans(chunks[pass_chunk[i]].second, passes[i]))
          if (!x.empty()) {
            box_r = std::max(box_r, kFwdTR + x.rmax - x.rmin + 3);
            box_c = std::max(box_c, kFwdTC + x.cmax - x.cmin);
          }
      box_r = std::max(4, round4(box_r));
      box_c = std::max(1, box_c);
    }
    P.fbox_r = box_r;
    P.fbox_c = box_c;
    std::vector<std::vector<uint32_t>> descs;
    std::vector<int> tiles, modes;
    for (size_t i = 0; i < passes.size(); ++i) {
      const int b0 = chunks[pass_chunk[i]].first, nb = chunks[pass_chunk[i]].second;
      std::vector<uint32_t> d;
      int t = 0;
      if (!forward_desc(P, b0, nb, passes[i], maxm, box_r, box_c, d, t))
        return fail(CTIS_ERR_TAP, "forward window overflow");
      if (d.empty()) continue;
      descs.push_back(std::move(d));
      tiles.push_back(t);
      modes.push_back(1000 * P.fwd_g + P.fwd_m);  // forward pages: "max_modes" encodes the template
    }
    pack_pages(P.fwd, true, descs, tiles, modes);
    build_strip_forward(P, chunks, chunk_modes);  // replaces the pages when the strip layout applies
  }
  // ---- back: NB (kernel template) chosen so that tiles x chunks fills the SMs; a chunk whose
  //      descriptor would not fit one 64 KB page is split further
  {
    P.back_tc = kBackTC;
    bool allow16 = true;
  back_layout:
    P.back_nb = choose_back_nb(P);
    if (allow16 && !P.throughput) {  // small TMA plans: 32 x 16 tiles (two voxels per thread) when 32 x 32 tiles leave CTA slots idle
      const long long t32 = (long long)((P.a + kBackTR - 1) / kBackTR) * ((P.alpha + kBackTC - 1) / kBackTC);
      const char* e = std::getenv("CTIS_BACK_TC");
      // measured: tiny 14.8 -> 13.3 us, C2 unchanged, C3 (208 items) 25.0 -> 25.2 us: only below one item per SM
      const bool want16 = e ? std::atoi(e) == 16 : t32 * ((P.w + P.back_nb - 1) / P.back_nb) < (long long)P.sms;
      if (want16 && P.tma_b) {
        P.back_tc = 16;
        P.back_nb = choose_back_nb(P);
      }
    }
    std::vector<std::pair<int, int>> todo = balanced_chunks(P.w, P.back_nb);
    std::vector<std::vector<Mode>> cms;
    for (auto [b0, nb] : todo) {
      std::vector<std::vector<TapXY>> cb(bands.begin() + b0, bands.begin() + b0 + nb);
      cms.push_back(cluster_modes(cb));
    }
    int box_r = 0, box_c = 0;
    if (P.tma_b) {
      for (const auto& ms : cms)
        for (const Mode& md : ms) {
          const Span sp = mode_span(md);
          box_r = std::max(box_r, kBackTR + sp.rmax - sp.rmin + 3);
          box_c = std::max(box_c, P.back_tc + sp.cmax - sp.cmin);
        }
      box_r = std::max(4, round4(box_r));
      box_c = std::max(1, box_c);
    }
    P.bbox_r = box_r;
    P.bbox_c = box_c;
    // The persistent TMA back kernel needs every window of every tile to be a plain FPA box (no
    // carry / wrap of Eq. 7); otherwise the plan uses the exact element-loader kernels.
    if (P.tma_b) {
      const int tiles_r = (P.a + kBackTR - 1) / kBackTR, tiles_c = (P.alpha + P.back_tc - 1) / P.back_tc;
      for (const auto& ms : cms) {
        for (const Mode& md : ms) {
          const Span sp = mode_span(md);
          const long long B0 = (long long)md.ref_dr + (long long)P.gamma * md.ref_dc + sp.rmin +
                               (long long)P.gamma * sp.cmin;
          const int lead = (int)(((B0 % 4) + 4) % 4);
          long long Bm = (B0 - lead) % P.n;
          if (Bm < 0) Bm += P.n;
          const int br = (int)(Bm % P.gamma), bc = (int)(Bm / P.gamma);
          for (int tc = 0; tc < tiles_c && P.tma_b; ++tc)
            for (int tr = 0; tr < tiles_r && P.tma_b; ++tr) {
              int R0 = tr * kBackTR + br, C0 = tc * P.back_tc + bc;
              if (R0 >= P.gamma) {
                R0 -= P.gamma;
                C0 += 1;
              }
              if (C0 >= P.xi) C0 -= P.xi;
              if (R0 + box_r > P.gamma || C0 + box_c > P.xi) P.tma_b = false;
            }
        }
      }
    }
    if (!P.tma_b && P.back_tc != kBackTC) {  // element-loader kernels use 32 x 32 tiles: lay out again
      P.back_tc = kBackTC;
      allow16 = false;
      goto back_layout;
    }
    std::vector<std::vector<uint32_t>> descs;
    std::vector<int> tiles;
    for (size_t k = 0; k < todo.size(); ++k) {
      const int b0 = todo[k].first, nb = todo[k].second;
      std::vector<uint32_t> d;
      int t = 0;
      if (!back_desc(P, b0, nb, P.back_nb, cms[k], invh, box_r, box_c, d, t))
        return fail(CTIS_ERR_TAP, "back window overflow");
      if ((int)d.size() + kPageHeader > kPageWords) {
        if (nb == 1) return fail(CTIS_ERR_TAP, "band has too many taps for one 64 KB tap page");
        // split the chunk in two and re-cluster both halves (box stays valid: spans only shrink)
        const int h = nb / 2;
        todo.insert(todo.begin() + (long)k + 1, {b0 + h, nb - h});
        todo[k].second = h;
        std::vector<std::vector<TapXY>> c1(bands.begin() + b0, bands.begin() + b0 + h);
        std::vector<std::vector<TapXY>> c2(bands.begin() + b0 + h, bands.begin() + b0 + nb);
        cms[k] = cluster_modes(c1);
        cms.insert(cms.begin() + (long)k + 1, cluster_modes(c2));
        --k;
        continue;
      }
      descs.push_back(std::move(d));
      tiles.push_back(t);
    }
    // Mode split (single-frame layouts with fewer work items than CTA slots, persistent TMA kernels):
    // re-emit every chunk as S descriptors over consecutive subsets of its modes
    P.back_split = 1;
    if (P.tma_b && !P.throughput && !P.shard) {
      long long items = 0;
      for (int t : tiles) items += t;
      // as many subsets as still fit ONE wave of CTA slots (2 per SM): a second wave costs a whole item's
      // latency again (measured: C3 2 subsets = 416 items, back 25 -> 50 us; T1w3 8 subsets, 22 vs 40 us)
      // only for plans that leave most SMs idle (< 1 item per 2 SMs): C2 (2 subsets) and T1w24 measured
      // slower split (18.9 vs 17.4 us per MLEM iteration), T1w3 (30 items, 8 subsets) 36.3 -> 18.1 us
      int S = items * 2 <= P.sms ? (int)std::min<long long>(8, (2LL * P.sms) / std::max<long long>(1, items)) : 1;
      if (const char* e = std::getenv("CTIS_BACK_SPLIT")) S = std::max(1, std::min(8, std::atoi(e)));
      size_t nm_min = SIZE_MAX;
      for (const auto& ms : cms) nm_min = std::min(nm_min, ms.size());
      S = (int)std::min<size_t>((size_t)S, std::max<size_t>(1, nm_min / 4));
      if (S > 1 && descs.size() == todo.size()) {
        std::vector<std::vector<uint32_t>> sd;
        std::vector<int> st;
        bool ok = true;
        for (size_t k = 0; k < todo.size() && ok; ++k) {
          const int b0 = todo[k].first, nb = todo[k].second;
          const size_t nm = cms[k].size();
          for (int j = 0; j < S && ok; ++j) {
            const size_t c0 = nm * j / S, c1 = nm * (j + 1) / S;
            if (c1 <= c0) continue;
            std::vector<Mode> sub(cms[k].begin() + (long)c0, cms[k].begin() + (long)c1);
            std::vector<uint32_t> d;
            int t = 0;
            ok = back_desc(P, b0, nb, P.back_nb, sub, invh, box_r, box_c, d, t);
            sd.push_back(std::move(d));
            st.push_back(t);
          }
        }
        if (ok) {
          descs.swap(sd);
          tiles.swap(st);
          P.back_split = S;
        }
      }
    }
    std::vector<int> nbs(descs.size(), P.back_nb);  // back pages: "max_modes" carries NB
    pack_pages(P.back, false, descs, tiles, nbs);
  }
  for (Page& pg : P.fwd) {
    pg.pair = P.pair;
    ctis_status st = load_page(pg, P.tma_f);
    if (st) return st;
  }
  for (Page& pg : P.back) {
    pg.back_tc = P.back_tc;
    pg.pair = P.pair;
    ctis_status st = load_page(pg, P.tma_b);
    if (st) return st;
  }
  return CTIS_OK;
}

ctis_status build_plan(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi, const int64_t* tap_ptr,
                       const int64_t* tap_offset, const float* tap_weight, int64_t b0, int64_t b1, bool shard,
                       int device, ctis_plan* out, bool throughput = false) {
  if (!out) return fail(CTIS_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!tap_ptr || !tap_offset || !tap_weight) return fail(CTIS_ERR_INVALID_ARGUMENT, "tap array is NULL");
  if (a < 1 || alpha < 1 || w < 1 || gamma < 1 || xi < 1)
    return fail(CTIS_ERR_DIMENSION, "a, alpha, w, gamma, xi must be >= 1");
  if (gamma < a || xi < alpha) return fail(CTIS_ERR_DIMENSION, "field stop must fit the FPA (gamma >= a, xi >= alpha)");
  // every factor below 2^30 before any product is formed (no int64 overflow); then the products
  if (a >= (int64_t(1) << 30) || alpha >= (int64_t(1) << 30) || w >= (int64_t(1) << 30) ||
      gamma >= (int64_t(1) << 30) || xi >= (int64_t(1) << 30))
    return fail(CTIS_ERR_DIMENSION, "n must be < 2^30 and m < 2^31");
  const int64_t n = gamma * xi, ell = a * alpha;
  if (n >= (int64_t(1) << 30) || ell >= (int64_t(1) << 30) || ell * w >= (int64_t(1) << 31))
    return fail(CTIS_ERR_DIMENSION, "n must be < 2^30 and m < 2^31");
  if (b0 < 0 || b1 > w || b0 >= b1) return fail(CTIS_ERR_DIMENSION, "band range must be a non-empty subrange of [0, w)");
  if (tap_ptr[0] != 0) return fail(CTIS_ERR_TAP, "tap_ptr[0] must be 0");
  std::vector<float> hband;
  for (int64_t l = 0; l < w; ++l) {
    if (tap_ptr[l + 1] <= tap_ptr[l])
      return fail(CTIS_ERR_TAP, "band " + std::to_string(l) + " has no taps (or tap_ptr decreases)");
    std::vector<int64_t> offs;
    double hs = 0.0;
    for (int64_t t = tap_ptr[l]; t < tap_ptr[l + 1]; ++t) {
      if (tap_offset[t] < 0 || tap_offset[t] >= n)
        return fail(CTIS_ERR_TAP, "tap offset outside [0, n) in band " + std::to_string(l));
      const float wt = tap_weight[t];
      if (!(wt > 0.f) || !std::isfinite(wt))
        return fail(CTIS_ERR_TAP, "tap weight not finite and > 0 in band " + std::to_string(l));
      offs.push_back(tap_offset[t]);
      hs += wt;
    }
    std::sort(offs.begin(), offs.end());
    if (std::adjacent_find(offs.begin(), offs.end()) != offs.end())
      return fail(CTIS_ERR_TAP, "duplicate tap offset in band " + std::to_string(l));
    if (!((float)hs > 0.f) || !std::isfinite((float)hs)) return fail(CTIS_ERR_ZERO_SENSITIVITY, "h_lambda not > 0");
    hband.push_back((float)hs);
  }
  // exchange range of the latency mode: every pixel a tap of any band can reach, E(j) <= E(l-1)
  int64_t ex_lo = n, ex_hi = -1;
  {
    const int64_t emax = (a - 1) + gamma * (alpha - 1);
    for (int64_t t = 0; t < tap_ptr[w]; ++t) {
      ex_lo = std::min(ex_lo, tap_offset[t]);
      ex_hi = std::max(ex_hi, tap_offset[t] + emax);
    }
    if (ex_hi >= n) {  // some tap wraps past n (Eq. 7): the whole FPA
      ex_lo = 0;
      ex_hi = n - 1;
    }
  }
  // reachable 2-D box (no-wrap taps of this plan's bands only)
  int64_t br0 = gamma, br1 = -1, bc0 = xi, bc1 = -1;
  bool box_ok = gamma % 4 == 0;
  for (int64_t t = tap_ptr[b0]; t < tap_ptr[b1] && box_ok; ++t) {
    const int64_t dr = tap_offset[t] % gamma, dc = tap_offset[t] / gamma;
    if (dr > gamma - a || dc > xi - alpha) box_ok = false;  // carries across columns / wraps (Eq. 7)
    br0 = std::min(br0, dr);
    br1 = std::max(br1, dr + a - 1);
    bc0 = std::min(bc0, dc);
    bc1 = std::max(bc1, dc + alpha - 1);
  }
  int ndev = 0;
  CTIS_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(CTIS_ERR_INVALID_ARGUMENT, "device ordinal out of range");
  cudaDeviceProp prop;
  CTIS_CUDA(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10) return fail(CTIS_ERR_UNSUPPORTED, std::string("device is not sm_100 (found ") + prop.name + ")");

  DeviceGuard dg(device);
  auto* p = new ctis_plan_s();
  p->sms = prop.multiProcessorCount;
  p->device = device;
  p->shard = shard;
  p->band_begin = b0;
  p->band_end = b1;
  p->ex_lo = ex_lo;
  p->ex_hi = ex_hi;
  // (only when the box saves >= 10 % of the FPA: C4's box is the whole FPA and the per-element index
  // arithmetic then costs 0.4 us per iteration; the paper's 89 x 80 field stop reaches ~1/3)
  if (box_ok && br1 >= br0 && !std::getenv("CTIS_NO_RATIO_BOX") &&
      ((br1 + 1 - (br0 & ~int64_t(3)) + 3) / 4 * 4) * (bc1 + 1 - bc0) * 10 < 9 * n) {
    p->rb_r0 = (int)(br0 & ~int64_t(3));
    p->rb_nr4 = (int)((br1 + 1 - p->rb_r0 + 3) / 4);
    p->rb_c0 = (int)bc0;
    p->rb_nc = (int)(bc1 + 1 - bc0);
  }
  p->a = (int)a;
  p->alpha = (int)alpha;
  p->w = (int)(b1 - b0);
  p->gamma = (int)gamma;
  p->xi = (int)xi;
  p->n = (int)n;
  p->ell = (int)ell;
  p->m = (int)(ell * p->w);
  std::vector<std::vector<TapXY>> bands(p->w);
  std::vector<float> invh(p->w), hloc(p->w);
  for (int lam = 0; lam < p->w; ++lam) {
    const int64_t l = b0 + lam;
    double hs = 0.0;
    std::vector<std::pair<int64_t, float>> bt;
    for (int64_t t = tap_ptr[l]; t < tap_ptr[l + 1]; ++t) {
      bt.emplace_back(tap_offset[t], tap_weight[t]);
      hs += tap_weight[t];
    }
    std::sort(bt.begin(), bt.end());
    for (auto& x : bt) bands[lam].push_back(TapXY{(int)(x.first % gamma), (int)(x.first / gamma), x.second});
    p->band_taps.push_back(bt);
    invh[lam] = (float)(1.0 / hs);
    hloc[lam] = hband[l];
    p->total_taps += (int64_t)bt.size();
  }
  p->inv_h = invh;
  if (cudaMalloc(&p->d_invh, sizeof(float) * p->w) != cudaSuccess ||
      cudaMemcpy(p->d_invh, invh.data(), sizeof(float) * p->w, cudaMemcpyHostToDevice) != cudaSuccess) {
    delete p;
    return fail(CTIS_ERR_OUT_OF_MEMORY, "1/h upload");
  }
  p->throughput = throughput;
  ctis_status st = build_tables(*p, bands, invh);
  cudaError_t e = cudaSuccess;
  if (!st) {
    e = cudaMalloc(&p->d_hband, sizeof(float) * p->w);
    if (e == cudaSuccess) e = cudaMemcpy(p->d_hband, hloc.data(), sizeof(float) * p->w, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_flag, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_gbar, 64);
    if (e == cudaSuccess) e = cudaMemset(p->d_gbar, 0, 64);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming);
    if (e != cudaSuccess) st = cuda_fail(e, "plan scratch");
  }
  if (st) {
    std::string msg = g_last_error;
    delete p;
    return fail(st, msg);
  }
  // The tap pages and h were uploaded with cudaMemcpy from pageable memory, which may return before
  // the DMA lands; kernels run on caller / side streams that need not order after the legacy stream.
  // Wait here so that the plan is complete when ctis_plan_create returns.
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "plan upload");
  }
  if (!throughput && !shard && p->tma_f && !std::getenv("CTIS_NO_TPUT")) {
    ctis_plan tp = nullptr;
    ctis_status ts = build_plan(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, b0, b1, shard, device, &tp, true);
    if (ts) {  // e.g. a band too dense for NB = 12 chunks in one page: keep the single-frame layout only
      *out = p;
      g_last_error.clear();
      return CTIS_OK;
    }
    size_t fc = 0, tfc = 0;
    for (const Page& pg : p->fwd) fc += pg.nchunks;
    for (const Page& pg : tp->fwd) tfc += pg.nchunks;
    if (fc == tfc && p->back_nb == tp->back_nb && p->back_tc == tp->back_tc && p->tma_b == tp->tma_b)
      delete tp;  // same layout: nothing to gain
    else
      p->tput = tp;
  }
  *out = p;
  g_last_error.clear();
  return CTIS_OK;
}

// Batched calls switch to the throughput layout once the frames give both projections >= 2 work items
// per CTA slot (2 CTAs per SM) in that layout.
ctis_plan_s* layout_for(ctis_plan_s& P, int64_t frames) {
  if (!P.tput || frames < 2 || P.projector != 0) return &P;
  long long fi = 0, bi = 0;
  for (const Page& pg : P.tput->fwd) fi += pg.total_items;
  for (const Page& pg : P.tput->back) bi += pg.total_items;
  if ((long long)frames * std::min(fi, bi) < 4LL * P.sms) return &P;
  ctis_plan_s* T = P.tput;
  T->validate = P.validate;
  T->use_graph = P.use_graph;
  T->fused_ratio = P.fused_ratio;
  return T;
}

bool aligned16(const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15u) == 0; }

ctis_status check_ptrs(std::initializer_list<const void*> ptrs) {
  for (const void* x : ptrs) {
    if (!x) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL device pointer");
    if (!aligned16(x)) return fail(CTIS_ERR_INVALID_ARGUMENT, "device pointer not 16-byte aligned");
  }
  return CTIS_OK;
}

ctis_status check_frames(int64_t frames) {
  if (frames < 1 || frames > 65535) return fail(CTIS_ERR_INVALID_ARGUMENT, "frames must be in [1, 65535]");
  return CTIS_OK;
}

// ---- launches --------------------------------------------------------------------------------
// Programmatic dependent launches between the MLEM kernels: off by default (CTIS_PDL=1 enables) —
// measured slower on B200 (C4 150.0 -> 155.2 us/iteration, C3 40.8 -> 46.9: tools/mlem_time.py).
bool pdl_enabled() {
  static bool v = [] {
    const char* e = std::getenv("CTIS_PDL");
    return e && std::atoi(e) == 1;
  }();
  return v;
}

int debug_flags() {
  static int v = [] {
    const char* e = std::getenv("CTIS_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// f as {a, alpha, w, frames} (forward) or r as {gamma, xi, frames} (back), fp32, zero OOB fill.
cudaError_t make_tensor_map(CUtensorMap* tm, bool forward, const ctis_plan_s& P, const float* base, int frames) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return cudaErrorNotSupported;
  CUresult r;
  if (forward) {
    const cuuint64_t dims[4] = {(cuuint64_t)P.a, (cuuint64_t)P.alpha, (cuuint64_t)P.w, (cuuint64_t)frames};
    const cuuint64_t pitch = (cuuint64_t)P.f_pitch;  // == a unless f was repacked (d_fpad)
    const cuuint64_t strides[3] = {4ull * pitch, 4ull * pitch * P.alpha, 4ull * pitch * P.alpha * P.w};
    // CTIS_DEBUG & 32 (profiling only, results invalid): half-width boxes, to measure what smaller
    // per-band windows would save in TMA traffic
    const cuuint32_t bc = (debug_flags() & 32) ? (cuuint32_t)std::max(1, P.fbox_c / 2) : (cuuint32_t)P.fbox_c;
    const cuuint32_t box[4] = {(cuuint32_t)P.fbox_r, bc, 1u, 1u};
    const cuuint32_t es[4] = {1u, 1u, 1u, 1u};
    r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {(cuuint64_t)P.gamma, (cuuint64_t)P.xi, (cuuint64_t)frames};
    const cuuint64_t strides[2] = {4ull * P.gamma, 4ull * P.n};
    const cuuint32_t bc = (debug_flags() & 32) ? (cuuint32_t)std::max(1, P.bbox_c / 2) : (cuuint32_t)P.bbox_c;
    const cuuint32_t box[3] = {(cuuint32_t)P.bbox_r, bc, 1u};
    const cuuint32_t es[3] = {1u, 1u, 1u};
    r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// g_hat as {gamma, xi, frames} with 32 x 16 boxes and the 128-byte swizzle: the strip forward's
// accumulator tiles are added into it with cp.reduce.async.bulk.tensor (out-of-range elements dropped).
cudaError_t make_ghat_map(CUtensorMap* tm, const ctis_plan_s& P, float* base, int frames) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[3] = {(cuuint64_t)P.gamma, (cuuint64_t)P.xi, (cuuint64_t)frames};
  const cuuint64_t strides[2] = {4ull * P.gamma, 4ull * P.n};
  const cuuint32_t box[3] = {(cuuint32_t)kFwdTR, (cuuint32_t)kFwdTC, 1u};
  const cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Launch with programmatic stream serialization (PDL): the kernel may start while its predecessor
// drains; it waits for the predecessor's results with griddepcontrol.wait (ctis_tables.cu pdl_enter).
cudaError_t launch_pdl(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t s,
                       bool cooperative = false) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() && !cooperative ? 1 : 0;
  attr[1].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barrier cannot deadlock
#ifdef CTIS_NO_COOP
  attr[1].val.cooperative = 0;  // measurement only: the grid barrier relies on co-residency
#else
  attr[1].val.cooperative = cooperative ? 1 : 0;
#endif
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// Fused extras of a projection launch: forward — ratio in place after a grid barrier (last page);
// back — zero the next iteration's accumulator (first page).
struct Fuse {
  int ratio_mode = 0;
  const float* meas = nullptr;
  long long ratio_count = 0;
  float* zero_buf = nullptr;
  long long zero_count = 0;
};


// Repack buffer for plans with f_pitch != a: allocated outside stream capture (entry points call this
// before capturing; inside a capture an undersized buffer is an error, never an allocation).
cudaError_t ensure_fpad(ctis_plan_s& P, int frames, cudaStream_t s) {
  if (P.f_pitch == P.a) return cudaSuccess;
  const size_t need = (size_t)P.f_pitch * P.alpha * P.w * (size_t)frames;
  if (need <= P.fpad_cap) return cudaSuccess;
  if (s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(s, &cs);
    if (e != cudaSuccess) return e;
    if (cs != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;
  }
  if (P.d_fpad) {
    cudaError_t e = cudaDeviceSynchronize();  // the old buffer may still be read by queued launches
    if (e != cudaSuccess) return e;
    cudaFree(P.d_fpad);
    P.d_fpad = nullptr;
    P.fpad_cap = 0;
  }
  cudaError_t e = cudaMalloc(&P.d_fpad, need * sizeof(float));
  if (e == cudaSuccess) P.fpad_cap = need;
  return e;
}

// Partial-z buffer of mode-split plans: allocated zeroed outside stream capture; the update pass keeps it
// zero between uses.
cudaError_t ensure_z(ctis_plan_s& P, int frames, cudaStream_t s) {
  if (P.back_split <= 1) return cudaSuccess;
  const size_t need = (size_t)P.m * (size_t)frames;
  if (need <= P.z_cap) return cudaSuccess;
  if (s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(s, &cs);
    if (e != cudaSuccess) return e;
    if (cs != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  if (P.d_z) cudaFree(P.d_z);
  P.d_z = nullptr;
  P.z_cap = 0;
  e = cudaMalloc(&P.d_z, need * sizeof(float));
  if (e == cudaSuccess) e = cudaMemset(P.d_z, 0, need * sizeof(float));
  if (e == cudaSuccess) P.z_cap = need;
  return e;
}

cudaError_t launch_pages(ctis_plan_s& P, const std::vector<Page>& pages, const float* src, float* dst,
                         long long src_frame, long long dst_frame, int frames, int mode, cudaStream_t s,
                         int64_t* count, const Fuse* fuse = nullptr) {
  if (pages.empty()) return cudaSuccess;
  const bool fwd = pages[0].forward;
  const bool tma = fwd ? P.tma_f : P.tma_b;
  const long long span = (long long)kModeSpanMax * (P.gamma + 1) + 1;  // max -E(u) over the u-space
  const long long kb = (span + P.n - 1) / P.n;
  const unsigned bias = (unsigned)(kb * P.n);
  // E(u) <= (a + kModeSpanMax) + gamma*(alpha + kModeSpanMax) < 2n (field stop fits the FPA), o_ref < n
  const long long emax = (long long)(P.a + kModeSpanMax) + (long long)P.gamma * (P.alpha + kModeSpanMax);
  const int nsub = (int)((bias + emax + P.n - 1) / P.n);
  const int box_r = fwd ? P.fbox_r : P.bbox_r, box_c = fwd ? P.fbox_c : P.bbox_c;
  const int cap = fwd ? kFwdWinFloats : kBackWinFloats;
  int slot = tma ? (box_r * box_c + 31) / 32 * 32 : cap;
  TabArgs A{src, dst, src_frame, dst_frame, P.a, P.alpha, P.gamma, P.xi, P.n, P.ell, mode, bias, nsub,
            slot, box_r, box_c, (unsigned)(4 * box_r * ((debug_flags() & 32) ? std::max(1, box_c / 2) : box_c)),
            debug_flags(), frames, P.nowrap ? 1 : 0,
            0, nullptr, 0, P.d_gbar, nullptr, 0};
  alignas(64) CUtensorMap tm, tg;
  std::memset(&tm, 0, sizeof(tm));
  std::memset(&tg, 0, sizeof(tg));
  if (tma && fwd && P.f_pitch != P.a) {  // repack f to the 16-byte row pitch of the TMA view
    cudaError_t e = ensure_fpad(P, frames, s);
    if (e != cudaSuccess) return e;
    e = launch_repack_rows(src, P.d_fpad, P.a, P.f_pitch, (long long)P.alpha * P.w * frames, s);
    if (e != cudaSuccess) return e;
    if (count) ++*count;
    src = P.d_fpad;
  }
  if (tma) {
    cudaError_t e = make_tensor_map(&tm, fwd, P, src, frames);
    if (e != cudaSuccess) return e;
  }
  A.tma_flush = 0;
  if (fwd && P.fwd_strip && P.nowrap && P.gamma % 4 == 0) {  // strip forward: g_hat as a TMA reduce target
    cudaError_t e = make_ghat_map(&tg, P, dst, frames);
    if (e != cudaSuccess) return e;
    A.tma_flush = 1;
  }
  const int threads = fwd ? (P.fwd_g == 2 ? kFwd2Threads : kFwdThreads) : (tma ? kBack4Threads : kBackThreads);
  const int stages = fwd ? kFwdStages : kBackStages;
  // + full mbarriers (8 B per stage) and 8 B per stage + 64 B for release counters / producer state
  const size_t smem = (size_t)stages * slot * sizeof(float) + 16 * stages + 64;
  A.frames = frames;
  for (size_t ip = 0; ip < pages.size(); ++ip) {
    const Page& pg = pages[ip];
    // TMA kernels are persistent (2 CTAs per SM walk the page's items); element-loader kernels are
    // one CTA per (tile, chunk, frame)
    const long long items = (long long)pg.total_items * frames;
    int per_sm = 2;  // resident CTAs per SM (persistent TMA kernels)
    if (!fwd && tma) {  // experiment switch: more resident back CTAs (kernels built with CTIS_BACK2_MINB)
      static const int env_per_sm = std::getenv("CTIS_BACK_PER_SM") ? std::atoi(std::getenv("CTIS_BACK_PER_SM")) : 0;
      if (env_per_sm > 0) per_sm = env_per_sm;
    }
    dim3 grid = tma ? dim3((unsigned)std::min<long long>(items, (long long)per_sm * P.sms), 1, 1)
                    : dim3(pg.max_tiles, pg.nchunks, frames);
    bool coop = false;
    A.ratio_mode = 0;
    A.zero_count = 0;
    if (fuse && tma) {
      if (fwd && ip + 1 == pages.size() && fuse->ratio_mode) {
        A.ratio_mode = fuse->ratio_mode;
        A.meas = fuse->meas;
        A.ratio_count = fuse->ratio_count;
        coop = true;
#ifdef CTIS_ZERO_IN_FWD
        A.zero_buf = fuse->zero_buf;
        A.zero_count = fuse->zero_count;
#endif
      }
      if (!fwd && ip == 0 && fuse->zero_count) {
        A.zero_buf = fuse->zero_buf;
        A.zero_count = fuse->zero_count;
      }
    }
    int nthreads = threads;
    size_t nsmem = smem;
    if (pg.strip) {  // warp-specialised strip forward: one CTA per SM, consumer warps + a producer warp
      nthreads = 32 * (pg.strip_warps + 1);
      // [ring][staging, 1024-byte aligned][mbarriers]; + 1 KB alignment slack of the dynamic base
      const size_t stage_b = (size_t)pg.strip_warps * kStripStage * sizeof(float);
      const size_t avail = 227 * 1024 - stage_b - 2048 - 128;
      A.stages = (int)std::min<size_t>(kStripStagesMax, avail / ((size_t)slot * sizeof(float)));
      if (const char* e = std::getenv("CTIS_STRIP_STAGES")) A.stages = std::max(2, std::min(A.stages, std::atoi(e)));
      nsmem = ((size_t)128 + (size_t)A.stages * slot * sizeof(float) + 1023) / 1024 * 1024 + 1024 + stage_b;
      grid = dim3((unsigned)std::min<long long>(items, (long long)P.sms), 1, 1);
    }
    void* args[] = {&A, &tm, &tg};
    cudaError_t e = launch_pdl((const void*)pg.kern, grid, dim3(nthreads), args, nsmem, s, coop);
    if (e != cudaSuccess) return e;
    if (count) ++*count;
  }
  return cudaSuccess;
}

// g_hat (accumulated with red.add: must be zero on entry) += H f
cudaError_t enqueue_forward(ctis_plan_s& P, const float* f, float* ghat, int frames, cudaStream_t s, int64_t* cnt,
                            const Fuse* fuse = nullptr) {
  if (P.projector == 1) {  // the paper's Fourier route (comparator arm)
    for (int z = 0; z < frames; ++z) {
      cudaError_t e = fft_forward_accumulate(P.fft, f + (size_t)z * P.m, ghat + (size_t)z * P.n, s, cnt);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  return launch_pages(P, P.fwd, f, ghat, P.m, P.n, frames, 0, s, cnt, fuse);
}

cudaError_t enqueue_back(ctis_plan_s& P, const float* r, float* fz, int frames, int mode, cudaStream_t s,
                         int64_t* cnt, const Fuse* fuse = nullptr) {
  if (P.projector == 1) {
    for (int z = 0; z < frames; ++z) {
      cudaError_t e = fft_back(P.fft, r + (size_t)z * P.n, fz + (size_t)z * P.m, mode, s, cnt);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (P.back_split > 1) {  // mode split: partial z of every mode subset accumulated with red.add
    const size_t count = (size_t)P.m * frames;
    if (mode == 0) {  // z = H^T r straight into the caller's buffer
      cudaError_t e = cudaMemsetAsync(fz, 0, sizeof(float) * count, s);
      if (e != cudaSuccess) return e;
      return launch_pages(P, P.back, r, fz, P.n, P.m, frames, 3, s, cnt, fuse);
    }
    cudaError_t e = ensure_z(P, frames, s);
    if (e != cudaSuccess) return e;
    e = launch_pages(P, P.back, r, P.d_z, P.n, P.m, frames, 3, s, cnt, fuse);
    if (e != cudaSuccess) return e;
    e = launch_split_update(fz, P.d_z, P.d_invh, P.ell, P.w, (long long)count, mode, s);
    if (cnt) ++*cnt;
    return e;
  }
  return launch_pages(P, P.back, r, fz, P.n, P.m, frames, mode, s, cnt, fuse);
}

ctis_status validate_data(ctis_plan_s& P, const float* g, const float* f, int64_t frames, cudaStream_t s) {
  CTIS_CUDA(cudaMemsetAsync(P.d_flag, 0, sizeof(int), s), "validate memset");
  CTIS_CUDA(launch_validate(g, (long long)P.n * frames, P.d_flag, s), "validate g");
  CTIS_CUDA(launch_validate(f, (long long)P.m * frames, P.d_flag, s), "validate f0");
  int flag = 0;
  CTIS_CUDA(cudaMemcpyAsync(&flag, P.d_flag, sizeof(int), cudaMemcpyDeviceToHost, s), "validate copy");
  CTIS_CUDA(cudaStreamSynchronize(s), "validate sync");
  if (flag) return fail(CTIS_ERR_DATA, "g or f0 contains a negative, NaN or Inf value");
  return CTIS_OK;
}

// One MLEM reconstruction: ws = [A: g_hat accumulator, frames*n][B: r, frames*n].
cudaError_t enqueue_mlem(ctis_plan_s& P, const float* g, float* f, float* ws, int frames, int iters, cudaStream_t s,
                         int64_t* cnt, int solver = 0) {
  float* A = ws;
  float* B = ws + (((size_t)P.n * frames + 3) & ~(size_t)3);  // 16-byte aligned second half
  const long long count = (long long)P.n * frames;
  if (P.fused_ratio && P.projector == 0 && P.tma_f && !P.fwd.empty()) {
    // two kernels per iteration: forward (+ ratio in place after its grid barrier) into the current
    // half, back (reading r there) zeroing the other half for the next iteration's forward
    cudaError_t e = cudaMemsetAsync(A, 0, sizeof(float) * (size_t)count, s);
    for (int k = 0; k < iters && e == cudaSuccess; ++k) {
      float* cur = (k & 1) ? B : A;
      float* nxt = (k & 1) ? A : B;
      Fuse ff;
      ff.ratio_mode = solver == 1 ? 2 : 1;
      ff.meas = g;
      ff.ratio_count = count;
      const bool last = k + 1 == iters;
#ifdef CTIS_ZERO_IN_FWD
      if (!last) {  // nxt was r of the previous iteration's back kernel, which has completed
        ff.zero_buf = nxt;
        ff.zero_count = count;
      }
#endif
      e = enqueue_forward(P, f, cur, frames, s, cnt, &ff);
      if (e != cudaSuccess) break;
      Fuse fb;
#ifdef CTIS_ZERO_IN_FWD
      e = enqueue_back(P, cur, f, frames, solver == 1 ? 2 : 1, s, cnt, &fb);
      continue;
#endif
      if (!last && P.tma_b) {
        fb.zero_buf = nxt;
        fb.zero_count = count;
      } else if (!last) {
        e = cudaMemsetAsync(nxt, 0, sizeof(float) * (size_t)count, s);
        if (e != cudaSuccess) break;
      }
      e = enqueue_back(P, cur, f, frames, solver == 1 ? 2 : 1, s, cnt, &fb);
    }
    return e;
  }
  static const bool inplace_env = [] {
    const char* v = std::getenv("CTIS_INPLACE_RATIO");
    return !(v && std::atoi(v) == 0);
  }();
  // in-place ratio: r overwrites g_hat (one buffer, no reset stream in the ratio pass); the accumulator
  // is cleared by a memset node after the back projection has read r.  Measured (B200, C4): 131.6 ->
  // 129.0 us per iteration (CTIS_INPLACE_RATIO=0 restores ratio-into-B + reset); the reachable-box ratio
  // (plans with rb_nr4 > 0) and SMART keep the two-buffer form
  const bool inplace = inplace_env && solver == 0 && !(P.rb_nr4 > 0 && P.projector == 0);
  cudaError_t e = cudaMemsetAsync(A, 0, sizeof(float) * (size_t)count, s);
  for (int k = 0; k < iters && e == cudaSuccess; ++k) {
    if (inplace && k > 0) e = cudaMemsetAsync(A, 0, sizeof(float) * (size_t)count, s);
    if (e == cudaSuccess) e = enqueue_forward(P, f, A, frames, s, cnt);
    if (e == cudaSuccess) {
      if (solver == 1)
        e = launch_log_ratio(g, A, B, count, s, pdl_enabled());
      else if (P.rb_nr4 > 0 && P.projector == 0)  // only the reachable FPA box (ctis_plan_s::rb_*)
        e = launch_ratio_box(g, A, B, P.n, P.gamma, P.rb_r0, P.rb_nr4, P.rb_c0, P.rb_nc, frames, s, pdl_enabled());
      else
        e = launch_ratio(g, A, inplace ? A : B, count, /*zero_ghat=*/!inplace, s, pdl_enabled());
      ++*cnt;
    }
    if (e == cudaSuccess) e = enqueue_back(P, inplace ? A : B, f, frames, solver == 1 ? 2 : 1, s, cnt);
  }
  return e;
}

ctis_status run_mlem(ctis_plan_s& P, const float* g, float* f, int64_t frames, int iters, void* ws, cudaStream_t s,
                     int solver = 0) {
  if (ctis_plan_s* T = layout_for(P, frames); T != &P) {
    ctis_status st = run_mlem(*T, g, f, frames, iters, ws, s, solver);
    P.last_launches = T->last_launches;
    return st;
  }
  if (P.shard)
    return fail(CTIS_ERR_INVALID_ARGUMENT,
                "mlem on a shard plan needs the collective: use ctis_forward + all-reduce + ctis_back_update_from_ghat");
  if (iters < 0) return fail(CTIS_ERR_INVALID_ARGUMENT, "iters < 0");
  ctis_status st = check_frames(frames);
  if (st) return st;
  if ((st = check_ptrs({g, f, ws}))) return st;
  DeviceGuard dg(P.device);
  CTIS_CUDA(ensure_fpad(P, (int)frames, nullptr), "f repack buffer");  // before any stream capture
  CTIS_CUDA(ensure_z(P, (int)frames, nullptr), "partial z buffer");
  P.last_launches = 0;
  if (P.validate) {
    if ((st = validate_data(P, g, f, frames, s))) return st;
    P.last_launches += 2;
  }
  if (iters == 0) return CTIS_OK;
  float* w = static_cast<float*>(ws);
  int64_t cnt = 0;
  if (!P.use_graph) {
    CTIS_CUDA(enqueue_mlem(P, g, f, w, (int)frames, iters, s, &cnt, solver), "mlem launch");
    P.last_launches += cnt;
    return CTIS_OK;
  }
  GraphKey key{g, f, ws, frames, iters, solver};
  auto it = P.graphs.find(key);
  if (it == P.graphs.end()) {
    if (P.graphs.size() >= 16) {
      for (auto& kv : P.graphs) cudaGraphExecDestroy(kv.second);
      P.graphs.clear();
    }
    cudaGraph_t graph = nullptr;
    CTIS_CUDA(cudaStreamBeginCapture(P.side, cudaStreamCaptureModeThreadLocal), "begin capture");
    cudaError_t e = enqueue_mlem(P, g, f, w, (int)frames, iters, P.side, &cnt, solver);
    cudaError_t e2 = cudaStreamEndCapture(P.side, &graph);
    if (e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return cuda_fail(e, "capture launch");
    }
    if (e2 != cudaSuccess) return cuda_fail(e2, "end capture");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
    e = cudaGraphUpload(exec, P.side);  // device-side setup now, not inside the first timed launch
    if (e != cudaSuccess) return cuda_fail(e, "graph upload");
    it = P.graphs.emplace(key, exec).first;
    P.graph_launches[key] = cnt;
  } else {
    cnt = P.graph_launches[key];
  }
  CTIS_CUDA(cudaEventRecord(P.ev_in, s), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(P.side, P.ev_in, 0), "stream wait");
  CTIS_CUDA(cudaGraphLaunch(it->second, P.side), "graph launch");
  CTIS_CUDA(cudaEventRecord(P.ev_out, P.side), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(s, P.ev_out, 0), "stream wait");
  P.last_launches += cnt;
  return CTIS_OK;
}

// Monitored MLEM (ctis_mlem_monitored): [memset g_hat, ll, counter] -> WHILE { forward; ratio + L;
// back + update; stop rule } as one instantiated graph; the WHILE body runs until the device-side
// check clears the condition.
ctis_status run_mlem_monitored(ctis_plan_s& P, const float* g, float* f, int max_iters, double rel_tol, void* ws,
                               double* ll, int* cnt, cudaStream_t s) {
  if (P.shard)
    return fail(CTIS_ERR_INVALID_ARGUMENT, "mlem on a shard plan needs the collective (see ctis_back_update_from_ghat)");
  if (max_iters < 0) return fail(CTIS_ERR_INVALID_ARGUMENT, "max_iters < 0");
  ctis_status st = check_ptrs({g, f, ws});
  if (st) return st;
  if (!ll || !cnt || (reinterpret_cast<uintptr_t>(ll) & 7u) || (reinterpret_cast<uintptr_t>(cnt) & 3u))
    return fail(CTIS_ERR_INVALID_ARGUMENT, "ll (8-byte aligned) and iters_done (4-byte aligned) must be device pointers");
  DeviceGuard dg(P.device);
  CTIS_CUDA(ensure_fpad(P, (int)1, nullptr), "f repack buffer");  // before any stream capture
  CTIS_CUDA(ensure_z(P, 1, nullptr), "partial z buffer");
  P.last_launches = 0;
  if (P.validate) {
    if ((st = validate_data(P, g, f, 1, s))) return st;
    P.last_launches += 2;
  }
  if (max_iters == 0) {
    CTIS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), s), "iters_done");
    return CTIS_OK;
  }
  float* A = static_cast<float*>(ws);
  float* B = A + (((size_t)P.n + 3) & ~(size_t)3);
  MonKey key{g, f, ws, ll, cnt, max_iters, rel_tol};
  auto it = P.mon_graphs.find(key);
  int64_t body_launches = 0;
  if (it == P.mon_graphs.end()) {
    if (P.mon_graphs.size() >= 16) {
      for (auto& kv : P.mon_graphs) cudaGraphExecDestroy(kv.second);
      P.mon_graphs.clear();
    }
    cudaGraph_t graph = nullptr;
    CTIS_CUDA(cudaGraphCreate(&graph, 0), "graph create");
    auto bail = [&](cudaError_t e, const char* where) {
      cudaGraphDestroy(graph);
      return e == cudaErrorNotSupported || e == cudaErrorInvalidValue
                 ? fail(CTIS_ERR_UNSUPPORTED, std::string(where) + ": " + cudaGetErrorString(e))
                 : cuda_fail(e, where);
    };
    cudaGraphNode_t prev = nullptr, node = nullptr;
    auto memset_node = [&](void* ptr, size_t words) -> cudaError_t {
      cudaMemsetParams mp{};
      mp.dst = ptr;
      mp.value = 0;
      mp.elementSize = 4;
      mp.width = words;
      mp.height = 1;
      mp.pitch = 0;
      cudaError_t e = cudaGraphAddMemsetNode(&node, graph, prev ? &prev : nullptr, prev ? 1 : 0, &mp);
      prev = node;
      return e;
    };
    cudaError_t e = memset_node(A, (size_t)P.n);
    if (e == cudaSuccess) e = memset_node(ll, 2 * (size_t)max_iters);
    if (e == cudaSuccess) e = memset_node(cnt, 1);
    if (e != cudaSuccess) return bail(e, "memset nodes");
    cudaGraphConditionalHandle handle;
    e = cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault);
    if (e != cudaSuccess) return bail(e, "cudaGraphConditionalHandleCreate");
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&node, graph, &prev, 1, &cp);
    if (e != cudaSuccess) return bail(e, "conditional WHILE node");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(P.side, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return bail(e, "capture to WHILE body");
    cudaError_t e1 = enqueue_forward(P, f, A, 1, P.side, &body_launches);
    if (e1 == cudaSuccess) {
      e1 = launch_ratio_ll(g, A, B, P.n, ll, cnt, P.side, pdl_enabled());
      ++body_launches;
    }
    if (e1 == cudaSuccess) e1 = enqueue_back(P, B, f, 1, 1, P.side, &body_launches);
    if (e1 == cudaSuccess) {
      e1 = launch_mlem_check(ll, cnt, max_iters, rel_tol, (unsigned long long)handle, P.side);
      ++body_launches;
    }
    cudaGraph_t captured = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(P.side, &captured);
    if (e1 != cudaSuccess) return bail(e1, "WHILE body launches");
    if (e2 != cudaSuccess) return bail(e2, "end capture (WHILE body)");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "graph instantiate (monitored MLEM)");
    it = P.mon_graphs.emplace(key, exec).first;
  } else {
    body_launches = (int64_t)P.fwd.size() + (int64_t)P.back.size() + 2;
  }
  CTIS_CUDA(cudaEventRecord(P.ev_in, s), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(P.side, P.ev_in, 0), "stream wait");
  CTIS_CUDA(cudaGraphLaunch(it->second, P.side), "graph launch");
  CTIS_CUDA(cudaEventRecord(P.ev_out, P.side), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(s, P.ev_out, 0), "stream wait");
  P.last_launches += body_launches;  // per iteration of the device-side loop
  return CTIS_OK;
}

// Latency-mode exchange layout (include/ctis.h): base B (16-byte aligned) and per-rank slice S (floats,
// multiple of 4) covering the plan's exchange range [ex_lo, ex_hi]; X holds >= max(n, B + P*S) floats.
struct Exchange {
  int64_t base, slice, floats;
};
Exchange exchange_layout(const ctis_plan_s& P, const ctis_comm_s& C) {
  Exchange e;
  e.base = P.ex_lo & ~int64_t(3);
  const int64_t len = P.ex_hi + 1 - e.base;
  e.slice = ((len + C.nranks - 1) / C.nranks + 3) & ~int64_t(3);
  e.floats = (std::max<int64_t>(P.n, e.base + e.slice * C.nranks) + 3) & ~int64_t(3);
  return e;
}

// One band-sharded MLEM reconstruction on stream s (kernels + NCCL calls; capturable).
ctis_status enqueue_band_sharded(ctis_plan_s& P, ctis_comm_s& C, const float* g, float* f, float* X, int iters,
                                 cudaStream_t s, int64_t* cnt) {
  const Exchange ex = exchange_layout(P, C);
  float* slice = X + ex.base + (int64_t)C.rank * ex.slice;
  const int64_t s0 = ex.base + (int64_t)C.rank * ex.slice;
  const int64_t ratio_count = s0 >= P.n ? 0 : std::min<int64_t>(ex.slice, P.n - s0);
  std::string err;
  CTIS_CUDA(cudaMemsetAsync(X, 0, sizeof(float) * (size_t)ex.floats, s), "exchange buffer memset");
  for (int k = 0; k < iters; ++k) {
    if (k > 0) CTIS_CUDA(cudaMemsetAsync(X + ex.base, 0, sizeof(float) * (size_t)(ex.slice * C.nranks), s), "memset");
    CTIS_CUDA(enqueue_forward(P, f, X, 1, s, cnt), "partial forward");
    if (P.exchange == 1) {  // f-1: reduce my slice over all ranks, ratio, store r to every rank: one kernel
      CTIS_CUDA(launch_exchange_ratio(C.nvls, ex.base, ex.slice, g, P.n, s), "fused exchange + ratio");
      ++*cnt;
      CTIS_CUDA(enqueue_back(P, X, f, 1, 1, s, cnt), "back update");
      continue;
    }
    if (!nccl_reduce_scatter_f32(X + ex.base, slice, (size_t)ex.slice, C.nccl, s, &err)) return fail(CTIS_ERR_CUDA, err);
    if (ratio_count > 0) {
      CTIS_CUDA(launch_ratio(g + s0, slice, slice, ratio_count, false, s), "slice ratio");
      ++*cnt;
    }
    if (!nccl_all_gather_f32(slice, X + ex.base, (size_t)ex.slice, C.nccl, s, &err)) return fail(CTIS_ERR_CUDA, err);
    CTIS_CUDA(enqueue_back(P, X, f, 1, 1, s, cnt), "back update");
  }
  return CTIS_OK;
}

ctis_status run_band_sharded(ctis_plan_s& P, ctis_comm_s& C, const float* g, float* f, int iters, void* ws,
                             cudaStream_t s) {
  if (iters < 0) return fail(CTIS_ERR_INVALID_ARGUMENT, "iters < 0");
  if (C.device != P.device) return fail(CTIS_ERR_INVALID_ARGUMENT, "communicator and plan are on different devices");
  ctis_status st = check_ptrs({g, f, ws});
  if (st) return st;
  DeviceGuard dg(P.device);
  CTIS_CUDA(ensure_fpad(P, (int)1, nullptr), "f repack buffer");  // before any stream capture
  CTIS_CUDA(ensure_z(P, 1, nullptr), "partial z buffer");
  P.last_launches = 0;
  if (iters == 0) return CTIS_OK;
  float* X = static_cast<float*>(ws);
  if (P.exchange == 1) {  // the exchange buffer is the communicator's symmetric window (collective setup)
    const size_t need = sizeof(float) * (size_t)exchange_layout(P, C).floats;
    if (C.nvls.bytes < need) {
      nvls_teardown(C.nccl, &C.nvls);
      std::string err;
      if (!nvls_setup(C.nccl, need, C.device, &C.nvls, &err)) return fail(CTIS_ERR_UNSUPPORTED, err);
      for (auto& kv : P.shard_graphs) cudaGraphExecDestroy(kv.second);
      P.shard_graphs.clear();
    }
    X = static_cast<float*>(C.nvls.buf);
  }
  int64_t cnt = 0;
  if (!P.use_graph) return enqueue_band_sharded(P, C, g, f, X, iters, s, &P.last_launches);
  GraphKey key{g, f, X, (int64_t)reinterpret_cast<intptr_t>(&C), iters, 2 + P.exchange};
  auto it = P.shard_graphs.find(key);
  if (it == P.shard_graphs.end()) {
    if (P.shard_graphs.size() >= 8) {
      for (auto& kv : P.shard_graphs) cudaGraphExecDestroy(kv.second);
      P.shard_graphs.clear();
    }
    cudaGraph_t graph = nullptr;
    CTIS_CUDA(cudaStreamBeginCapture(P.side, cudaStreamCaptureModeThreadLocal), "begin capture");
    ctis_status est = enqueue_band_sharded(P, C, g, f, X, iters, P.side, &cnt);
    cudaError_t e2 = cudaStreamEndCapture(P.side, &graph);
    if (est) {
      if (graph) cudaGraphDestroy(graph);
      return est;
    }
    if (e2 != cudaSuccess) return cuda_fail(e2, "end capture (band-sharded)");
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "graph instantiate (band-sharded)");
    it = P.shard_graphs.emplace(key, exec).first;
  } else {
    cnt = (int64_t)iters * ((int64_t)P.fwd.size() + (int64_t)P.back.size() + 1);
  }
  CTIS_CUDA(cudaEventRecord(P.ev_in, s), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(P.side, P.ev_in, 0), "stream wait");
  CTIS_CUDA(cudaGraphLaunch(it->second, P.side), "graph launch");
  CTIS_CUDA(cudaEventRecord(P.ev_out, P.side), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(s, P.ev_out, 0), "stream wait");
  P.last_launches = cnt;
  return CTIS_OK;
}

}  // namespace

extern "C" {

ctis_status ctis_comm_unique_id(uint8_t id[128]) {
  if (!id) return fail(CTIS_ERR_INVALID_ARGUMENT, "id is NULL");
  std::string err;
  if (!nccl_available(&err)) return fail(CTIS_ERR_UNSUPPORTED, err);
  if (!nccl_unique_id(id, &err)) return fail(CTIS_ERR_CUDA, err);
  return CTIS_OK;
}

ctis_status ctis_comm_create(int nranks, int rank, const uint8_t id[128], int device, ctis_comm* out) {
  if (!out || !id) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CTIS_ERR_INVALID_ARGUMENT, "rank / nranks out of range");
  std::string err;
  if (!nccl_available(&err)) return fail(CTIS_ERR_UNSUPPORTED, err);
  int ndev = 0;
  CTIS_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(CTIS_ERR_INVALID_ARGUMENT, "device ordinal out of range");
  DeviceGuard dg(device);
  CTIS_CUDA(cudaSetDevice(device), "cudaSetDevice");
  auto* c = new ctis_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (!nccl_comm_init(&c->nccl, nranks, rank, id, &err)) {
    delete c;
    return fail(CTIS_ERR_CUDA, err);
  }
  *out = c;
  return CTIS_OK;
}

void ctis_comm_destroy(ctis_comm comm) { delete comm; }

size_t ctis_band_sharded_workspace_bytes(ctis_plan p, ctis_comm c) {
  if (!p || !c) return 0;
  return sizeof(float) * (size_t)exchange_layout(*p, *c).floats;
}

ctis_status ctis_mlem_band_sharded(ctis_plan p, ctis_comm c, const float* g, float* f_local, int iters, void* ws,
                                   ctis_stream stream) {
  if (!p || !c) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan or communicator");
  std::lock_guard<std::mutex> lk(p->mu);
  return run_band_sharded(*p, *c, g, f_local, iters, ws, (cudaStream_t)stream);
}

ctis_status ctis_plan_create(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi, const int64_t* tap_ptr,
                             const int64_t* tap_offset, const float* tap_weight, int device, ctis_plan* out) {
  return build_plan(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, 0, w, false, device, out);
}

ctis_status ctis_plan_create_shard(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                                   const int64_t* tap_ptr, const int64_t* tap_offset, const float* tap_weight,
                                   int64_t band_begin, int64_t band_end, int device, ctis_plan* out) {
  return build_plan(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, band_begin, band_end, true, device, out);
}

void ctis_plan_destroy(ctis_plan plan) { delete plan; }

ctis_status ctis_plan_dims(ctis_plan p, int64_t out[10]) {
  if (!p || !out) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL argument");
  const int64_t v[10] = {p->a, p->alpha, p->w, p->gamma, p->xi, p->n, p->m, p->band_begin, p->band_end, p->total_taps};
  std::memcpy(out, v, sizeof(v));
  return CTIS_OK;
}

ctis_status ctis_plan_info(ctis_plan p, int64_t out[10]) {
  if (!p || !out) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL argument");
  int64_t fch = 0, bch = 0, fitems = 0;
  for (const Page& pg : p->fwd) {
    fch += pg.nchunks;
    fitems += pg.total_items;
  }
  for (const Page& pg : p->back) bch += pg.nchunks;
  int64_t fwd_kind = p->fwd_m;  // classic forward: modes per group; strip forward: -(consumer warps)
  if (p->fwd_strip) {
    fwd_kind = 0;
    for (const Page& pg : p->fwd) fwd_kind = std::min<int64_t>(fwd_kind, -pg.strip_warps);
  }
  const int64_t v[10] = {(int64_t)p->fwd.size(), (int64_t)p->back.size(), fch, bch, p->tma_f ? 1 : 0,
                         p->tma_b ? 1 : 0, p->back_nb, p->back_tc, fwd_kind, fitems};
  std::memcpy(out, v, sizeof(v));
  return CTIS_OK;
}

ctis_status ctis_set_option(ctis_plan p, int option, int64_t value) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  std::lock_guard<std::mutex> lk(p->mu);
  switch (option) {
    case CTIS_OPT_VALIDATE_DATA: p->validate = value != 0; return CTIS_OK;
    case CTIS_OPT_USE_GRAPH: p->use_graph = value != 0; return CTIS_OK;
    case CTIS_OPT_PROJECTOR: {
      if (value != 0 && value != 1) return fail(CTIS_ERR_INVALID_ARGUMENT, "projector must be 0 (taps) or 1 (FFT)");
      if (value == 1 && !p->fft) {
        if ((long long)p->w * ((long long)p->n / 2 + 1) >= (1LL << 31))
          return fail(CTIS_ERR_UNSUPPORTED, "FFT projector: w * (n/2 + 1) must be < 2^31");
        DeviceGuard dg(p->device);
        cudaError_t e = fft_create(&p->fft, p->a, p->alpha, p->w, p->gamma, p->xi, p->band_taps, p->inv_h);
        if (e == cudaErrorMemoryAllocation) return fail(CTIS_ERR_OUT_OF_MEMORY, "FFT projector buffers");
        if (e != cudaSuccess) return cuda_fail(e, "FFT projector setup (cuFFT)");
      }
      if (p->projector != (int)value) {  // captured graphs bake the projector in
        for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
        p->graphs.clear();
        for (auto& kv : p->mon_graphs) cudaGraphExecDestroy(kv.second);
        p->mon_graphs.clear();
      }
      p->projector = (int)value;
      return CTIS_OK;
    }
    case CTIS_OPT_EXCHANGE:
      if (value != 0 && value != 1) return fail(CTIS_ERR_INVALID_ARGUMENT, "exchange must be 0 (NCCL) or 1 (fused)");
      p->exchange = (int)value;
      return CTIS_OK;
    case CTIS_OPT_FUSED_RATIO:
      if (p->fused_ratio != (value != 0)) {
        for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
        p->graphs.clear();
      }
      p->fused_ratio = value != 0;
      return CTIS_OK;
    default: return fail(CTIS_ERR_INVALID_ARGUMENT, "unknown option");
  }
}

size_t ctis_workspace_bytes(ctis_plan p, int64_t frames) {
  if (!p || frames < 1) return 0;
  return 2 * (((size_t)p->n * (size_t)frames + 3) & ~(size_t)3) * sizeof(float);
}

ctis_status ctis_forward_batched(ctis_plan p, const float* f, float* g_hat, int64_t frames, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_frames(frames);
  if (st) return st;
  if ((st = check_ptrs({f, g_hat}))) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  ctis_plan_s& Q = *layout_for(*p, frames);
  p->last_launches = 0;
  CTIS_CUDA(cudaMemsetAsync(g_hat, 0, sizeof(float) * (size_t)p->n * frames, s), "forward memset");
  CTIS_CUDA(enqueue_forward(Q, f, g_hat, (int)frames, s, &p->last_launches), "forward");
  return CTIS_OK;
}

ctis_status ctis_forward_accumulate(ctis_plan p, const float* f, float* g_hat, int64_t frames, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_frames(frames);
  if (st) return st;
  if ((st = check_ptrs({f, g_hat}))) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  p->last_launches = 0;
  CTIS_CUDA(enqueue_forward(*layout_for(*p, frames), f, g_hat, (int)frames, (cudaStream_t)stream, &p->last_launches),
            "forward");
  return CTIS_OK;
}

ctis_status ctis_forward(ctis_plan p, const float* f, float* g_hat, ctis_stream stream) {
  return ctis_forward_batched(p, f, g_hat, 1, stream);
}

ctis_status ctis_backproject(ctis_plan p, const float* r, float* z, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({r, z});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  p->last_launches = 0;
  CTIS_CUDA(enqueue_back(*p, r, z, 1, 0, (cudaStream_t)stream, &p->last_launches), "backproject");
  return CTIS_OK;
}

ctis_status ctis_sensitivity(ctis_plan p, float* h, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({h});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  CTIS_CUDA(launch_sensitivity(p->d_hband, h, p->ell, p->m, (cudaStream_t)stream), "sensitivity");
  p->last_launches = 1;
  return CTIS_OK;
}

ctis_status ctis_forward_ratio(ctis_plan p, const float* f, const float* g, float* r, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({f, g, r});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  p->last_launches = 0;
  CTIS_CUDA(cudaMemsetAsync(r, 0, sizeof(float) * (size_t)p->n, s), "forward_ratio memset");
  CTIS_CUDA(enqueue_forward(*p, f, r, 1, s, &p->last_launches), "forward_ratio forward");
  CTIS_CUDA(launch_ratio(g, r, r, p->n, false, s), "forward_ratio ratio");
  p->last_launches += 1;
  return CTIS_OK;
}

ctis_status ctis_back_update(ctis_plan p, const float* r, float* f, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({r, f});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  p->last_launches = 0;
  CTIS_CUDA(enqueue_back(*p, r, f, 1, 1, (cudaStream_t)stream, &p->last_launches), "back_update");
  return CTIS_OK;
}

ctis_status ctis_mlem(ctis_plan p, const float* g, float* f, int iters, void* ws, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  std::lock_guard<std::mutex> lk(p->mu);
  return run_mlem(*p, g, f, 1, iters, ws, (cudaStream_t)stream);
}

ctis_status ctis_mlem_batched(ctis_plan p, const float* g, float* f, int64_t frames, int iters, void* ws,
                              ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  std::lock_guard<std::mutex> lk(p->mu);
  return run_mlem(*p, g, f, frames, iters, ws, (cudaStream_t)stream);
}

ctis_status ctis_smart(ctis_plan p, const float* g, float* f, int64_t frames, int iters, void* ws,
                       ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  std::lock_guard<std::mutex> lk(p->mu);
  return run_mlem(*p, g, f, frames, iters, ws, (cudaStream_t)stream, /*solver=*/1);
}

ctis_status ctis_mlem_monitored(ctis_plan p, const float* g, float* f, int max_iters, double rel_tol, void* ws,
                                double* ll, int* iters_done, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "plan is NULL");
  std::lock_guard<std::mutex> lk(p->mu);
  return run_mlem_monitored(*p, g, f, max_iters, rel_tol, ws, ll, iters_done, (cudaStream_t)stream);
}

ctis_status ctis_back_update_from_ghat(ctis_plan p, const float* g, const float* g_hat, float* f, void* ws,
                                       ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({g, g_hat, f, ws});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  float* r = static_cast<float*>(ws);
  p->last_launches = 1;
  CTIS_CUDA(launch_ratio(g, const_cast<float*>(g_hat), r, p->n, false, s), "ratio");
  CTIS_CUDA(enqueue_back(*p, r, f, 1, 1, s, &p->last_launches), "back update");
  return CTIS_OK;
}

ctis_status ctis_mlem_host(ctis_plan p, const float* g_host, float* f_host, int64_t frames, int iters,
                           ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  if (!g_host || !f_host) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL host pointer");
  ctis_status st = check_frames(frames);
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (p->host_frames < frames) {
    for (void* q : {(void*)p->d_g, (void*)p->d_f, p->d_ws})
      if (q) cudaFree(q);
    p->d_g = p->d_f = nullptr;
    p->d_ws = nullptr;
    p->host_frames = 0;
    for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
    p->graphs.clear();
    CTIS_CUDA(cudaMalloc(&p->d_g, sizeof(float) * (size_t)p->n * frames), "host-path alloc g");
    CTIS_CUDA(cudaMalloc(&p->d_f, sizeof(float) * (size_t)p->m * frames), "host-path alloc f");
    CTIS_CUDA(cudaMalloc(&p->d_ws, ctis_workspace_bytes(p, frames)), "host-path alloc ws");
    p->host_frames = frames;
  }
  const size_t gb = sizeof(float) * (size_t)p->n * frames, fb = sizeof(float) * (size_t)p->m * frames;
  CTIS_CUDA(cudaMemcpyAsync(p->d_g, g_host, gb, cudaMemcpyHostToDevice, s), "H2D g");
  CTIS_CUDA(cudaMemcpyAsync(p->d_f, f_host, fb, cudaMemcpyHostToDevice, s), "H2D f0");
  if ((st = run_mlem(*p, p->d_g, p->d_f, frames, iters, p->d_ws, s))) return st;
  CTIS_CUDA(cudaMemcpyAsync(f_host, p->d_f, fb, cudaMemcpyDeviceToHost, s), "D2H f");
  CTIS_CUDA(cudaStreamSynchronize(s), "host-path sync");
  return CTIS_OK;
}

int64_t ctis_last_launch_count(ctis_plan p) { return p ? p->last_launches : 0; }

const char* ctis_last_error(void) { return g_last_error.c_str(); }

const char* ctis_version(void) { return "libctis 0.2.0 (sm_100a, per-plan __constant__ tap pages)"; }

}  // extern "C"
