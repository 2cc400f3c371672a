// ctis_api.cu — the C ABI of libctis (include/ctis.h): plan builder, validation,
// stream-ordered entry points, CUDA-graph replay of the MLEM iterations.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ctis.h"
#include "ctis_internal.h"

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

#define CTIS_CUDA(call, where)                    \
  do {                                            \
    cudaError_t e__ = (call);                     \
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
  bool operator<(const GraphKey& o) const {
    return std::tie(g, f, ws, frames, iters) < std::tie(o.g, o.f, o.ws, o.frames, o.iters);
  }
};

}  // namespace

struct ctis_plan_s {
  int device = 0;
  Dims d{};
  int64_t band_begin = 0, band_end = 0, w_total = 0, total_taps = 0;
  bool shard = false;
  bool validate = true;
  bool use_graph = true;
  DevTables t{};
  std::vector<void*> allocations;
  int* d_flag = nullptr;
  // host-buffer path
  float* d_g = nullptr;
  float* d_f = nullptr;
  void* d_ws = nullptr;
  int64_t host_frames = 0;
  // graphs
  cudaStream_t side = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  int64_t last_launches = 0;
  std::mutex mu;

  ~ctis_plan_s() {
    DeviceGuard dg(device);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (side) cudaStreamDestroy(side);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    for (void* p : allocations) cudaFree(p);
    if (d_g) cudaFree(d_g);
    if (d_f) cudaFree(d_f);
    if (d_ws) cudaFree(d_ws);
  }
};

namespace {

template <typename T>
ctis_status upload(ctis_plan p, const std::vector<T>& v, const T** out, const char* what) {
  void* ptr = nullptr;
  size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
  CTIS_CUDA(cudaMalloc(&ptr, bytes), what);
  p->allocations.push_back(ptr);
  if (!v.empty()) CTIS_CUDA(cudaMemcpy(ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), what);
  *out = static_cast<const T*>(ptr);
  return CTIS_OK;
}

// One rectangle piece of a tap: field-stop rows [r0,r1) x cols [c0,c1) map to FPA (r+sr, c+sc).
struct Piece {
  int lam;
  float w;
  int r0, r1, c0, c1;
  int sr, sc;
};

// Split the 1-D cyclic shift by o (Eq. 7) into <= 4 pure 2-D translations.
void decompose_tap(const Dims& d, int lam, int64_t o, float w, std::vector<Piece>& out) {
  const int dr = (int)(o % d.gamma), dc = (int)(o / d.gamma);
  for (int carry = 0; carry < 2; ++carry) {
    const int r0 = carry ? std::max(0, d.gamma - dr) : 0;
    const int r1 = carry ? d.a : std::min(d.a, d.gamma - dr);
    if (r0 >= r1) continue;
    const int sr = carry ? dr - d.gamma : dr;
    const int dc1 = dc + carry;  // <= xi
    for (int wrap = 0; wrap < 2; ++wrap) {
      const int c0 = wrap ? std::max(0, d.xi - dc1) : 0;
      const int c1 = wrap ? d.alpha : std::min(d.alpha, d.xi - dc1);
      if (c0 >= c1) continue;
      const int sc = wrap ? dc1 - d.xi : dc1;
      out.push_back(Piece{lam, w, r0, r1, c0, c1, sr, sc});
    }
  }
}

ctis_status build_plan(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi, const int64_t* tap_ptr,
                       const int64_t* tap_offset, const float* tap_weight, int64_t b0, int64_t b1, bool shard,
                       int device, ctis_plan* out) {
  if (!out) return fail(CTIS_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!tap_ptr || !tap_offset || !tap_weight) return fail(CTIS_ERR_INVALID_ARGUMENT, "tap array is NULL");
  if (a < 1 || alpha < 1 || w < 1 || gamma < 1 || xi < 1)
    return fail(CTIS_ERR_DIMENSION, "a, alpha, w, gamma, xi must be >= 1");
  if (gamma < a || xi < alpha) return fail(CTIS_ERR_DIMENSION, "field stop must fit the FPA (gamma >= a, xi >= alpha)");
  const int64_t n = gamma * xi, ell = a * alpha;
  if (n >= (int64_t(1) << 31) || ell * w >= (int64_t(1) << 31))
    return fail(CTIS_ERR_DIMENSION, "n and m must be < 2^31");
  if (b0 < 0 || b1 > w || b0 >= b1) return fail(CTIS_ERR_DIMENSION, "band range must be a non-empty subrange of [0, w)");
  // --- taps: CSR, range, weights, duplicates (validated over ALL bands, shard or not)
  if (tap_ptr[0] != 0) return fail(CTIS_ERR_TAP, "tap_ptr[0] must be 0");
  for (int64_t l = 0; l < w; ++l) {
    if (tap_ptr[l + 1] <= tap_ptr[l]) return fail(CTIS_ERR_TAP, "band " + std::to_string(l) + " has no taps (or tap_ptr decreases)");
    std::vector<int64_t> offs;
    double hs = 0.0;
    for (int64_t t = tap_ptr[l]; t < tap_ptr[l + 1]; ++t) {
      if (tap_offset[t] < 0 || tap_offset[t] >= n)
        return fail(CTIS_ERR_TAP, "tap offset outside [0, n) in band " + std::to_string(l));
      const float wt = tap_weight[t];
      if (!(wt > 0.f) || !std::isfinite(wt)) return fail(CTIS_ERR_TAP, "tap weight not finite and > 0 in band " + std::to_string(l));
      offs.push_back(tap_offset[t]);
      hs += wt;
    }
    std::sort(offs.begin(), offs.end());
    if (std::adjacent_find(offs.begin(), offs.end()) != offs.end())
      return fail(CTIS_ERR_TAP, "duplicate tap offset in band " + std::to_string(l));
    if (!((float)hs > 0.f) || !std::isfinite((float)hs)) return fail(CTIS_ERR_ZERO_SENSITIVITY, "h_lambda not > 0");
  }
  int ndev = 0;
  CTIS_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(CTIS_ERR_INVALID_ARGUMENT, "device ordinal out of range");
  cudaDeviceProp prop;
  CTIS_CUDA(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10) return fail(CTIS_ERR_UNSUPPORTED, std::string("device is not sm_100 (found ") + prop.name + ")");

  DeviceGuard dg(device);
  auto* p = new ctis_plan_s();
  p->device = device;
  p->shard = shard;
  p->band_begin = b0;
  p->band_end = b1;
  p->w_total = w;
  const int wl = (int)(b1 - b0);
  p->d = Dims{(int)a, (int)alpha, wl, (int)gamma, (int)xi, (int)n, (int)ell, (int)(ell * wl)};
  const Dims& d = p->d;

  // --- per-band tables (local band index lam = l - b0), sorted by offset
  std::vector<int> band_ptr4(wl + 1, 0), band_cnt(wl, 0), toff;
  std::vector<float> tw, invh(wl), hb(wl);
  std::vector<Piece> pieces;
  for (int lam = 0; lam < wl; ++lam) {
    const int64_t l = b0 + lam;
    std::vector<std::pair<int64_t, float>> bt;
    double hs = 0.0;
    for (int64_t t = tap_ptr[l]; t < tap_ptr[l + 1]; ++t) {
      bt.emplace_back(tap_offset[t], tap_weight[t]);
      hs += tap_weight[t];
    }
    std::sort(bt.begin(), bt.end());
    band_ptr4[lam] = (int)toff.size();
    band_cnt[lam] = (int)bt.size();
    for (auto& x : bt) {
      toff.push_back((int)x.first);
      tw.push_back(x.second);
      decompose_tap(d, lam, x.first, x.second, pieces);
    }
    while (toff.size() % 4) {
      toff.push_back(0);
      tw.push_back(0.f);
    }
    hb[lam] = (float)hs;
    invh[lam] = (float)(1.0 / hs);
    p->total_taps += (int64_t)bt.size();
  }
  band_ptr4[wl] = (int)toff.size();

  // --- forward tile binning: CSR of FwdEntry per FPA tile
  const int tiles_r = (d.gamma + kFwdTileR - 1) / kFwdTileR, tiles_c = (d.xi + kFwdTileC - 1) / kFwdTileC;
  const int ntiles = tiles_r * tiles_c;
  std::vector<int> cnt(ntiles + 1, 0);
  auto for_each_tile = [&](const Piece& pc, auto&& fn) {
    const int R0 = pc.r0 + pc.sr, R1 = pc.r1 + pc.sr, C0 = pc.c0 + pc.sc, C1 = pc.c1 + pc.sc;
    for (int tc = C0 / kFwdTileC; tc <= (C1 - 1) / kFwdTileC; ++tc)
      for (int tr = R0 / kFwdTileR; tr <= (R1 - 1) / kFwdTileR; ++tr) fn(tr, tc, R0, R1, C0, C1);
  };
  for (const Piece& pc : pieces)
    for_each_tile(pc, [&](int tr, int tc, int, int, int, int) { cnt[tc * tiles_r + tr + 1]++; });
  for (int i = 0; i < ntiles; ++i) cnt[i + 1] += cnt[i];
  std::vector<FwdEntry> ent(cnt[ntiles]);
  std::vector<int> fill(cnt.begin(), cnt.end() - 1);
  for (const Piece& pc : pieces) {
    for_each_tile(pc, [&](int tr, int tc, int R0, int R1, int C0, int C1) {
      const int tR0 = tr * kFwdTileR, tR1 = tR0 + kFwdTileR, tC0 = tc * kFwdTileC, tC1 = tC0 + kFwdTileC;
      FwdEntry e{};
      e.base = pc.lam * d.ell - pc.sr - d.a * pc.sc;
      e.w = pc.w;
      e.R0 = std::max(R0, tR0);
      e.R1 = std::min(R1, tR1);
      e.C0 = std::max(C0, tC0);
      e.C1 = std::min(C1, tC1);
      e.full = (e.R0 == tR0 && e.R1 == tR1 && e.C0 == tC0 && e.C1 == tC1 && tR1 <= d.gamma && tC1 <= d.xi) ? 1 : 0;
      ent[fill[tc * tiles_r + tr]++] = e;
    });
  }

  ctis_status st;
  if ((st = upload(p, ent, &p->t.fwd_entries, "upload fwd entries")) ||
      (st = upload(p, cnt, &p->t.fwd_tile_ptr, "upload tile ptr")) ||
      (st = upload(p, band_ptr4, &p->t.band_ptr4, "upload band ptr")) ||
      (st = upload(p, band_cnt, &p->t.band_cnt, "upload band cnt")) ||
      (st = upload(p, toff, &p->t.tap_off, "upload tap offsets")) ||
      (st = upload(p, tw, &p->t.tap_w, "upload tap weights")) ||
      (st = upload(p, invh, &p->t.inv_h, "upload inv_h")) || (st = upload(p, hb, &p->t.h, "upload h"))) {
    std::string msg = g_last_error;
    delete p;
    return fail(st, msg);
  }
  p->t.tiles_r = tiles_r;
  p->t.tiles_c = tiles_c;
  cudaError_t e = cudaMalloc(&p->d_flag, sizeof(int));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_out, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "plan scratch");
  }
  p->allocations.push_back(p->d_flag);
  *out = p;
  g_last_error.clear();
  return CTIS_OK;
}

bool aligned16(const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15u) == 0; }

ctis_status check_ptrs(std::initializer_list<const void*> ptrs) {
  for (const void* x : ptrs) {
    if (!x) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL device pointer");
    if (!aligned16(x)) return fail(CTIS_ERR_INVALID_ARGUMENT, "device pointer not 16-byte aligned");
  }
  return CTIS_OK;
}

ctis_status validate_data(ctis_plan p, const float* g, const float* f, int64_t frames, cudaStream_t s) {
  CTIS_CUDA(cudaMemsetAsync(p->d_flag, 0, sizeof(int), s), "validate memset");
  CTIS_CUDA(launch_validate(g, (int64_t)p->d.n * frames, p->d_flag, s), "validate g");
  CTIS_CUDA(launch_validate(f, (int64_t)p->d.m * frames, p->d_flag, s), "validate f0");
  int flag = 0;
  CTIS_CUDA(cudaMemcpyAsync(&flag, p->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s), "validate copy");
  CTIS_CUDA(cudaStreamSynchronize(s), "validate sync");
  if (flag) return fail(CTIS_ERR_DATA, "g or f0 contains a negative, NaN or Inf value");
  return CTIS_OK;
}

// Enqueue `iters` MLEM iterations (2 kernels each) on stream s.
cudaError_t enqueue_iterations(ctis_plan p, const float* g, float* f, float* r, int frames, int iters,
                               cudaStream_t s) {
  for (int k = 0; k < iters; ++k) {
    cudaError_t e = launch_forward(p->d, p->t, f, g, r, frames, /*ratio=*/true, s);
    if (e != cudaSuccess) return e;
    e = launch_back(p->d, p->t, r, f, frames, kBackUpdate, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

ctis_status run_mlem(ctis_plan p, const float* g, float* f, int64_t frames, int iters, void* ws, cudaStream_t s) {
  if (p->shard) return fail(CTIS_ERR_INVALID_ARGUMENT, "mlem on a shard plan needs the collective: use ctis_forward + "
                                                       "all-reduce + ctis_back_update_from_ghat");
  if (iters < 0) return fail(CTIS_ERR_INVALID_ARGUMENT, "iters < 0");
  if (frames < 1 || frames > 65535) return fail(CTIS_ERR_INVALID_ARGUMENT, "frames must be in [1, 65535]");
  ctis_status st = check_ptrs({g, f, ws});
  if (st) return st;
  DeviceGuard dg(p->device);
  p->last_launches = 0;
  if (p->validate) {
    if ((st = validate_data(p, g, f, frames, s))) return st;
    p->last_launches += 2;
  }
  if (iters == 0) return CTIS_OK;
  float* r = static_cast<float*>(ws);
  if (!p->use_graph) {
    CTIS_CUDA(enqueue_iterations(p, g, f, r, (int)frames, iters, s), "mlem launch");
    p->last_launches += 2LL * iters;
    return CTIS_OK;
  }
  GraphKey key{g, f, ws, frames, iters};
  auto it = p->graphs.find(key);
  if (it == p->graphs.end()) {
    if (p->graphs.size() >= 16) {
      for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
      p->graphs.clear();
    }
    cudaGraph_t graph = nullptr;
    CTIS_CUDA(cudaStreamBeginCapture(p->side, cudaStreamCaptureModeThreadLocal), "begin capture");
    cudaError_t e = enqueue_iterations(p, g, f, r, (int)frames, iters, p->side);
    cudaError_t e2 = cudaStreamEndCapture(p->side, &graph);
    if (e != cudaSuccess) return cuda_fail(e, "capture launch");
    if (e2 != cudaSuccess) return cuda_fail(e2, "end capture");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
    it = p->graphs.emplace(key, exec).first;
  }
  CTIS_CUDA(cudaEventRecord(p->ev_in, s), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(p->side, p->ev_in, 0), "stream wait");
  CTIS_CUDA(cudaGraphLaunch(it->second, p->side), "graph launch");
  CTIS_CUDA(cudaEventRecord(p->ev_out, p->side), "event record");
  CTIS_CUDA(cudaStreamWaitEvent(s, p->ev_out, 0), "stream wait");
  p->last_launches += 2LL * iters;
  return CTIS_OK;
}

}  // namespace

extern "C" {

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
  const int64_t v[10] = {p->d.a, p->d.alpha, p->d.w, p->d.gamma, p->d.xi, p->d.n, p->d.m,
                         p->band_begin, p->band_end, p->total_taps};
  std::memcpy(out, v, sizeof(v));
  return CTIS_OK;
}

ctis_status ctis_set_option(ctis_plan p, int option, int64_t value) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  std::lock_guard<std::mutex> lk(p->mu);
  switch (option) {
    case CTIS_OPT_VALIDATE_DATA: p->validate = value != 0; return CTIS_OK;
    case CTIS_OPT_USE_GRAPH: p->use_graph = value != 0; return CTIS_OK;
    default: return fail(CTIS_ERR_INVALID_ARGUMENT, "unknown option");
  }
}

size_t ctis_workspace_bytes(ctis_plan p, int64_t frames) {
  if (!p || frames < 1) return 0;
  return (size_t)p->d.n * (size_t)frames * sizeof(float);
}

ctis_status ctis_forward_batched(ctis_plan p, const float* f, float* g_hat, int64_t frames, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  if (frames < 1 || frames > 65535) return fail(CTIS_ERR_INVALID_ARGUMENT, "frames must be in [1, 65535]");
  ctis_status st = check_ptrs({f, g_hat});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  CTIS_CUDA(launch_forward(p->d, p->t, f, nullptr, g_hat, (int)frames, false, (cudaStream_t)stream), "forward");
  p->last_launches = 1;
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
  CTIS_CUDA(launch_back(p->d, p->t, r, z, 1, kBackOnly, (cudaStream_t)stream), "backproject");
  p->last_launches = 1;
  return CTIS_OK;
}

ctis_status ctis_sensitivity(ctis_plan p, float* h, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({h});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  CTIS_CUDA(launch_sensitivity(p->d, p->t, h, (cudaStream_t)stream), "sensitivity");
  p->last_launches = 1;
  return CTIS_OK;
}

ctis_status ctis_mlem(ctis_plan p, const float* g, float* f, int iters, void* ws, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  std::lock_guard<std::mutex> lk(p->mu);
  return run_mlem(p, g, f, 1, iters, ws, (cudaStream_t)stream);
}

ctis_status ctis_mlem_batched(ctis_plan p, const float* g, float* f, int64_t frames, int iters, void* ws,
                              ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  std::lock_guard<std::mutex> lk(p->mu);
  return run_mlem(p, g, f, frames, iters, ws, (cudaStream_t)stream);
}

ctis_status ctis_forward_ratio(ctis_plan p, const float* f, const float* g, float* r, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({f, g, r});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  CTIS_CUDA(launch_forward(p->d, p->t, f, g, r, 1, true, (cudaStream_t)stream), "forward_ratio");
  p->last_launches = 1;
  return CTIS_OK;
}

ctis_status ctis_back_update(ctis_plan p, const float* r, float* f, ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({r, f});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  CTIS_CUDA(launch_back(p->d, p->t, r, f, 1, kBackUpdate, (cudaStream_t)stream), "back_update");
  p->last_launches = 1;
  return CTIS_OK;
}

ctis_status ctis_back_update_from_ghat(ctis_plan p, const float* g, const float* g_hat, float* f, void* ws,
                                       ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  ctis_status st = check_ptrs({g, g_hat, f, ws});
  if (st) return st;
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  float* r = static_cast<float*>(ws);
  CTIS_CUDA(launch_ratio(g, g_hat, r, p->d.n, (cudaStream_t)stream), "ratio");
  CTIS_CUDA(launch_back(p->d, p->t, r, f, 1, kBackUpdate, (cudaStream_t)stream), "back update");
  p->last_launches = 2;
  return CTIS_OK;
}

ctis_status ctis_mlem_host(ctis_plan p, const float* g_host, float* f_host, int64_t frames, int iters,
                           ctis_stream stream) {
  if (!p) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL plan");
  if (!g_host || !f_host) return fail(CTIS_ERR_INVALID_ARGUMENT, "NULL host pointer");
  if (frames < 1 || frames > 65535) return fail(CTIS_ERR_INVALID_ARGUMENT, "frames must be in [1, 65535]");
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (p->host_frames < frames) {
    if (p->d_g) cudaFree(p->d_g);
    if (p->d_f) cudaFree(p->d_f);
    if (p->d_ws) cudaFree(p->d_ws);
    p->d_g = p->d_f = nullptr;
    p->d_ws = nullptr;
    p->host_frames = 0;
    for (auto& kv : p->graphs) cudaGraphExecDestroy(kv.second);
    p->graphs.clear();
    CTIS_CUDA(cudaMalloc(&p->d_g, sizeof(float) * (size_t)p->d.n * frames), "host-path alloc g");
    CTIS_CUDA(cudaMalloc(&p->d_f, sizeof(float) * (size_t)p->d.m * frames), "host-path alloc f");
    CTIS_CUDA(cudaMalloc(&p->d_ws, sizeof(float) * (size_t)p->d.n * frames), "host-path alloc ws");
    p->host_frames = frames;
  }
  const size_t gb = sizeof(float) * (size_t)p->d.n * frames, fb = sizeof(float) * (size_t)p->d.m * frames;
  CTIS_CUDA(cudaMemcpyAsync(p->d_g, g_host, gb, cudaMemcpyHostToDevice, s), "H2D g");
  CTIS_CUDA(cudaMemcpyAsync(p->d_f, f_host, fb, cudaMemcpyHostToDevice, s), "H2D f0");
  ctis_status st = run_mlem(p, p->d_g, p->d_f, frames, iters, p->d_ws, s);
  if (st) return st;
  CTIS_CUDA(cudaMemcpyAsync(f_host, p->d_f, fb, cudaMemcpyDeviceToHost, s), "D2H f");
  CTIS_CUDA(cudaStreamSynchronize(s), "host-path sync");
  return CTIS_OK;
}

int64_t ctis_last_launch_count(ctis_plan p) { return p ? p->last_launches : 0; }

const char* ctis_last_error(void) { return g_last_error.c_str(); }

const char* ctis_version(void) { return "libctis 0.1.0 (sm_100a)"; }

}  // extern "C"
