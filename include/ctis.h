/*
 * ctis.h — C ABI of libctis: the B200 (sm_100a) hot path of the shift-invariant
 * CTIS MLEM reconstruction of arXiv 2006.01573 (White, Bell, Haygood).
 *
 * The operator (PAPER.md line numbers, "P:<line>"):
 *   A CTIS maps a datacube f (a x alpha field stop, w wavelength bands) onto an
 *   FPA image g (gamma x xi pixels) by the linear model g = H f (Eq. 1).
 *   By shift-invariance H = (C_1 E ... C_w E) (Eqs. 3-8): E embeds a
 *   band's a x alpha block into the FPA (Eqs. 5-6; index map P:131-133)
 *   and C_lambda is the n x n circulant whose first column c_lambda is the band's
 *   calibration image for a point source at field-stop pixel (0,0) (Eq. 7;
 *   P:24).  This library stores each c_lambda as a sparse list of taps
 *   (offset o, weight w): o is the column-major FPA index of a nonzero of
 *   c_lambda, so voxel (r, c) of band lambda adds w * f to FPA pixel
 *   (r + gamma*c + o) mod n — exactly the 1-D circulant of Eq. 7, including the
 *   carry into the next FPA column and the wrap past pixel n-1.
 *
 * Layouts (column-major everywhere, reading R1; P:24 allows either):
 *   f      float32[w][alpha][a]   element (lam, c, r) at lam*a*alpha + c*a + r    (Eq. 9)
 *   g, g_hat, r  float32[xi][gamma]  pixel (R, C) at R + gamma*C
 *   batched:  g[F][n], f[F][m] (frame-major, contiguous).
 *
 * Conventions for every entry point:
 *   - sizes are int64_t; n = gamma*xi, l = a*alpha, m = l*w (or l*(band_end-band_begin)
 *     for a shard plan, "m_local"); n must be < 2^30 and m < 2^31.
 *   - float* arguments of the stream-ordered calls are DEVICE pointers on the plan's
 *     device, owned by the caller, 16-byte aligned, non-overlapping unless stated.
 *     The plan owns only its tap tables and a few bytes of scratch.
 *   - calls are stream-ordered and asynchronous: CTIS_OK means "validated and
 *     enqueued on `stream`" (NULL = the legacy default stream).  Kernel faults
 *     surface as CTIS_ERR_CUDA on a later call or at stream synchronisation.
 *   - on any error nothing is enqueued, outputs are unspecified, inputs untouched;
 *     ctis_last_error() gives a one-line reason (thread-local).
 *   - a plan may be used from several host threads, calls are serialised internally.
 *   - no CPU fallback: every arithmetic step runs in sm_100a kernels; on a device
 *     that is not compute capability 10.x plan creation fails with CTIS_ERR_UNSUPPORTED.
 */
#ifndef CTIS_H_
#define CTIS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define CTIS_API __attribute__((visibility("default")))
#else
#define CTIS_API
#endif

typedef struct ctis_plan_s* ctis_plan;
/* Identical to cudaStream_t (struct CUstream_st*). */
typedef struct CUstream_st* ctis_stream;

typedef enum {
  CTIS_OK = 0,
  CTIS_ERR_INVALID_ARGUMENT = 1, /* null pointer, iters < 0, frames < 1, misaligned pointer,
                                    wrong call for the plan kind (mlem on a shard plan) */
  CTIS_ERR_DIMENSION = 2,        /* a, alpha, w, gamma, xi < 1; gamma < a; xi < alpha; n >= 2^30; m >= 2^31;
                                    band range outside [0, w) or empty */
  CTIS_ERR_TAP = 3,              /* tap_ptr not a CSR over w bands; offset outside [0, n);
                                    weight <= 0 or non-finite; duplicate offset within a band;
                                    band with no taps */
  CTIS_ERR_ZERO_SENSITIVITY = 4, /* h_lambda = sum_t w_t not > 0 in float32 */
  CTIS_ERR_DATA = 5,             /* g or f0 negative, NaN or Inf (validated by ctis_mlem*) */
  CTIS_ERR_CUDA = 6,             /* CUDA runtime error; see ctis_last_error() */
  CTIS_ERR_OUT_OF_MEMORY = 7,
  CTIS_ERR_UNSUPPORTED = 8       /* device is not compute capability 10.x (sm_100) */
} ctis_status;

/* Options for ctis_set_option. */
typedef enum {
  CTIS_OPT_VALIDATE_DATA = 1,   /* 1 (default): ctis_mlem* check g >= 0, f0 >= 0, finite, with one
                                   reduction kernel and ONE host synchronisation per call;
                                   0: skip (the call is then fully asynchronous). */
  CTIS_OPT_USE_GRAPH = 2,       /* 1 (default): ctis_mlem* replay a captured CUDA graph of the
                                   iterations; 0: launch kernels directly on `stream`. */
  CTIS_OPT_PROJECTOR = 3,       /* 0 (default): the tap projector.  1: the paper's own Fourier route
                                   (Eqs. 13 and 17 with cuFFT, d_i = F c_i precomputed; Alg. 1
                                   lines 6-11) for every ctis_forward / _backproject / _mlem* call on the
                                   plan — a comparator arm.  Allocates O(w n) complex
                                   scratch owned by the plan (CTIS_ERR_OUT_OF_MEMORY if it does not fit):
                                   calls on one plan must then not run concurrently on different streams. */
  CTIS_OPT_FUSED_RATIO = 4,     /* 1: ctis_mlem / ctis_mlem_batched / ctis_smart on plans with
                                   persistent (TMA) forward kernels run two kernels per iteration: the
                                   forward's last launch is cooperative and, after a grid-wide barrier,
                                   turns g_hat into r = g (/) g_hat in place (Alg. 1 line 8); the back
                                   kernel zeroes the other workspace half for the next forward.
                                   0 (default): three kernels per iteration (separate ratio pass),
                                   measured faster on B200 (C4 149.5 vs 150.8 us per iteration). */
  CTIS_OPT_EXCHANGE = 5         /* latency mode (ctis_mlem_band_sharded) exchange: 0 (default) NCCL
                                   reduce-scatter + ratio kernel + all-gather; 1 ONE fused kernel over
                                   NVLink peer memory: the exchange buffer is an NCCL
                                   symmetric-memory window owned by the communicator, each rank reduces
                                   its pixel slice across all ranks (multimem.ld_reduce over NVSwitch when
                                   NVLS is available, else peer loads), forms r = g (/) g_hat and stores it
                                   to every rank (multimem.st / peer stores).  Needs NCCL >= 2.28; the
                                   `ws` argument is then unused. */
} ctis_option;

/* Create a plan for the full operator H (all w bands).
 *   a, alpha   field stop rows x columns
 *   w          number of wavelength bands
 *   gamma, xi  FPA rows x columns
 *   tap_ptr    HOST, w+1 entries, CSR: band lam owns taps [tap_ptr[lam], tap_ptr[lam+1])
 *   tap_offset HOST, column-major FPA index in [0, n) of a nonzero of c_lam
 *   tap_weight HOST, the value of c_lam there: finite, > 0
 *   device     CUDA device ordinal the plan (and every buffer passed to it) lives on
 * The calibration is copied and pre-processed (sorted, split into rectangle
 * pieces, binned per FPA tile); the host arrays may be freed on return.
 * The per-band sensitivity h_lam = sum_t w_t (every column of a circulant
 * block has the same sum) is computed in double and must be > 0. */
CTIS_API ctis_status ctis_plan_create(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                             const int64_t* tap_ptr, const int64_t* tap_offset,
                             const float* tap_weight, int device, ctis_plan* out);

/* Latency-mode shard plan: same full CSR, but the plan keeps only bands
 * [band_begin, band_end) (Eq. 3: H's block columns).  Its f is the
 * m_local = a*alpha*(band_end-band_begin) slice of those bands; ctis_forward
 * writes the PARTIAL sum over its bands (summed across shards by the caller's
 * collective); ctis_mlem / ctis_mlem_batched return CTIS_ERR_INVALID_ARGUMENT. */
CTIS_API ctis_status ctis_plan_create_shard(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                                   const int64_t* tap_ptr, const int64_t* tap_offset,
                                   const float* tap_weight, int64_t band_begin, int64_t band_end,
                                   int device, ctis_plan* out);

CTIS_API void ctis_plan_destroy(ctis_plan plan);

/* Plan dimensions: out[0..9] = a, alpha, w_local, gamma, xi, n, m_local, band_begin,
 * band_end, total taps stored.  Host-side, no device work. */
CTIS_API ctis_status ctis_plan_dims(ctis_plan plan, int64_t out[10]);

/* Plan layout (host-side, no device work; tests and profiling): out[0..9] = forward tap pages,
 * back tap pages, forward chunk passes, back chunks, forward uses TMA (0/1), back uses TMA (0/1),
 * back bands per chunk (NB), back tile columns, forward kernel (> 0: classic forward with this many
 * modes per pass; < 0: strip forward with -out[8] consumer warps), forward work items
 * per frame.  A page is one 64 KB __constant__ bank of tap tables (one kernel launch per page and
 * projection).  CTIS_ERR_INVALID_ARGUMENT if plan or out is NULL.
 *
 * Plan-owned scratch, allocated on first use outside any stream capture: a row-repacked copy of f
 * for field stops with a % 4 != 0 (frames x round4(a) x alpha x w floats; the TMA forward needs a
 * 16-byte row pitch) and a partial-z buffer (frames x m floats) for plans whose back projection is
 * mode-split (too few work items to fill the SMs).  ctis_mlem* allocate them before capturing their
 * CUDA graph; a first forward / back projection captured into the CALLER's graph fails with
 * CTIS_ERR_CUDA (stream capture) — run one uncaptured call first. */
CTIS_API ctis_status ctis_plan_info(ctis_plan plan, int64_t out[10]);

CTIS_API ctis_status ctis_set_option(ctis_plan plan, int option, int64_t value);

/* Bytes of caller-allocated device workspace needed by ctis_mlem* and
 * ctis_back_update_from_ghat for `frames` frames (frames >= 1): holds r = g / g_hat. */
CTIS_API size_t ctis_workspace_bytes(ctis_plan plan, int64_t frames);

/* g_hat = H f (Eqs. 8-13): f[m_local] -> g_hat[n], overwritten. */
CTIS_API ctis_status ctis_forward(ctis_plan plan, const float* f, float* g_hat, ctis_stream stream);

/* Batched forward: f[frames][m_local] -> g_hat[frames][n]. */
CTIS_API ctis_status ctis_forward_batched(ctis_plan plan, const float* f, float* g_hat, int64_t frames,
                                 ctis_stream stream);

/* g_hat += H f without clearing g_hat first (the forward kernels accumulate band-chunk
 * partials with red.global.add): f[frames][m_local], g_hat[frames][n]. */
CTIS_API ctis_status ctis_forward_accumulate(ctis_plan plan, const float* f, float* g_hat, int64_t frames,
                                             ctis_stream stream);

/* z = H^T r (Eqs. 14-17): r[n] -> z[m_local], overwritten. */
CTIS_API ctis_status ctis_backproject(ctis_plan plan, const float* r, float* z, ctis_stream stream);

/* h = H^T 1: h[m_local], overwritten; h_j = sum of band lam(j)'s tap weights. */
CTIS_API ctis_status ctis_sensitivity(ctis_plan plan, float* h, ctis_stream stream);

/* MLEM (Eq. 2, Alg. 1): `iters` iterations of
 *   g_hat = H f;  r = g (/) g_hat  (r_p = 0 where g_hat_p = 0);  f <- f (.) (H^T r) (/) h
 * in place on f (in: f^(1), out: f^(iters+1)); g[n] is read only; ws must hold
 * ctis_workspace_bytes(plan, 1) bytes.  iters = 0 leaves f unchanged. */
CTIS_API ctis_status ctis_mlem(ctis_plan plan, const float* g, float* f, int iters, void* ws,
                      ctis_stream stream);

/* Snapshot-video batch: `frames` independent reconstructions sharing the plan;
 * g[frames][n], f[frames][m] in place, ws >= ctis_workspace_bytes(plan, frames). */
CTIS_API ctis_status ctis_mlem_batched(ctis_plan plan, const float* g, float* f, int64_t frames, int iters,
                              void* ws, ctis_stream stream);

/* The two fused kernels of one MLEM iteration, exposed for step-wise drivers and timing:
 *   ctis_forward_ratio: r = g (/) (H f), r_p = 0 where (H f)_p = 0     (Alg. 1 lines 6-8)
 *                       f[m], g[n] -> r[n] (r may be the ctis_mlem workspace)
 *   ctis_back_update:   f <- f (.) (H^T r) (/) h, in place             (Alg. 1 lines 9-12) */
CTIS_API ctis_status ctis_forward_ratio(ctis_plan plan, const float* f, const float* g, float* r,
                                        ctis_stream stream);
CTIS_API ctis_status ctis_back_update(ctis_plan plan, const float* r, float* f, ctis_stream stream);

/* Latency mode, second half of an iteration on a shard plan: given the measured
 * g[n] and the all-reduced g_hat[n] = H f (sum over all shards), compute
 * r = g (/) g_hat into ws and update this shard's f[m_local] <- f (.) (H_shard^T r) (/) h. */
CTIS_API ctis_status ctis_back_update_from_ghat(ctis_plan plan, const float* g, const float* g_hat, float* f,
                                       void* ws, ctis_stream stream);

/* SMART, the simultaneous form of the MART solver on the
 * same projector, testing the paper's "solver agnostic" claim:
 *   g_hat = H f;  r_p = log(g_p / g_hat_p) where g_p > 0 and g_hat_p > 0, else 0;
 *   f <- f (.) exp( (H^T r) (/) h )
 * `frames` >= 1 independent frames g[frames][n], f[frames][m] in place; ws as ctis_mlem_batched;
 * iters = 0 leaves f unchanged.  Errors as ctis_mlem_batched. */
CTIS_API ctis_status ctis_smart(ctis_plan plan, const float* g, float* f, int64_t frames, int iters, void* ws,
                                ctis_stream stream);

/* MLEM with the per-iteration Poisson log-likelihood and an early stop (the paper
 * recommends stopping early after Hagen; L is the objective EM ascends, shepp1982maximum):
 *   iteration k (k = 1, 2, ...): g_hat = H f^(k); ll[k-1] = L_k = sum_p [g_p log g_hat_p - g_hat_p]
 *   (pixels with g_hat_p <= 0 add 0 if g_p = 0, else -inf); r = g (/) g_hat; f^(k+1) = f (.) (H^T r) (/) h;
 *   after update k >= 2 stop if L_k - L_{k-1} <= rel_tol * |L_k| (rel_tol <= 0: only an exact
 *   stall stops), and always after max_iters updates.
 * Single frame.  g[n] read only, f[m] in place (f^(1) in, f^(iters_done+1) out), ws as ctis_mlem.
 * ll: DEVICE array of max_iters doubles (8-byte aligned; entries >= iters_done are 0);
 * iters_done: DEVICE int (4-byte aligned), the number of updates performed.  The loop runs on the
 * device (a CUDA-graph conditional WHILE node): no host round trip per iteration.  L is accumulated
 * in fp64 from fp32 g_hat (logf).  Errors: as ctis_mlem; CTIS_ERR_UNSUPPORTED if the driver lacks
 * conditional graph nodes; max_iters < 0 -> CTIS_ERR_INVALID_ARGUMENT; max_iters = 0 sets
 * *iters_done = 0 and leaves f unchanged. */
CTIS_API ctis_status ctis_mlem_monitored(ctis_plan plan, const float* g, float* f, int max_iters, double rel_tol,
                                         void* ws, double* ll, int* iters_done, ctis_stream stream);

/* ---- Latency mode over NCCL ---------------------------------------------
 * H = (H_1 ... H_w) is a row of per-band block columns (Eq. 3), so with the bands
 * split over P ranks g_hat = H f = sum over ranks of H_shard f_shard.  One iteration of
 * ctis_mlem_band_sharded on every rank (Alg. 1):
 *   X <- 0 on the exchange range; X += H_shard f_shard (partial forward, lines 6-7);
 *   reduce-scatter(X) (NCCL, sum): rank k holds g_hat on its slice k of the exchange range;
 *   X_k <- g_k (/) X_k on that slice (line 8; 0 where g_hat <= 0, reading R4);
 *   all-gather(X): every rank holds r = g (/) g_hat on the whole range;
 *   f_shard <- f_shard (.) (H_shard^T r) (/) h (lines 9-12).
 * The exchange range is the contiguous FPA index range [lo, hi] that any tap of ANY band can reach
 * (min_t o_t .. max_t o_t + E(l-1); the whole [0, n) if a tap wraps), split into P equal 16-byte
 * aligned slices: pixels outside it are zero in every partial and never read.  All `iters`
 * iterations are enqueued as ONE CUDA graph (kernels and NCCL calls), replayed without host
 * synchronisation.  NCCL is loaded at run time (libnccl.so.2); without it these calls return
 * CTIS_ERR_UNSUPPORTED. */
typedef struct ctis_comm_s* ctis_comm;

/* 128-byte NCCL unique id, created on one rank and broadcast to all (the caller's side channel). */
CTIS_API ctis_status ctis_comm_unique_id(uint8_t id[128]);

/* Collective: every rank of the group calls it with the same id and nranks, its own rank and the
 * device its shard plans use.  *out is owned by the caller (ctis_comm_destroy). */
CTIS_API ctis_status ctis_comm_create(int nranks, int rank, const uint8_t id[128], int device, ctis_comm* out);
CTIS_API void ctis_comm_destroy(ctis_comm comm);

/* Device workspace bytes for ctis_mlem_band_sharded on this shard plan and communicator (the
 * exchange buffer X, >= n floats, 16-byte aligned). */
CTIS_API size_t ctis_band_sharded_workspace_bytes(ctis_plan shard, ctis_comm comm);

/* `iters` band-sharded MLEM iterations (above).  Collective over `comm`: every rank calls it with
 * its own shard plan (band ranges partitioning [0, w), all created from the same full tap CSR).
 * g: DEVICE, n floats, the full measurement (replicated on every rank; read only).
 * f_local: DEVICE, m_local floats of this rank's bands, updated in place (f^(1) in, f^(iters+1) out).
 * ws: DEVICE, ctis_band_sharded_workspace_bytes bytes.  Stream-ordered on `stream`.
 * Errors: CTIS_ERR_INVALID_ARGUMENT (NULL / misaligned pointers, iters < 0, a plan of another
 * device), CTIS_ERR_UNSUPPORTED (no NCCL), CTIS_ERR_CUDA (CUDA or NCCL failure, text in
 * ctis_last_error).  iters = 0 leaves f_local unchanged. */
CTIS_API ctis_status ctis_mlem_band_sharded(ctis_plan shard, ctis_comm comm, const float* g, float* f_local,
                                            int iters, void* ws, ctis_stream stream);

/* End-to-end convenience on HOST buffers: copies g_host[frames][n] and
 * f_host[frames][m] (f0) to plan-owned device buffers, runs ctis_mlem_batched,
 * copies f back into f_host and synchronises `stream` before returning.
 * Pinned host memory gives full PCIe/NVLink-C2C bandwidth; pageable works too. */
CTIS_API ctis_status ctis_mlem_host(ctis_plan plan, const float* g_host, float* f_host, int64_t frames,
                           int iters, ctis_stream stream);

/* Number of kernel launches the last ctis_* call on this plan enqueued (graph
 * replays count the kernels inside the graph). */
CTIS_API int64_t ctis_last_launch_count(ctis_plan plan);

/* One-line description of the last error on this host thread ("" if none). */
CTIS_API const char* ctis_last_error(void);

/* Library version string. */
CTIS_API const char* ctis_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CTIS_H_ */
