/*
 * ctis_oracle.c — plain, slow, double-precision CPU oracle for the CTIS MLEM
 * hot path of arXiv 2006.01573 (White, Bell, Haygood).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or execute this
 * file.  It shares no code, header, table or constant with the CUDA path
 * (paper_2006_01573_b200/), and nothing in the product imports it.
 *
 * What it computes, step by step in the paper's notation (PAPER.md line numbers):
 *   geometry      a x alpha field stop, gamma x xi FPA, w bands;
 *                 n = gamma*xi, l = a*alpha, m = l*w
 *   embed  v = (I_w (x) E) f as the zero-based index map                  (Eq. 11)
 *          i = j - s*l + (gamma-a)*floor((j - s*l)/a) + s*n,  s = floor(j/l)
 *   forward g = H f = sum_i C_i v_i, C_i circulant with first column c_i   (Eq. 7,
 *                                                                           P:135-139 Eq. 12)
 *          (C v)[p] = sum_k c[(p-k) mod n] v[k]; c_i is sparse: taps (o_t, w_t)
 *          so every nonzero v[k] adds w_t*v[k] to p = (k + o_t) mod n.
 *   back   z_i = C_i^T u, zeta = (I_w (x) E)^T z                           (Eqs. 14-15)
 *          (C^T u)[k] = sum_p c[(p-k) mod n] u[p] = sum_t w_t u[(k + o_t) mod n]
 *          extract map: zeta_i = z_j, j = i - s*l + (gamma-a)*floor((i-s*l)/a) + s*n
 *   sens.  h_j = sum_i H_ij = (H^T 1)_j
 *   MLEM   Alg. 1: for k = 1..K:
 *            g^(k) = H f^(k)            (lines 6-7)
 *            u = g (/) g^(k)            (line 8; u_p = 0 where g^(k)_p = 0, R4)
 *            zeta = H^T u               (lines 9-11)
 *            f^(k+1) = (f^(k) (.) zeta) (/) h   (line 12, Alg. 1's operation order, R7)
 *
 * Summation order (so that the dense product of the tests is matched bit for bit):
 *   forward: each g[p] accumulates its terms in ascending voxel index j, starting
 *            from +0.0 (the order of the dense sum_j H_pj f_j);
 *   back:    each zeta[j] accumulates its terms in ascending FPA index p
 *            (the order of the dense sum_p H_pj u_p): the band's taps are sorted by
 *            offset and the walk starts at the first tap that wraps past n.
 * Build with -O2 -ffp-contract=off (no fused multiply-add, no fast-math).
 *
 * Threads (oracle_set_threads, OpenMP): the paper-sized configurations (C4: 321 M tap incidences
 * per projection) take seconds per iteration on one core.  With more than one thread, MLEM, SMART
 * and the monitored MLEM run forward/back through oracle_forward_par / oracle_backproject_par and
 * split their element-wise loops over threads.  Every output element still receives exactly the
 * same sequence of floating-point operations as in the serial functions (the parallel forward walks
 * each pixel's terms in ascending j, see oracle_forward_par), so the results are bit-identical to the
 * serial path; tests/test_oracle_pins.py pins that.  The serial oracle_forward / oracle_backproject
 * stay the functions checked against the dense H.
 *
 * Pins (tests/test_oracle_*.py, all -m "not gpu"): dense H built literally from
 * Eqs. 3-7 (bit-exact), the paper's own FFT algorithm Eqs. 13/17 (<= 1e-12),
 * scipy convolve2d/correlate2d for non-wrapping taps, impulse/shift identities,
 * adjointness, closed-form column sums, MLEM invariants (nonnegativity,
 * conservation, monotone Poisson likelihood, fixed point, zero image) and
 * Richardson-Lucy for w = 1.
 */
#include <stdint.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Error codes of the oracle (small, independent of the product's). */
#define OR_OK 0
#define OR_EDIM 1
#define OR_ETAP 2
#define OR_ENOMEM 3

static int check_geom(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi) {
    if (a < 1 || alpha < 1 || w < 1 || gamma < a || xi < alpha) return OR_EDIM;
    return OR_OK;
}

/* Eq. 11: index of voxel j of f inside v = (I_w (x) E) f. */
int64_t oracle_embed_index(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                           int64_t j) {
    (void)w;
    int64_t n = gamma * xi, l = a * alpha;
    int64_t s = j / l;
    return j - s * l + (gamma - a) * ((j - s * l) / a) + s * n;
}

/* Eq. 15: index into z read by zeta_i (same formula with i <-> j). */
int64_t oracle_extract_index(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                             int64_t i) {
    return oracle_embed_index(a, alpha, w, gamma, xi, i);
}

static int check_taps(int64_t w, int64_t n, const int64_t* ptr, const int64_t* off) {
    if (ptr[0] != 0) return OR_ETAP;
    for (int64_t s = 0; s < w; ++s) {
        if (ptr[s + 1] < ptr[s]) return OR_ETAP;
        for (int64_t t = ptr[s]; t < ptr[s + 1]; ++t)
            if (off[t] < 0 || off[t] >= n) return OR_ETAP;
    }
    return OR_OK;
}

/* g = H f  (Eq. 12 with v from Eq. 11).  f: m doubles, g: n doubles (overwritten). */
int oracle_forward(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                   const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                   const double* f, double* g) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi, m = a * alpha * w;
    if ((rc = check_taps(w, n, tap_ptr, tap_offset))) return rc;
    for (int64_t p = 0; p < n; ++p) g[p] = 0.0;
    for (int64_t j = 0; j < m; ++j) {                 /* ascending j */
        int64_t i = oracle_embed_index(a, alpha, w, gamma, xi, j);
        int64_t s = i / n, k = i - s * n;              /* v_s[k] = f[j] */
        for (int64_t t = tap_ptr[s]; t < tap_ptr[s + 1]; ++t) {
            int64_t p = (k + tap_offset[t]) % n;       /* C_s[p,k] = c_s[(p-k) mod n] */
            double prod = tap_weight[t] * f[j];
            g[p] = g[p] + prod;
        }
    }
    return OR_OK;
}

/* Sort tap indices of one band by offset (insertion sort: small, obviously correct). */
static void sort_band(const int64_t* off, int64_t begin, int64_t end, int64_t* idx) {
    int64_t cnt = end - begin;
    for (int64_t q = 0; q < cnt; ++q) idx[q] = begin + q;
    for (int64_t q = 1; q < cnt; ++q) {
        int64_t v = idx[q], r = q - 1;
        while (r >= 0 && off[idx[r]] > off[v]) { idx[r + 1] = idx[r]; --r; }
        idx[r + 1] = v;
    }
}

/* zeta = H^T u  (Eqs. 14-15).  u: n doubles, zeta: m doubles (overwritten). */
int oracle_backproject(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                       const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                       const double* u, double* zeta) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi, m = a * alpha * w;
    if ((rc = check_taps(w, n, tap_ptr, tap_offset))) return rc;
    int64_t nnz = tap_ptr[w];
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    if (!order) return OR_ENOMEM;
    for (int64_t s = 0; s < w; ++s) sort_band(tap_offset, tap_ptr[s], tap_ptr[s + 1], order + tap_ptr[s]);
    for (int64_t i = 0; i < m; ++i) {
        int64_t jj = oracle_extract_index(a, alpha, w, gamma, xi, i);
        int64_t s = jj / n, k = jj - s * n;            /* zeta_i = z_s[k] = (C_s^T u)[k] */
        const int64_t* ord = order + tap_ptr[s];
        int64_t cnt = tap_ptr[s + 1] - tap_ptr[s];
        /* first tap (in ascending offset) whose destination wraps: o >= n - k */
        int64_t start = 0;
        while (start < cnt && tap_offset[ord[start]] < n - k) ++start;
        double acc = 0.0;
        for (int64_t q = 0; q < cnt; ++q) {            /* ascending destination p */
            int64_t t = ord[(start + q) % cnt];
            int64_t p = (k + tap_offset[t]) % n;
            double prod = tap_weight[t] * u[p];
            acc = acc + prod;
        }
        zeta[i] = acc;
    }
    free(order);
    return OR_OK;
}

/* ---- thread count for MLEM / SMART / monitored MLEM (1 = the plain serial functions) ---------- */
static int g_threads = 1;

int oracle_set_threads(int nthreads) {
#ifdef _OPENMP
    g_threads = nthreads < 1 ? 1 : nthreads;
#else
    (void)nthreads;
    g_threads = 1;
#endif
    return g_threads;
}

int oracle_get_threads(void) { return g_threads; }

static int check_distinct(int64_t w, const int64_t* ptr, const int64_t* off, const int64_t* order) {
    for (int64_t s = 0; s < w; ++s)
        for (int64_t q = ptr[s] + 1; q < ptr[s + 1]; ++q)
            if (off[order[q]] == off[order[q - 1]]) return OR_ETAP;
    return OR_OK;
}

/* g = H f, the same sums as oracle_forward, split over threads by ranges of output pixels p.
 * oracle_forward adds the terms of g[p] in ascending voxel index j = s*l + (k's row + a*k's column),
 * i.e. band s ascending, then ascending k = (p - o) mod n within the band.  Here each thread owns
 * pixels [P0, P1) and, band by band, applies the band's taps so that every pixel sees them in that
 * same order: for a fixed p, ascending k means first the taps with o <= p in descending o (k = p - o),
 * then the taps with o > p in descending o (k = p - o + n > p).  The set {o <= p} only changes at
 * p = o, so [P0, P1) is cut at every tap offset inside it; on each piece [q0, q1) one tap order holds
 * for all its pixels, and each tap covers the contiguous k range [q0 - o, q1 - o) (mod n), walked over
 * the columns of the field-stop image E (Eq. 11) it meets.  Offsets must be distinct within a band
 * (OR_ETAP otherwise; the serial function accepts duplicates). */
int oracle_forward_par(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                       const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                       const double* f, double* g, int nthreads) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi, l = a * alpha;
    if ((rc = check_taps(w, n, tap_ptr, tap_offset))) return rc;
    int64_t nnz = tap_ptr[w];
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    if (!order) return OR_ENOMEM;
    for (int64_t s = 0; s < w; ++s) sort_band(tap_offset, tap_ptr[s], tap_ptr[s + 1], order + tap_ptr[s]);
    if ((rc = check_distinct(w, tap_ptr, tap_offset, order))) { free(order); return rc; }
    int64_t nchunks = (int64_t)(nthreads < 1 ? 1 : nthreads) * 16;
    if (nchunks > n) nchunks = n;
    #pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads < 1 ? 1 : nthreads)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        int64_t P0 = n * ch / nchunks, P1 = n * (ch + 1) / nchunks;
        for (int64_t p = P0; p < P1; ++p) g[p] = 0.0;
        for (int64_t s = 0; s < w; ++s) {
            const int64_t* ord = order + tap_ptr[s];
            int64_t cnt = tap_ptr[s + 1] - tap_ptr[s];
            if (cnt == 0) continue;
            int64_t c = 0;                                  /* taps with o <= q0 */
            while (c < cnt && tap_offset[ord[c]] <= P0) ++c;
            int64_t q0 = P0;
            while (q0 < P1) {
                int64_t q1 = (c < cnt && tap_offset[ord[c]] < P1) ? tap_offset[ord[c]] : P1;
                for (int64_t q = 0; q < cnt; ++q) {          /* descending o, starting below q0 */
                    int64_t t = ord[((c - 1 - q) % cnt + cnt) % cnt];
                    int64_t o = tap_offset[t];
                    int64_t k0 = o <= q0 ? q0 - o : q0 - o + n, k1 = k0 + (q1 - q0);
                    for (int64_t col = k0 / gamma; col < alpha && col * gamma < k1; ++col) {
                        int64_t r0 = k0 - col * gamma > 0 ? k0 - col * gamma : 0;
                        int64_t r1 = k1 - col * gamma < a ? k1 - col * gamma : a;
                        for (int64_t r = r0; r < r1; ++r) {
                            int64_t k = col * gamma + r;
                            int64_t p = (k + o) % n;
                            int64_t j = s * l + r + a * col;
                            double prod = tap_weight[t] * f[j];
                            g[p] = g[p] + prod;
                        }
                    }
                }
                q0 = q1;
                while (c < cnt && tap_offset[ord[c]] <= q0) ++c;
            }
        }
    }
    free(order);
    return OR_OK;
}

/* zeta = H^T u, the same per-voxel sums as oracle_backproject (every zeta_i is independent), split
 * over threads by voxel. */
int oracle_backproject_par(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                           const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                           const double* u, double* zeta, int nthreads) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi, m = a * alpha * w;
    if ((rc = check_taps(w, n, tap_ptr, tap_offset))) return rc;
    int64_t nnz = tap_ptr[w];
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    if (!order) return OR_ENOMEM;
    for (int64_t s = 0; s < w; ++s) sort_band(tap_offset, tap_ptr[s], tap_ptr[s + 1], order + tap_ptr[s]);
    #pragma omp parallel for schedule(static) num_threads(nthreads < 1 ? 1 : nthreads)
    for (int64_t i = 0; i < m; ++i) {
        int64_t jj = oracle_extract_index(a, alpha, w, gamma, xi, i);
        int64_t s = jj / n, k = jj - s * n;
        const int64_t* ord = order + tap_ptr[s];
        int64_t cnt = tap_ptr[s + 1] - tap_ptr[s];
        int64_t start = 0;
        while (start < cnt && tap_offset[ord[start]] < n - k) ++start;
        double acc = 0.0;
        for (int64_t q = 0; q < cnt; ++q) {
            int64_t t = ord[(start + q) % cnt];
            int64_t p = (k + tap_offset[t]) % n;
            double prod = tap_weight[t] * u[p];
            acc = acc + prod;
        }
        zeta[i] = acc;
    }
    free(order);
    return OR_OK;
}

/* forward / back as used by the iterations: serial functions unless oracle_set_threads(> 1) */
static int fwd(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi, const int64_t* tp,
               const int64_t* to, const double* tw, const double* f, double* g) {
    return g_threads > 1 ? oracle_forward_par(a, alpha, w, gamma, xi, tp, to, tw, f, g, g_threads)
                         : oracle_forward(a, alpha, w, gamma, xi, tp, to, tw, f, g);
}
static int back(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi, const int64_t* tp,
                const int64_t* to, const double* tw, const double* u, double* z) {
    return g_threads > 1 ? oracle_backproject_par(a, alpha, w, gamma, xi, tp, to, tw, u, z, g_threads)
                         : oracle_backproject(a, alpha, w, gamma, xi, tp, to, tw, u, z);
}

/* h = H^T 1: column sums h_j = sum_i H_ij. */
int oracle_sensitivity(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                       const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                       double* h) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi;
    double* ones = (double*)malloc(sizeof(double) * (size_t)n);
    if (!ones) return OR_ENOMEM;
    for (int64_t p = 0; p < n; ++p) ones[p] = 1.0;
    rc = back(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, ones, h);
    free(ones);
    return rc;
}

/* K iterations of Alg. 1 from the caller's f (= f^(1)); f is overwritten with f^(K+1).
 * If ghat_out is non-NULL it receives g^(K) = H f^(K) of the last iteration. */
int oracle_mlem(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                const double* g, double* f, int64_t iters, double* ghat_out) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi, m = a * alpha * w;
    double* h = (double*)malloc(sizeof(double) * (size_t)m);
    double* gk = (double*)malloc(sizeof(double) * (size_t)n);
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    double* zeta = (double*)malloc(sizeof(double) * (size_t)m);
    if (!h || !gk || !u || !zeta) { rc = OR_ENOMEM; goto done; }
    if ((rc = oracle_sensitivity(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, h))) goto done;
    for (int64_t k = 0; k < iters; ++k) {
        if ((rc = fwd(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, f, gk))) goto done;
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t p = 0; p < n; ++p) u[p] = gk[p] > 0.0 ? g[p] / gk[p] : 0.0;
        if ((rc = back(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, u, zeta))) goto done;
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t j = 0; j < m; ++j) f[j] = (f[j] * zeta[j]) / h[j];
        if (ghat_out) memcpy(ghat_out, gk, sizeof(double) * (size_t)n);
    }
done:
    free(h); free(gk); free(u); free(zeta);
    return rc;
}

/* Poisson log-likelihood of the measurement g under the model ghat = H f, without the
 * f-independent -log(g_p!) term: L = sum_p [ g_p log ghat_p - ghat_p ] (the objective MLEM
 * ascends, Shepp & Vardi, cited at PAPER.md P:34).  Pixels with ghat_p <= 0 contribute 0 when
 * g_p = 0 and -infinity otherwise (reading R15).  Sum in ascending p. */
double oracle_loglik(int64_t n, const double* g, const double* ghat) {
    double L = 0.0;
    for (int64_t p = 0; p < n; ++p) {
        if (ghat[p] > 0.0) L += g[p] * log(ghat[p]) - ghat[p];
        else if (g[p] > 0.0) L += -INFINITY;
    }
    return L;
}

/* MLEM (Alg. 1) with the early stop Hagen recommends: iteration k evaluates
 * L_k = L(f^(k)) on ghat = H f^(k) (Alg. 1 line 7), then updates f.  After update k >= 2 it stops
 * when L_k - L_{k-1} <= rel_tol * |L_k| (reading R16), or after max_iters updates.
 * ll[k-1] = L_k; returns the number of updates performed in *iters_done. */
int oracle_mlem_monitored(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                          const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                          const double* g, double* f, int64_t max_iters, double rel_tol, double* ll,
                          int64_t* iters_done) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi, m = a * alpha * w;
    double* h = (double*)malloc(sizeof(double) * (size_t)m);
    double* gk = (double*)malloc(sizeof(double) * (size_t)n);
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    double* zeta = (double*)malloc(sizeof(double) * (size_t)m);
    *iters_done = 0;
    if (!h || !gk || !u || !zeta) { rc = OR_ENOMEM; goto done; }
    if ((rc = oracle_sensitivity(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, h))) goto done;
    for (int64_t k = 1; k <= max_iters; ++k) {
        if ((rc = fwd(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, f, gk))) goto done;
        ll[k - 1] = oracle_loglik(n, g, gk);
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t p = 0; p < n; ++p) u[p] = gk[p] > 0.0 ? g[p] / gk[p] : 0.0;
        if ((rc = back(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, u, zeta))) goto done;
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t j = 0; j < m; ++j) f[j] = (f[j] * zeta[j]) / h[j];
        *iters_done = k;
        if (k >= 2 && ll[k - 1] - ll[k - 2] <= rel_tol * fabs(ll[k - 1])) break;
    }
done:
    free(h); free(gk); free(u); free(zeta);
    return rc;
}

/* SMART, the simultaneous (data-parallel) form of the MART solver the paper lists (
 * gordon1970algebraic), on the same projector:
 *   f_j <- f_j * exp( (1/h_j) sum_i H_ij log(g_i / (H f)_i) )
 * with log-ratio r_i = log(g_i / ghat_i) where g_i > 0 and ghat_i > 0, else 0 (R17).
 * Step order as Alg. 1 with the ratio replaced by the log-ratio and the update by the exponential. */
int oracle_smart(int64_t a, int64_t alpha, int64_t w, int64_t gamma, int64_t xi,
                 const int64_t* tap_ptr, const int64_t* tap_offset, const double* tap_weight,
                 const double* g, double* f, int64_t iters) {
    int rc = check_geom(a, alpha, w, gamma, xi);
    if (rc) return rc;
    int64_t n = gamma * xi, m = a * alpha * w;
    double* h = (double*)malloc(sizeof(double) * (size_t)m);
    double* gk = (double*)malloc(sizeof(double) * (size_t)n);
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    double* zeta = (double*)malloc(sizeof(double) * (size_t)m);
    if (!h || !gk || !u || !zeta) { rc = OR_ENOMEM; goto done; }
    if ((rc = oracle_sensitivity(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, h))) goto done;
    for (int64_t k = 0; k < iters; ++k) {
        if ((rc = fwd(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, f, gk))) goto done;
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t p = 0; p < n; ++p) u[p] = (g[p] > 0.0 && gk[p] > 0.0) ? log(g[p] / gk[p]) : 0.0;
        if ((rc = back(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, u, zeta))) goto done;
        #pragma omp parallel for schedule(static) if (g_threads > 1) num_threads(g_threads)
        for (int64_t j = 0; j < m; ++j) f[j] = f[j] * exp(zeta[j] / h[j]);
    }
done:
    free(h); free(gk); free(u); free(zeta);
    return rc;
}

