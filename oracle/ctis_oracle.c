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
    rc = oracle_backproject(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, ones, h);
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
        if ((rc = oracle_forward(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, f, gk))) goto done;
        for (int64_t p = 0; p < n; ++p) u[p] = gk[p] > 0.0 ? g[p] / gk[p] : 0.0;
        if ((rc = oracle_backproject(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, u, zeta))) goto done;
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
        if ((rc = oracle_forward(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, f, gk))) goto done;
        ll[k - 1] = oracle_loglik(n, g, gk);
        for (int64_t p = 0; p < n; ++p) u[p] = gk[p] > 0.0 ? g[p] / gk[p] : 0.0;
        if ((rc = oracle_backproject(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, u, zeta))) goto done;
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
        if ((rc = oracle_forward(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, f, gk))) goto done;
        for (int64_t p = 0; p < n; ++p) u[p] = (g[p] > 0.0 && gk[p] > 0.0) ? log(g[p] / gk[p]) : 0.0;
        if ((rc = oracle_backproject(a, alpha, w, gamma, xi, tap_ptr, tap_offset, tap_weight, u, zeta))) goto done;
        for (int64_t j = 0; j < m; ++j) f[j] = f[j] * exp(zeta[j] / h[j]);
    }
done:
    free(h); free(gk); free(u); free(zeta);
    return rc;
}

