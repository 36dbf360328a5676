/*
 * kfac_oracle.c -- the plain, slow, obviously-correct fp64 CPU oracle for the
 * distributed K-FAC hot path of Osawa et al., arXiv 1811.12019.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_1811_12019_b200/), and the CUDA path never calls it.
 *
 * Every function is the plain definition written out with explicit loops in
 * fp64 (no blocking, no fusion, no reordering beyond the definition).  Half-
 * precision inputs are the raw 16-bit patterns the GPU consumes, up-cast
 * exactly to fp64.  Citations: P:NNN = PAPER.md line, S:NNN =
 * SPEC.md line (interfaces only).  Readings of the paper are listed in
 * DESIGN.md §Readings (R-n).
 *
 * Threading: OpenMP over independent output rows/columns only; every sum runs
 * in a fixed order, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_EXPORT __attribute__((visibility("default")))

/* ---- half-precision decoding (exact) ---------------------------------- */
/* fmt 0: bfloat16 (1-8-7), fmt 1: IEEE binary16 (1-5-10).                  */
static double dec_half(uint16_t b, int fmt) {
    if (fmt == 0) {
        uint32_t u = ((uint32_t)b) << 16;
        float f;
        memcpy(&f, &u, 4);
        return (double)f;
    }
    int s = (b >> 15) & 1, e = (b >> 10) & 31, m = b & 1023;
    double v;
    if (e == 0) v = ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = ldexp(1.0 + m / 1024.0, e - 15);
    return s ? -v : v;
}

OR_EXPORT double or_decode_half(uint16_t b, int fmt) { return dec_half(b, fmt); }

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

OR_EXPORT int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- im2col patch ("A is computed from the activation"; KFC) ----
 * ã[(i*kw + j)*C + c] = x[n, oh*sh - ph + i, ow*sw - pw + j, c] if in bounds
 * else 0 (zero padding, R-7); ã[dA-1] = 1 when the layer has a bias (R-5).
 * Feature order (kh, kw, c), c fastest (R-6).  x is NHWC.                 */
static double patch_elem(const uint16_t *x, int fmt, int H, int W, int C, int kw,
                         int sh, int sw, int ph, int pw, int n, int oh, int ow, int f) {
    int kk = f / C, c = f % C;
    int i = kk / kw, j = kk % kw;
    int h = oh * sh - ph + i, w = ow * sw - pw + j;
    if (h < 0 || h >= H || w < 0 || w >= W) return 0.0;
    return dec_half(x[(((int64_t)n * H + h) * W + w) * C + c], fmt);
}

/* A = alpha * sum_rows ã ãᵀ, full dA x dA row-major (P:245, P:313-318 stage 1;
 * SPEC compute_a_factor S:197-205).  Rows are (n, oh, ow) in ascending order. */
OR_EXPORT int or_factor_A(int N, int H, int W, int C, int kh, int kw, int sh, int sw,
                          int ph, int pw, int bias, const uint16_t *x, int fmt,
                          double alpha, double *A, int nthreads) {
    if (N < 1) return 1;
    int Ho = (H + 2 * ph - kh) / sh + 1, Wo = (W + 2 * pw - kw) / sw + 1;
    int dF = C * kh * kw, dA = dF + (bias ? 1 : 0);
    memset(A, 0, sizeof(double) * (size_t)dA * dA);
    set_threads(nthreads);
#pragma omp parallel
    {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        T = omp_get_num_threads();
#endif
        double *a = (double *)malloc(sizeof(double) * dA);
        for (int n = 0; n < N; n++)
            for (int oh = 0; oh < Ho; oh++)
                for (int ow = 0; ow < Wo; ow++) {
                    for (int f = 0; f < dF; f++)
                        a[f] = patch_elem(x, fmt, H, W, C, kw, sh, sw, ph, pw, n, oh, ow, f);
                    if (bias) a[dA - 1] = 1.0;
                    /* thread t owns rows i = t, t+T, ... (cyclic: balances the triangle) */
                    for (int i = t; i < dA; i += T) {
                        double ai = a[i];
                        double *Ai = A + (size_t)i * dA;
                        for (int j = i; j < dA; j++) Ai[j] += ai * a[j];
                    }
                }
        free(a);
    }
    for (int i = 0; i < dA; i++)
        for (int j = i; j < dA; j++) {
            A[(size_t)i * dA + j] *= alpha;
            A[(size_t)j * dA + i] = A[(size_t)i * dA + j];
        }
    return 0;
}

/* Selected entries A[i][j] = alpha * sum_rows ã_i ã_j, one by one (for
 * full-size parity checks on sampled outputs). ij holds m (i, j) pairs.    */
OR_EXPORT int or_factor_A_entries(int N, int H, int W, int C, int kh, int kw, int sh, int sw,
                                  int ph, int pw, int bias, const uint16_t *x, int fmt,
                                  double alpha, const int64_t *ij, int64_t m, double *out,
                                  int nthreads) {
    int Ho = (H + 2 * ph - kh) / sh + 1, Wo = (W + 2 * pw - kw) / sw + 1;
    int dF = C * kh * kw;
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < m; q++) {
        int i = (int)ij[2 * q], j = (int)ij[2 * q + 1];
        double s = 0.0;
        for (int n = 0; n < N; n++)
            for (int oh = 0; oh < Ho; oh++)
                for (int ow = 0; ow < Wo; ow++) {
                    double ai = (i < dF) ? patch_elem(x, fmt, H, W, C, kw, sh, sw, ph, pw, n, oh, ow, i)
                                         : (bias ? 1.0 : 0.0);
                    double aj = (j < dF) ? patch_elem(x, fmt, H, W, C, kw, sh, sw, ph, pw, n, oh, ow, j)
                                         : (bias ? 1.0 : 0.0);
                    s += ai * aj;
                }
        out[q] = alpha * s;
    }
    return 0;
}

/* G = alpha * sum_rows g gᵀ over output-gradient pixels g = gy[row, :]
 * ("G is computed from the gradient ... w.r.t. the output"). */
OR_EXPORT int or_factor_G(int64_t rows, int C, const uint16_t *gy, int fmt, double alpha,
                          double *G, int nthreads) {
    if (rows < 1) return 1;
    memset(G, 0, sizeof(double) * (size_t)C * C);
    set_threads(nthreads);
#pragma omp parallel
    {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        T = omp_get_num_threads();
#endif
        double *g = (double *)malloc(sizeof(double) * C);
        for (int64_t r = 0; r < rows; r++) {
            for (int c = 0; c < C; c++) g[c] = dec_half(gy[r * C + c], fmt);
            for (int i = t; i < C; i += T) {
                double gi = g[i];
                double *Gi = G + (size_t)i * C;
                for (int j = i; j < C; j++) Gi[j] += gi * g[j];
            }
        }
        free(g);
    }
    for (int i = 0; i < C; i++)
        for (int j = i; j < C; j++) {
            G[(size_t)i * C + j] *= alpha;
            G[(size_t)j * C + i] = G[(size_t)i * C + j];
        }
    return 0;
}

OR_EXPORT int or_factor_G_entries(int64_t rows, int C, const uint16_t *gy, int fmt, double alpha,
                                  const int64_t *ij, int64_t m, double *out, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < m; q++) {
        int64_t i = ij[2 * q], j = ij[2 * q + 1];
        double s = 0.0;
        for (int64_t r = 0; r < rows; r++) s += dec_half(gy[r * C + i], fmt) * dec_half(gy[r * C + j], fmt);
        out[q] = alpha * s;
    }
    return 0;
}

/* ---- symmetry-aware packing ("only need to send the upper
 * triangular matrix of size N(N+1)/2"); order = upper, row-major (R-10).  */
OR_EXPORT void or_pack_upper(const double *M, int n, double *p) {
    int64_t k = 0;
    for (int i = 0; i < n; i++)
        for (int j = i; j < n; j++) p[k++] = M[(size_t)i * n + j];
}

OR_EXPORT void or_unpack_upper(const double *p, int n, double *M) {
    int64_t k = 0;
    for (int i = 0; i < n; i++)
        for (int j = i; j < n; j++) {
            M[(size_t)i * n + j] = p[k];
            M[(size_t)j * n + i] = p[k];
            k++;
        }
}

/* ---- factored Tikhonov damping (reading R-1) -----
 * pi = sqrt((tr A / dA) / (tr G / dG)), pi = 1 if a trace is 0;
 * A_d = A + pi*sqrt(gamma) I, G_d = G + sqrt(gamma)/pi I (in place).      */
OR_EXPORT int or_damp(double *A, int dA, double *G, int dG, double gamma, double *pi_out) {
    if (!(gamma > 0.0)) return 1;
    double ta = 0.0, tg = 0.0;
    for (int i = 0; i < dA; i++) ta += A[(size_t)i * dA + i];
    for (int i = 0; i < dG; i++) tg += G[(size_t)i * dG + i];
    double pi = 1.0;
    if (ta != 0.0 && tg != 0.0) pi = sqrt((ta / dA) / (tg / dG));
    double sg = sqrt(gamma);
    for (int i = 0; i < dA; i++) A[(size_t)i * dA + i] += pi * sg;
    for (int i = 0; i < dG; i++) G[(size_t)i * dG + i] += sg / pi;
    if (pi_out) *pi_out = pi;
    return 0;
}

/* ---- inverse of a damped factor (P:247-260 Eq. inv_fim, stage 4 P:328;
 * reading R-12: dense Cholesky L Lᵀ, then L⁻¹, then L⁻ᵀ L⁻¹).     */
/* Returns 0, or (pivot index + 1) when M is not positive definite.         */
OR_EXPORT int or_cholesky(const double *M, int n, double *L, int nthreads) {
    memset(L, 0, sizeof(double) * (size_t)n * n);
    set_threads(nthreads);
    for (int j = 0; j < n; j++) {
        double s = M[(size_t)j * n + j];
        for (int k = 0; k < j; k++) s -= L[(size_t)j * n + k] * L[(size_t)j * n + k];
        if (!(s > 0.0)) return j + 1;
        double ljj = sqrt(s);
        L[(size_t)j * n + j] = ljj;
#pragma omp parallel for schedule(static)
        for (int i = j + 1; i < n; i++) {
            double t = M[(size_t)i * n + j];
            for (int k = 0; k < j; k++) t -= L[(size_t)i * n + k] * L[(size_t)j * n + k];
            L[(size_t)i * n + j] = t / ljj;
        }
    }
    return 0;
}

/* Li = L⁻¹ for lower-triangular L, column by column (forward substitution).
 * Column c is built in a contiguous buffer and then stored (a layout choice
 * for the cache only: the arithmetic and its order are the substitution's). */
OR_EXPORT void or_tri_inv_lower(const double *L, int n, double *Li, int nthreads) {
    memset(Li, 0, sizeof(double) * (size_t)n * n);
    set_threads(nthreads);
#pragma omp parallel
    {
        double *col = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 4)
        for (int c = 0; c < n; c++) {
            col[c] = 1.0 / L[(size_t)c * n + c];
            for (int i = c + 1; i < n; i++) {
                double s = 0.0;
                for (int k = c; k < i; k++) s += L[(size_t)i * n + k] * col[k];
                col[i] = -s / L[(size_t)i * n + i];
            }
            for (int i = c; i < n; i++) Li[(size_t)i * n + c] = col[i];
        }
        free(col);
    }
}

OR_EXPORT int or_inverse_spd(const double *M, int n, double *X, int nthreads) {
    double *L = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *Li = (double *)malloc(sizeof(double) * (size_t)n * n);
    int st = or_cholesky(M, n, L, nthreads);
    if (st) {
        free(L);
        free(Li);
        return st;
    }
    or_tri_inv_lower(L, n, Li, nthreads);
    /* X = Liᵀ Li : X[i][j] = sum_{k >= max(i,j)} Li[k][i] Li[k][j].  The
     * columns of Li are read from its transpose T = Liᵀ (T[i][k] = Li[k][i]),
     * a copy for contiguous access; same products, same order.             */
    double *T = L; /* L is no longer needed: reuse it for Liᵀ */
    for (int i = 0; i < n; i++)
        for (int k = 0; k < n; k++) T[(size_t)i * n + k] = Li[(size_t)k * n + i];
#pragma omp parallel for schedule(dynamic, 4)
    for (int i = 0; i < n; i++)
        for (int j = i; j < n; j++) {
            double s = 0.0;
            for (int k = j; k < n; k++) s += T[(size_t)i * n + k] * T[(size_t)j * n + k];
            X[(size_t)i * n + j] = s;
            X[(size_t)j * n + i] = s;
        }
    free(L);
    free(Li);
    return 0;
}

/* ---- preconditioned gradient (P:264-282 Eqs. K-FAC update; reading R-14):
 * 𝒢 = G⁻¹ · ∇W · A⁻¹ with ∇W in R^{dG x dA} row-major (bias column last).  */
OR_EXPORT void or_precondition(const double *Ginv, int dG, const double *Ainv, int dA,
                               const double *dW, double *out, int nthreads) {
    /* Columns of Ainv and of T = ∇W·Ainv are read from transposed copies
     * (AiT[j][k] = Ainv[k][j], TT[j][k] = T[k][j]) for contiguous access;
     * the products and their order are those of the plain triple loops.   */
    double *T = (double *)malloc(sizeof(double) * (size_t)dG * dA);
    double *AiT = (double *)malloc(sizeof(double) * (size_t)dA * dA);
    double *TT = (double *)malloc(sizeof(double) * (size_t)dG * dA);
    set_threads(nthreads);
    for (int k = 0; k < dA; k++)
        for (int j = 0; j < dA; j++) AiT[(size_t)j * dA + k] = Ainv[(size_t)k * dA + j];
#pragma omp parallel for schedule(static)
    for (int i = 0; i < dG; i++)
        for (int j = 0; j < dA; j++) {
            double s = 0.0;
            for (int k = 0; k < dA; k++) s += dW[(size_t)i * dA + k] * AiT[(size_t)j * dA + k];
            T[(size_t)i * dA + j] = s;
        }
    for (int k = 0; k < dG; k++)
        for (int j = 0; j < dA; j++) TT[(size_t)j * dG + k] = T[(size_t)k * dA + j];
#pragma omp parallel for schedule(static)
    for (int i = 0; i < dG; i++)
        for (int j = 0; j < dA; j++) {
            double s = 0.0;
            for (int k = 0; k < dG; k++) s += Ginv[(size_t)i * dG + k] * TT[(size_t)j * dG + k];
            out[(size_t)i * dA + j] = s;
        }
    free(T);
    free(AiT);
    free(TT);
}

/* Selected entries of 𝒢 one by one: out[q] = sum_{k,l} Ginv[i][k] dW[k][l] Ainv[l][j]. */
OR_EXPORT void or_precondition_entries(const double *Ginv, int dG, const double *Ainv, int dA,
                                       const double *dW, const int64_t *ij, int64_t m, double *out,
                                       int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < m; q++) {
        int64_t i = ij[2 * q], j = ij[2 * q + 1];
        double s = 0.0;
        for (int k = 0; k < dG; k++) {
            double t = 0.0;
            for (int l = 0; l < dA; l++) t += dW[(size_t)k * dA + l] * Ainv[(size_t)l * dA + j];
            s += Ginv[(size_t)i * dG + k] * t;
        }
        out[q] = s;
    }
}
