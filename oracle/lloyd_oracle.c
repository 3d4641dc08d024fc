/*
 * lloyd_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of Lloyd's K-means as
 * described in arXiv 2405.12052, written step by step in the
 * paper's order and notation so a reader can check it against the paper by
 * eye.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_2405_12052_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or constant with the CUDA path.
 *
 * Build (see __graft_entry__.build / oracle/build.sh):
 *   gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared \
 *       -o oracle/liblloyd_oracle.so oracle/lloyd_oracle.c -lm
 * -ffp-contract=off: no a*b+c contraction except the explicit fmaf() calls.
 *
 * Numerical contract:
 *   - points are fp32, the fp64 centroid mu^t is rounded once to fp32 (RN)
 *     before distances (R5, R7);
 *   - distance "form D":  e_j = fl32(x_j - c_j);  s = fl32(e_0*e_0);
 *     s = fmaf(e_j, e_j, s) for j = 1..d-1  (R6);
 *   - argmin scans k = 0..K-1 ascending with strict '<' (lowest index wins
 *     ties, R1);
 *   - sums, means, E and inertia are fp64, counts int64 (R5);
 *   - an empty cluster keeps mu^t (R2);
 *   - E is the squared form of PAPER.md:68 (R4); stop when E < tol or at
 *     max_iter (R3).
 *
 * Every function returns 0 on success and a negative code on invalid input
 * (-1 invalid argument, -2 non-finite input).
 *
 * Parity pins for every function live in tests/test_oracle_*.py; none is
 * "parity unpinned".
 */
#include <float.h>
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if !defined(FLT_EVAL_METHOD) || FLT_EVAL_METHOD != 0
#error "the oracle needs FLT_EVAL_METHOD == 0 (no excess float precision)"
#endif

#define ORACLE_EINVAL (-1)
#define ORACLE_ENONFINITE (-2)

/* ---------------------------------------------------------------------
 * Squared L2 distance, form D ("||x_i - mu_k^t||_2^2";
 * the op order is reading R6 of DESIGN.md).
 * x and c each hold d floats.
 * ------------------------------------------------------------------- */
float oracle_dist(const float* x, const float* c, int d)
{
    float e0 = x[0] - c[0];          /* fl32(x_0 - c_0) */
    float s = e0 * e0;               /* fl32(e_0 * e_0), no contraction */
    for (int j = 1; j < d; ++j) {
        float ej = x[j] - c[j];      /* fl32(x_j - c_j) */
        s = fmaf(ej, ej, s);         /* one rounding */
    }
    return s;
}

/* ---------------------------------------------------------------------
 * Reassignment:  z_i^{t+1} = argmin_k ||x_i - mu_k^t||^2.
 * c32 holds the fp32-rounded centroids (K x d).  Lowest k wins ties (R1).
 * Writes the label and the minimal distance.
 * ------------------------------------------------------------------- */
static void nearest(const float* x, const float* c32, int K, int d,
                    int32_t* label, float* dmin)
{
    float best = oracle_dist(x, &c32[0], d);
    int32_t lab = 0;
    for (int k = 1; k < K; ++k) {
        float dk = oracle_dist(x, &c32[(size_t)k * d], d);
        if (dk < best) {
            best = dk;
            lab = k;
        }
    }
    *label = lab;
    *dmin = best;
}

/* E = sum_{i=1}^{K} ||mu_i^{t+1} - mu_i^t||_2^2, in fp64,
 * k-major with j inner, in that order. */
double oracle_shift_error(const double* mu_prev, const double* mu_next, int K, int d)
{
    double E = 0.0;
    for (int k = 0; k < K; ++k) {
        for (int j = 0; j < d; ++j) {
            double diff = mu_next[(size_t)k * d + j] - mu_prev[(size_t)k * d + j];
            E += diff * diff;
        }
    }
    return E;
}

static int all_finite_f(const float* v, int64_t n)
{
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

static int all_finite_d(const double* v, int64_t n)
{
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* ---------------------------------------------------------------------
 * Partial sums of one Lloyd iteration over a contiguous slice of points
 * (the paper's OpenMP "local cluster means" before the merge, PAPER.md:97,
 * kept as sums and counts, never as averaged means -- reading R16).
 *
 *   X        : n x d row-major fp32 points (this slice only)
 *   mu       : K x d fp64 centroids mu^t
 *   labels   : out, n (may be NULL)
 *   dmin     : out, n (may be NULL)
 *   sums     : out, K x d fp64, S_k = sum_{z_i = k} (double) x_i
 *   counts   : out, K int64,  n_k = sum_i 1(z_i = k)
 *   J        : out, sum_i (double) dmin_i   (inertia J(z^{t+1}, mu^t), R10)
 * Points are visited sequentially in i; every sum is accumulated in i order.
 * ------------------------------------------------------------------- */
int oracle_partials(const float* X, int64_t n, int d, int K, const double* mu,
                    int32_t* labels, float* dmin, double* sums, int64_t* counts,
                    double* J)
{
    if (!X || !mu || !sums || !counts || !J || n < 0 || d < 1 || K < 1)
        return ORACLE_EINVAL;
    if (!all_finite_d(mu, (int64_t)K * d)) return ORACLE_ENONFINITE;

    /* Stage: c_k = (float) mu_k^t, round to nearest even (R7). */
    float* c32 = (float*)malloc(sizeof(float) * (size_t)K * d);
    if (!c32) return ORACLE_EINVAL;
    for (int64_t q = 0; q < (int64_t)K * d; ++q) c32[q] = (float)mu[q];

    for (int64_t q = 0; q < (int64_t)K * d; ++q) sums[q] = 0.0;
    for (int k = 0; k < K; ++k) counts[k] = 0;
    double Jacc = 0.0;

    for (int64_t i = 0; i < n; ++i) {
        const float* xi = &X[(size_t)i * d];
        int32_t z;
        float m;
        nearest(xi, c32, K, d, &z, &m);
        if (labels) labels[i] = z;
        if (dmin) dmin[i] = m;
        for (int j = 0; j < d; ++j)                     /* numerator of PAPER.md:52 */
            sums[(size_t)z * d + j] += (double)xi[j];
        counts[z] += 1;                                 /* denominator of PAPER.md:52 */
        Jacc += (double)m;                              /* abstract */
    }
    *J = Jacc;
    free(c32);
    return 0;
}

/* ---------------------------------------------------------------------
 * Mean calculation, PAPER.md:50-62:
 *   mu_k^{t+1} = sum_i 1(z_i = k) x_i / sum_i 1(z_i = k)
 * fp64 IEEE division per coordinate; an empty cluster keeps mu_k^t (R2).
 * Then E.
 * ------------------------------------------------------------------- */
int oracle_update(const double* sums, const int64_t* counts, const double* mu_prev,
                  int K, int d, double* mu_next, double* E)
{
    if (!sums || !counts || !mu_prev || !mu_next || !E || K < 1 || d < 1)
        return ORACLE_EINVAL;
    for (int k = 0; k < K; ++k) {
        for (int j = 0; j < d; ++j) {
            size_t q = (size_t)k * d + j;
            if (counts[k] > 0)
                mu_next[q] = sums[q] / (double)counts[k];
            else
                mu_next[q] = mu_prev[q];
        }
    }
    *E = oracle_shift_error(mu_prev, mu_next, K, d);
    return 0;
}

/* One full Lloyd iteration: steps 2 and 3 of PAPER.md:45-62 plus E. */
int oracle_step(const float* X, int64_t N, int d, int K, const double* mu,
                int32_t* labels, float* dmin, double* sums, int64_t* counts,
                double* J, double* mu_next, double* E)
{
    if (!X || N < 1 || K < 1 || K > N || d < 1) return ORACLE_EINVAL;
    if (!all_finite_f(X, N * (int64_t)d)) return ORACLE_ENONFINITE;
    int rc = oracle_partials(X, N, d, K, mu, labels, dmin, sums, counts, J);
    if (rc) return rc;
    return oracle_update(sums, counts, mu, K, d, mu_next, E);
}

/* ---------------------------------------------------------------------
 * The serial Lloyd loop of PAPER.md:65-70.
 *
 *   X         : N x d row-major fp32 points
 *   init_idx  : K distinct indices in [0, N)  ("randomly selecting K points
 *               from the dataset"; the random choice is made
 *               by the caller, reading R8)
 *   tol       : stop when E < tol (strict; tol = 0 runs max_iter), R3
 *   max_iter  : >= 1
 * Outputs: labels z^{iters} (N), centroids mu^{iters} (K x d), iters,
 * inertia = J of the last iteration, optional E / J traces (max_iter each).
 * ------------------------------------------------------------------- */
int oracle_fit(const float* X, int64_t N, int d, int K, const int64_t* init_idx,
               double tol, int max_iter, int32_t* labels, double* centroids,
               int* iters, double* inertia, double* E_trace, double* J_trace)
{
    /* Step 1 of the validation in SURVEY.md §8(c). */
    if (!X || !init_idx || !labels || !centroids || !iters || !inertia)
        return ORACLE_EINVAL;
    if (N < 1 || d < 1 || K < 1 || K > N || max_iter < 1 || !(tol >= 0.0))
        return ORACLE_EINVAL;
    for (int k = 0; k < K; ++k) {
        if (init_idx[k] < 0 || init_idx[k] >= N) return ORACLE_EINVAL;
        for (int q = 0; q < k; ++q)
            if (init_idx[q] == init_idx[k]) return ORACLE_EINVAL;
    }
    if (!all_finite_f(X, N * (int64_t)d)) return ORACLE_ENONFINITE;

    size_t Kd = (size_t)K * d;
    double* mu = (double*)malloc(sizeof(double) * Kd);
    double* mu_next = (double*)malloc(sizeof(double) * Kd);
    double* sums = (double*)malloc(sizeof(double) * Kd);
    int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)K);
    if (!mu || !mu_next || !sums || !counts) {
        free(mu); free(mu_next); free(sums); free(counts);
        return ORACLE_EINVAL;
    }

    /* Initialisation: mu_k^0 = x_{init_idx[k]}. */
    for (int k = 0; k < K; ++k)
        for (int j = 0; j < d; ++j)
            mu[(size_t)k * d + j] = (double)X[(size_t)init_idx[k] * d + j];

    int t = 0;
    double J = 0.0, E = 0.0;
    for (;;) {
        /* Steps 2 and 3, then E. */
        oracle_partials(X, N, d, K, mu, labels, NULL, sums, counts, &J);
        oracle_update(sums, counts, mu, K, d, mu_next, &E);
        if (E_trace) E_trace[t] = E;
        if (J_trace) J_trace[t] = J;
        memcpy(mu, mu_next, sizeof(double) * Kd);
        t += 1;
        /* "compared with a tolerance ... inside the loop" */
        if (E < tol || t == max_iter) break;
    }
    memcpy(centroids, mu, sizeof(double) * Kd);
    *iters = t;
    *inertia = J;
    free(mu); free(mu_next); free(sums); free(counts);
    return 0;
}
