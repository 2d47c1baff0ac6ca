/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * implementation of what the hot path computes.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code, header or constant with the
 * CUDA path (paper_1809_09175_b200/csrc) and never includes it.
 *
 * Citations: P:NNN = /root/reference/PAPER.md line, S:NNN = SPEC.md line.
 * Compiled with -O2 -ffp-contract=off (no fused multiply-add) so each
 * floating-point step is exactly the one written here.
 *
 * Functions and what pins them (tests/test_oracle.py):
 *   oracle_perm          stable counting sort        -> SPEC examples, invariants,
 *                                                       numpy stable argsort
 *   oracle_mttkrp        Eq. (2) loop                -> dense brute force,
 *                                                       planted closed form, special cases
 *   oracle_mttkrp_rows   Eq. (2) on a row subset     -> equality with oracle_mttkrp
 *   oracle_mttkrp_omp    row-owned OpenMP timing form-> bit-identical to oracle_mttkrp
 *   oracle_cp_als        textbook CP-ALS (Kolda-Bader), readings in DESIGN.md §2
 *                                                    -> planted recovery, rank-1,
 *                                                       monotone residual, dense fit
 *   oracle_gram / oracle_chol_solve / oracle_normalize -> SPEC examples S:162
 *   oracle_merge_duplicates  merge-sum     -> SPEC example S:56, dense
 *                                                       equality (np.add.at), first-occurrence order
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_EZERONORM (-2)
#define OR_ESINGULAR (-3)
#define OR_ENOMEM (-4)

/* ------------------------------------------------------------------------ */
/* Permutation ("a permutation array for each mode that sorts the
 * tensor nonzeros in increasing index along that mode"; stable per P:584 and
 * S:82).  Counting sort: histogram of keys, exclusive scan, left-to-right
 * scatter.  rowptr (optional, In+1 entries) is the exclusive scan. */
int oracle_perm(int64_t P, int N, const uint32_t *idx, int n, int64_t In,
                uint32_t *perm, uint32_t *rowptr)
{
    if (P < 0 || N < 1 || n < 0 || n >= N || In < 1) return OR_EINVAL;
    uint64_t *count = (uint64_t *)calloc((size_t)In + 1, sizeof(uint64_t));
    if (!count) return OR_ENOMEM;
    for (int64_t i = 0; i < P; ++i) {
        uint32_t k = idx[(size_t)i * N + n];
        if ((int64_t)k >= In) { free(count); return OR_EINVAL; }
        count[k + 1] += 1;
    }
    for (int64_t k = 0; k < In; ++k) count[k + 1] += count[k]; /* count[k] = start of row k */
    if (rowptr)
        for (int64_t k = 0; k <= In; ++k) rowptr[k] = (uint32_t)count[k];
    for (int64_t i = 0; i < P; ++i) {
        uint32_t k = idx[(size_t)i * N + n];
        perm[count[k]++] = (uint32_t)i;
    }
    free(count);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* MTTKRP, Eq. (2):
 *   v(k,j) = lambda_j * sum_{i : l_in = k} x_i * prod_{m != n} a^(m)(l_im, j)
 * Visits nonzeros in storage order; the product is taken over modes in
 * increasing order; lambda (NULL = all ones) is applied once per entry at the
 * end (algebraically equal to the per-nonzero factor in Eq. (2); DESIGN.md
 * reading Z1).  acc_long != 0 accumulates in long double (reading Z17). */
int oracle_mttkrp(int N, const int64_t *dims, int64_t P, const uint32_t *idx,
                  const double *vals, int64_t R, const double *const *A, int n,
                  const double *lambda, int acc_long, double *V)
{
    if (N < 1 || n < 0 || n >= N || R < 1 || P < 0) return OR_EINVAL;
    const int64_t In = dims[n];
    if (acc_long) {
        long double *acc = (long double *)calloc((size_t)(In * R), sizeof(long double));
        if (!acc) return OR_ENOMEM;
        for (int64_t i = 0; i < P; ++i) {
            const uint32_t *c = idx + (size_t)i * N;
            const int64_t k = c[n];
            for (int64_t j = 0; j < R; ++j) {
                double t = vals[i];
                for (int m = 0; m < N; ++m)
                    if (m != n) t *= A[m][(size_t)c[m] * R + j];
                acc[k * R + j] += (long double)t;
            }
        }
        for (int64_t k = 0; k < In; ++k)
            for (int64_t j = 0; j < R; ++j) {
                double v = (double)acc[k * R + j];
                V[k * R + j] = lambda ? v * lambda[j] : v;
            }
        free(acc);
        return OR_OK;
    }
    memset(V, 0, sizeof(double) * (size_t)(In * R));
    for (int64_t i = 0; i < P; ++i) {
        const uint32_t *c = idx + (size_t)i * N;
        const int64_t k = c[n];
        for (int64_t j = 0; j < R; ++j) {
            double t = vals[i];
            for (int m = 0; m < N; ++m)
                if (m != n) t *= A[m][(size_t)c[m] * R + j];
            V[k * R + j] += t;
        }
    }
    if (lambda)
        for (int64_t k = 0; k < In; ++k)
            for (int64_t j = 0; j < R; ++j) V[k * R + j] *= lambda[j];
    return OR_OK;
}

/* Eq. (2) restricted to the rows listed in `rows` (distinct, each < dims[n]);
 * Vrows is nrows x R.  One pass over all nonzeros in storage order, so every
 * entry equals the corresponding entry of oracle_mttkrp bit for bit. */
int oracle_mttkrp_rows(int N, const int64_t *dims, int64_t P, const uint32_t *idx,
                       const double *vals, int64_t R, const double *const *A, int n,
                       const double *lambda, int acc_long, int64_t nrows,
                       const int64_t *rows, double *Vrows)
{
    if (N < 1 || n < 0 || n >= N || R < 1 || P < 0 || nrows < 0) return OR_EINVAL;
    const int64_t In = dims[n];
    int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * (size_t)In);
    long double *acc = (long double *)calloc((size_t)(nrows * R) + 1, sizeof(long double));
    double *accd = (double *)calloc((size_t)(nrows * R) + 1, sizeof(double));
    if (!slot || !acc || !accd) { free(slot); free(acc); free(accd); return OR_ENOMEM; }
    for (int64_t k = 0; k < In; ++k) slot[k] = -1;
    for (int64_t s = 0; s < nrows; ++s) {
        if (rows[s] < 0 || rows[s] >= In) { free(slot); free(acc); free(accd); return OR_EINVAL; }
        slot[rows[s]] = s;
    }
    for (int64_t i = 0; i < P; ++i) {
        const uint32_t *c = idx + (size_t)i * N;
        const int64_t s = slot[c[n]];
        if (s < 0) continue;
        for (int64_t j = 0; j < R; ++j) {
            double t = vals[i];
            for (int m = 0; m < N; ++m)
                if (m != n) t *= A[m][(size_t)c[m] * R + j];
            if (acc_long) acc[s * R + j] += (long double)t;
            else accd[s * R + j] += t;
        }
    }
    for (int64_t s = 0; s < nrows; ++s)
        for (int64_t j = 0; j < R; ++j) {
            double v = acc_long ? (double)acc[s * R + j] : accd[s * R + j];
            Vrows[s * R + j] = lambda ? v * lambda[j] : v;
        }
    free(slot); free(acc); free(accd);
    return OR_OK;
}

/* Timing form used as the CPU baseline: the oracle's own
 * stable counting sort, then OpenMP over output rows ("row-owned", no
 * atomics).  Each row sums its nonzeros in storage order, so the result is
 * bit-identical to oracle_mttkrp(acc_long = 0).  Returns threads used via
 * *threads_used. */
int oracle_mttkrp_omp(int N, const int64_t *dims, int64_t P, const uint32_t *idx,
                      const double *vals, int64_t R, const double *const *A, int n,
                      const double *lambda, const uint32_t *perm, const uint32_t *rowptr,
                      double *V, int *threads_used)
{
    if (N < 1 || n < 0 || n >= N || R < 1 || P < 0) return OR_EINVAL;
    const int64_t In = dims[n];
    int nt = 1;
#pragma omp parallel
    {
#ifdef _OPENMP
#pragma omp single
        nt = omp_get_num_threads();
#endif
#pragma omp for schedule(dynamic, 64)
        for (int64_t k = 0; k < In; ++k) {
            double *v = V + k * R;
            for (int64_t j = 0; j < R; ++j) v[j] = 0.0;
            for (uint32_t q = rowptr[k]; q < rowptr[k + 1]; ++q) {
                const uint32_t i = perm[q];
                const uint32_t *c = idx + (size_t)i * N;
                for (int64_t j = 0; j < R; ++j) {
                    double t = vals[i];
                    for (int m = 0; m < N; ++m)
                        if (m != n) t *= A[m][(size_t)c[m] * R + j];
                    v[j] += t;
                }
            }
            if (lambda)
                for (int64_t j = 0; j < R; ++j) v[j] *= lambda[j];
        }
    }
    if (threads_used) *threads_used = nt;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* CP-ALS pieces.  The paper omits the algorithm ("Details are omitted here",
 * P:124-127) and defers to Kolda & Bader; these are the textbook steps, with
 * each choice recorded in DESIGN.md §2 (readings Z11, Z12). */

/* G = A^T A  (I x R row-major -> R x R). */
void oracle_gram(int64_t I, int64_t R, const double *A, double *G)
{
    for (int64_t a = 0; a < R; ++a)
        for (int64_t b = 0; b < R; ++b) {
            double s = 0.0;
            for (int64_t k = 0; k < I; ++k) s += A[k * R + a] * A[k * R + b];
            G[a * R + b] = s;
        }
}

/* Cholesky G = L L^T in place (lower triangle of L returned in Lout).
 * Pivot j fails unless d_j > tau * G_jj (DESIGN.md §2 reading Z23: a relative
 * pivot below 1e-12 is a numerically singular G; tau = 0 is the plain
 * positive-definiteness test). */
static int chol(int64_t R, const double *G, double *L, double tau)
{
    memset(L, 0, sizeof(double) * (size_t)(R * R));
    for (int64_t j = 0; j < R; ++j) {
        double d = G[j * R + j];
        for (int64_t k = 0; k < j; ++k) d -= L[j * R + k] * L[j * R + k];
        if (!(d > tau * G[j * R + j])) return OR_ESINGULAR;
        const double ljj = sqrt(d);
        L[j * R + j] = ljj;
        for (int64_t i = j + 1; i < R; ++i) {
            double s = G[i * R + j];
            for (int64_t k = 0; k < j; ++k) s -= L[i * R + k] * L[j * R + k];
            L[i * R + j] = s / ljj;
        }
    }
    return OR_OK;
}

/* Solve (L L^T) x = b for one right-hand side (forward then back substitution). */
static void chol_apply(int64_t R, const double *L, const double *b, double *x)
{
    for (int64_t i = 0; i < R; ++i) {
        double s = b[i];
        for (int64_t k = 0; k < i; ++k) s -= L[i * R + k] * x[k];
        x[i] = s / L[i * R + i];
    }
    for (int64_t i = R - 1; i >= 0; --i) {
        double s = x[i];
        for (int64_t k = i + 1; k < R; ++k) s -= L[k * R + i] * x[k];
        x[i] = s / L[i * R + i];
    }
}

/* Cholesky factorisation of an SPD matrix with one ridge retry
 * (G + 1e-12 * (tr G / R) * I) when a pivot fails the relative test
 * (DESIGN.md §2 Z23; the retry tests d_j > 0), then row-wise solves
 * X = B G^{-1} for nrhs rows of B (nrhs x R).  S:347. */
int oracle_chol_solve(int64_t R, const double *G, int64_t nrhs, const double *B, double *X)
{
    double *L = (double *)malloc(sizeof(double) * (size_t)(R * R));
    double *Gr = (double *)malloc(sizeof(double) * (size_t)(R * R));
    if (!L || !Gr) { free(L); free(Gr); return OR_ENOMEM; }
    int st = chol(R, G, L, 1e-12);
    if (st != OR_OK) {
        double tr = 0.0;
        for (int64_t j = 0; j < R; ++j) tr += G[j * R + j];
        memcpy(Gr, G, sizeof(double) * (size_t)(R * R));
        for (int64_t j = 0; j < R; ++j) Gr[j * R + j] += 1e-12 * (tr / (double)R);
        st = chol(R, Gr, L, 0.0);
    }
    if (st == OR_OK)
        for (int64_t k = 0; k < nrhs; ++k) chol_apply(R, L, B + k * R, X + k * R);
    free(L); free(Gr);
    return st;
}

/* Column normalisation to unit 2-norm ("unit-norm in some norm";
 * 2-norm per S:200).  lambda_j = ||A(:,j)||_2; a zero column becomes e_1
 * with lambda_j = 0. */
void oracle_normalize(int64_t I, int64_t R, double *A, double *lambda)
{
    for (int64_t j = 0; j < R; ++j) {
        double s = 0.0;
        for (int64_t k = 0; k < I; ++k) s += A[k * R + j] * A[k * R + j];
        const double nrm = sqrt(s);
        lambda[j] = nrm;
        if (nrm == 0.0) {
            for (int64_t k = 0; k < I; ++k) A[k * R + j] = (k == 0) ? 1.0 : 0.0;
        } else {
            for (int64_t k = 0; k < I; ++k) A[k * R + j] /= nrm;
        }
    }
}

/* Textbook CP-ALS (Kolda & Bader, cited at P:97-98):
 *   for it = 1..max_iters, for n = 0..N-1:
 *     V = MTTKRP(X, A, n) (lambda = 1);  Gamma = Hadamard_{m != n} A_m^T A_m
 *     A_n = V Gamma^{-1} (Cholesky, ridge retry);  lambda = column 2-norms;
 *     normalise A_n
 *   fit = 1 - ||X - M|| / ||X||, ||X - M||^2 = max(0, ||X||^2 + ||M||^2 - 2<X,M>)
 *   with <X,M> = sum_j lambda_j sum_k A_{N-1}(k,j) V(k,j) (last mode's V)
 *   and ||M||^2 = lambda^T (Hadamard_m A_m^T A_m) lambda.
 *   Stops when tol > 0 and |fit - fit_prev| < tol; tol = 0 runs all iterations
 *   (the paper's fixed 10).
 * A[m] holds the initial factors on entry and the result on exit. */
int oracle_cp_als(int N, const int64_t *dims, int64_t P, const uint32_t *idx,
                  const double *vals, int64_t R, int max_iters, double tol,
                  double *const *A, double *lambda, double *fit_out, int *iters_out,
                  double *fit_trace)
{
    if (N < 2 || R < 1 || max_iters < 0 || P < 0) return OR_EINVAL;
    double normX2 = 0.0;
    for (int64_t i = 0; i < P; ++i) normX2 += vals[i] * vals[i];
    if (!(normX2 > 0.0)) return OR_EZERONORM;

    int64_t Imax = 0;
    for (int m = 0; m < N; ++m) if (dims[m] > Imax) Imax = dims[m];
    double *V = (double *)malloc(sizeof(double) * (size_t)(Imax * R));
    double *G = (double *)malloc(sizeof(double) * (size_t)(N * R * R));
    double *Gam = (double *)malloc(sizeof(double) * (size_t)(R * R));
    if (!V || !G || !Gam) { free(V); free(G); free(Gam); return OR_ENOMEM; }

    for (int64_t j = 0; j < R; ++j) lambda[j] = 1.0;
    for (int m = 0; m < N; ++m) oracle_gram(dims[m], R, A[m], G + (size_t)m * R * R);

    double fit = 0.0, fit_prev = 0.0;
    int it = 0, st = OR_OK;
    for (it = 0; it < max_iters; ++it) {
        for (int n = 0; n < N; ++n) {
            st = oracle_mttkrp(N, dims, P, idx, vals, R, (const double *const *)A, n,
                               NULL, 0, V);
            if (st) goto done;
            for (int64_t e = 0; e < R * R; ++e) {
                double h = 1.0;
                for (int m = 0; m < N; ++m)
                    if (m != n) h *= G[(size_t)m * R * R + e];
                Gam[e] = h;
            }
            st = oracle_chol_solve(R, Gam, dims[n], V, A[n]);
            if (st) goto done;
            oracle_normalize(dims[n], R, A[n], lambda);
            oracle_gram(dims[n], R, A[n], G + (size_t)n * R * R);
        }
        /* fit, using the last mode's V (A[N-1] now normalised). */
        const int n = N - 1;
        double inner = 0.0;
        for (int64_t j = 0; j < R; ++j) {
            double s = 0.0;
            for (int64_t k = 0; k < dims[n]; ++k) s += A[n][k * R + j] * V[k * R + j];
            inner += lambda[j] * s;
        }
        double normM2 = 0.0;
        for (int64_t a = 0; a < R; ++a)
            for (int64_t b = 0; b < R; ++b) {
                double h = 1.0;
                for (int m = 0; m < N; ++m) h *= G[(size_t)m * R * R + a * R + b];
                normM2 += lambda[a] * h * lambda[b];
            }
        double res2 = normX2 + normM2 - 2.0 * inner;
        if (res2 < 0.0) res2 = 0.0;
        fit = 1.0 - sqrt(res2) / sqrt(normX2);
        if (fit_trace) fit_trace[it] = fit;
        if (tol > 0.0 && fabs(fit - fit_prev) < tol) { ++it; break; }
        fit_prev = fit;
    }
done:
    if (fit_out) *fit_out = fit;
    if (iters_out) *iters_out = it;
    free(V); free(G); free(Gam);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Duplicate merge (SPEC from_coo merge-sum): equal coordinates are
 * combined into one nonzero whose value is the sum of the run's values in
 * storage order, kept at the position of the first occurrence; the output
 * keeps the storage order of first occurrences.  qsort of (coordinates,
 * position) pairs, then one pass.  Returns the new nnz via *Pout. */
static int g_merge_N;
static const uint32_t *g_merge_idx;

static int merge_cmp(const void *pa, const void *pb)
{
    const int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    for (int m = 0; m < g_merge_N; ++m) {
        const uint32_t x = g_merge_idx[(size_t)a * g_merge_N + m];
        const uint32_t y = g_merge_idx[(size_t)b * g_merge_N + m];
        if (x != y) return x < y ? -1 : 1;
    }
    return a < b ? -1 : (a > b ? 1 : 0);
}

int oracle_merge_duplicates(int64_t P, int N, const uint32_t *idx, const double *vals,
                            uint32_t *idx_out, double *vals_out, int64_t *Pout)
{
    if (P < 0 || N < 1) return OR_EINVAL;
    int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
    char *keep = (char *)calloc((size_t)(P > 0 ? P : 1), 1);
    double *sum = (double *)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
    if (!ord || !keep || !sum) { free(ord); free(keep); free(sum); return OR_ENOMEM; }
    for (int64_t i = 0; i < P; ++i) ord[i] = i;
    g_merge_N = N;
    g_merge_idx = idx;
    qsort(ord, (size_t)P, sizeof(int64_t), merge_cmp);
    for (int64_t i = 0; i < P;) {
        int64_t j = i + 1;
        double s = vals[ord[i]];
        while (j < P && memcmp(idx + (size_t)ord[j] * N, idx + (size_t)ord[i] * N,
                               sizeof(uint32_t) * (size_t)N) == 0) {
            s += vals[ord[j]];
            ++j;
        }
        keep[ord[i]] = 1;
        sum[ord[i]] = s;
        i = j;
    }
    int64_t q = 0;
    for (int64_t i = 0; i < P; ++i) {
        if (!keep[i]) continue;
        memcpy(idx_out + (size_t)q * N, idx + (size_t)i * N, sizeof(uint32_t) * (size_t)N);
        vals_out[q] = sum[i];
        ++q;
    }
    *Pout = q;
    free(ord); free(keep); free(sum);
    return OR_OK;
}
