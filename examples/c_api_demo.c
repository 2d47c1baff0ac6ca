/* c_api_demo.c -- the C ABI (include/sptk.h) used from plain C: no Python,
 * no torch.  A random 3-way tensor is created from HOST buffers, the
 * permutations are built, one MTTKRP per mode runs on device factors (CUDA
 * runtime for the buffers) and is checked against Eq. (2) computed here, and
 * 10 CP-ALS iterations run with host factor buffers.
 * Build (see tests/test_gpu.py::test_c_api_demo):
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_demo.c \
 *       -L paper_1809_09175_b200 -lsptk -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,<repo>/paper_1809_09175_b200 -lm -o examples/c_api_demo */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "sptk.h"

static uint64_t s_rng = 88172645463325252ull;
static double urand(void) {
    s_rng ^= s_rng << 13;
    s_rng ^= s_rng >> 7;
    s_rng ^= s_rng << 17;
    return (double)(s_rng >> 11) * 0x1.0p-53;
}

#define CHECK(x)                                                                        \
    do {                                                                                \
        sptk_status _s = (x);                                                           \
        if (_s != SPTK_OK) {                                                            \
            fprintf(stderr, "%s failed: %d %s\n", #x, (int)_s, sptk_last_error());     \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

int main(void) {
    enum { N = 3 };
    const int64_t dims[N] = {200, 150, 100}, P = 20000, R = 16;
    int64_t *idx = malloc(sizeof(int64_t) * P * N);
    double *vals = malloc(sizeof(double) * P);
    for (int64_t i = 0; i < P; ++i) {
        for (int m = 0; m < N; ++m) idx[i * N + m] = (int64_t)(urand() * dims[m]);
        vals[i] = 1.0 - urand();
    }
    double *A[N];
    void *dA[N];
    for (int m = 0; m < N; ++m) {
        A[m] = malloc(sizeof(double) * dims[m] * R);
        for (int64_t e = 0; e < dims[m] * R; ++e) A[m][e] = urand();
        if (cudaMalloc(&dA[m], sizeof(double) * dims[m] * R) != cudaSuccess) return 2;
        cudaMemcpy(dA[m], A[m], sizeof(double) * dims[m] * R, cudaMemcpyHostToDevice);
    }

    sptk_tensor t;
    CHECK(sptk_sptensor_create(N, dims, P, idx, SPTK_IDX_I64, vals, SPTK_F64, 0, NULL, &t));
    CHECK(sptk_build_perm(t, -1, NULL));

    double worst = 0.0;
    for (int n = 0; n < N; ++n) {
        void *dV;
        double *V = malloc(sizeof(double) * dims[n] * R);
        double *ref = calloc((size_t)(dims[n] * R), sizeof(double));
        cudaMalloc(&dV, sizeof(double) * dims[n] * R);
        CHECK(sptk_mttkrp(t, n, R, (const void *const *)dA, NULL, dV, NULL, NULL));
        cudaMemcpy(V, dV, sizeof(double) * dims[n] * R, cudaMemcpyDeviceToHost);
        for (int64_t i = 0; i < P; ++i)          /* Eq. (2), storage order */
            for (int64_t j = 0; j < R; ++j) {
                double p = vals[i];
                for (int m = 0; m < N; ++m)
                    if (m != n) p *= A[m][idx[i * N + m] * R + j];
                ref[idx[i * N + n] * R + j] += p;
            }
        double num = 0.0, den = 0.0;
        for (int64_t e = 0; e < dims[n] * R; ++e) {
            num += (V[e] - ref[e]) * (V[e] - ref[e]);
            den += ref[e] * ref[e];
        }
        const double rel = sqrt(num / den);
        if (rel > worst) worst = rel;
        cudaFree(dV);
        free(V);
        free(ref);
    }
    printf("mttkrp: worst relative Frobenius error over modes %.3e\n", worst);
    if (!(worst <= 1e-12)) return 1;

    double *F[N], lam[16], fit = 0.0, trace[10];
    int iters = 0;
    for (int m = 0; m < N; ++m) F[m] = malloc(sizeof(double) * dims[m] * R);
    const void *init[N] = {A[0], A[1], A[2]};
    void *outp[N] = {F[0], F[1], F[2]};
    CHECK(sptk_cp_als(t, R, 10, 0.0, 1, init, outp, lam, &fit, &iters, trace, NULL, NULL));
    for (int m = 0; m < N; ++m)                  /* unit 2-norm columns */
        for (int j = 0; j < R; ++j) {
            double s = 0.0;
            for (int64_t k = 0; k < dims[m]; ++k) s += F[m][k * R + j] * F[m][k * R + j];
            if (fabs(s - 1.0) > 1e-10) return 1;
        }
    printf("cp_als: %d iterations, fit %.6f\n", iters, fit);
    CHECK(sptk_sptensor_destroy(t));
    printf("c_api_demo ok (%s)\n", sptk_version());
    return 0;
}
