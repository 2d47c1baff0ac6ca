// als.cu -- CP-ALS glue and the sptk_cp_als driver.
// The paper omits the algorithm ("Details are omitted here") and
// defers to Kolda & Bader; these are the textbook steps (DESIGN.md §2
// readings Z11, Z12):
//   per mode n:  V = MTTKRP(X, A, n)          (mttkrp.cuh, lambda = NULL)
//                Gamma = Hadamard_{m!=n} G_m  (G_m = A_m^T A_m, cached)
//                Gamma^{-1} by unpivoted Gauss-Jordan (one block; ridge retry;
//                the Cholesky L^{-T} L^{-1} kernel with SPTK_GAMMA_INV=chol)
//                A_n = V Gamma^{-1}           (row-parallel product, fused with the
//                                              column sums of squares for lambda)
//                lambda_j = ||A_n(:,j)||_2, normalise (zero column -> e_1)
//                G_n = A_n^T A_n
//   per iteration: fit = 1 - sqrt(max(0, ||X||^2 + ||M||^2 - 2<X,M>)) / ||X||
//                <X,M> = sum_j lambda_j sum_k A_{N-1}(k,j) V(k,j)
//                ||M||^2 = lambda^T (Hadamard_m G_m) lambda
// All glue reductions are fixed-order (per-block partials, then a fixed
// shuffle tree); the MTTKRP's boundary-row atomics are not, so runs agree to
// rounding, not bit for bit.  One small D2H (fit, status) per iteration.  The oracle solves with the Cholesky factor row by row; using
// the explicit inverse differs only at rounding level.
// Multi-GPU: each rank solves its own row range of every mode, the R column
// sums of squares and <X,M> partials are all-reduced, the rows broadcast.
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "common.cuh"

namespace sptk {

constexpr int kMaxAlsRank = 128;
constexpr int kGramTileRows = 128;  // rows staged per shared-memory tile (R <= 32 kernels)

// ---------------------------------------------------------------- kernels
// Counter generator of DESIGN.md §3 (same text as synth/), for init = NULL.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Entry (row, col) of an I x Rl factor takes counter row*Rl + col; it is
// stored at row*ld + col (ld > Rl: padded rank, pad columns written 0).
template <typename T>
__global__ void init_factor_kernel(uint64_t seed, uint64_t stream, int64_t I, int Rl, int ld,
                                   T *__restrict__ out) {
    const int64_t n = I * ld;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / ld;
        const int col = (int)(i - row * ld);
        if (col >= Rl) {
            out[i] = T(0);
            continue;
        }
        const uint64_t k = (uint64_t)(row * Rl + col);
        const uint64_t d = splitmix64(seed ^ (k * 0x9E3779B97F4A7C15ull) ^
                                      (stream * 0xD1B54A32D192ED03ull));
        out[i] = (T)((double)(d >> 11) * 0x1.0p-53);
    }
}

// partial[b][e] = sum over the rows of block b of A(k,a) A(k,c), e = a*R + c;
// KE = Gram entries per thread per pass (1 for R <= 16, 4 for R <= 32)
template <typename T, int KE>
__global__ void __launch_bounds__(256)
    gram_partial_kernel(const T *__restrict__ A, int64_t I, int R, int64_t rows_per_block,
                        double *__restrict__ partial) {
    constexpr int TR = kGramTileRows;  // rows staged per tile
    extern __shared__ double tile[];  // TR x R
    const int RR = R * R;
    const int64_t r0 = blockIdx.x * rows_per_block;
    const int64_t r1 = min(I, r0 + rows_per_block);
    for (int e0 = 0; e0 < RR; e0 += 256 * KE) {
        double acc[KE];
#pragma unroll
        for (int k = 0; k < KE; ++k) acc[k] = 0.0;
        for (int64_t rt = r0; rt < r1; rt += TR) {
            const int nr = (int)min((int64_t)TR, r1 - rt);
            __syncthreads();
#pragma unroll 4
            for (int x = threadIdx.x; x < nr * R; x += blockDim.x)
                tile[x] = (double)A[rt * R + x];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < KE; ++k) {
                const int e = e0 + k * 256 + threadIdx.x;
                if (e < RR) {
                    const int a = e / R, c = e % R;
                    double s = acc[k];
                    for (int r = 0; r < nr; ++r) s += tile[r * R + a] * tile[r * R + c];
                    acc[k] = s;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < KE; ++k) {
            const int e = e0 + k * 256 + threadIdx.x;
            if (e < RR) partial[(int64_t)blockIdx.x * RR + e] = acc[k];
        }
    }
}

// out[e] = sum_b partial[b][e]: one warp per entry, lanes stride over the
// blocks, fixed-order shuffle tree (deterministic).
__global__ void __launch_bounds__(256)
    reduce_partials_kernel(const double *__restrict__ partial, int nb, int ne,
                           double *__restrict__ out) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < ne;
         e += (gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int b = lane; b < nb; b += 32) s += partial[(int64_t)b * ne + e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[e] = s;
    }
}

// Pivot test of the first factorisation attempt (DESIGN.md §2 reading Z23, as
// the oracle): pivot j counts as a failure unless d_j > kPivotRel * Gamma_jj.
// d_j / Gamma_jj is the squared sine of the angle between column j and the
// span of the columns before it; below 1e-12 Gamma is numerically singular
// (duplicate CP components: cond ~ 1e300 on LBNL after 5 iterations) and its
// inverse amplifies rounding without bound, so the ridge retry takes over.
// The retry keeps the plain d_j > 0 test.
constexpr double kPivotRel = 1e-12;

// Gamma = Hadamard_{m != n} G_m; Cholesky Gamma = L L^T (one ridge retry with
// 1e-12 tr(Gamma)/R, as the oracle); Gamma^{-1} = L^{-T} L^{-1} -> Ginv.
// One block.  Shared memory: R x R (L in the lower triangle, L^{-1}
// transposed in the strict upper triangle) + R (diagonal of L^{-1}).
__global__ void __launch_bounds__(256)
    chol_inv_kernel(const double *__restrict__ G, int N, int n, int R, int Rl,
                    double *__restrict__ Ginv, int *__restrict__ status) {
    extern __shared__ double sm[];
    double *L = sm;             // R x R
    double *dinv = sm + R * R;  // R
    __shared__ int bad;
    __shared__ double ridge;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto gamma = [&](int i, int j) {  // padded rank (i or j >= Rl): identity block
        if (i >= Rl || j >= Rl) return i == j ? 1.0 : 0.0;
        double h = 1.0;
        for (int m = 0; m < N; ++m)
            if (m != n) h *= G[(int64_t)m * R * R + i * R + j];
        return h;
    };
    if (tid == 0) {
        ridge = 0.0;
        bad = 0;
    }
    __syncthreads();
    for (int attempt = 0; attempt < 2; ++attempt) {
        const double tau = attempt == 0 ? kPivotRel : 0.0;
        for (int e = tid; e < R * R; e += blockDim.x) {
            const int i = e / R, j = e % R;
            if (j <= i) L[e] = gamma(i, j) + (i == j && i < Rl ? ridge : 0.0);
        }
        __syncthreads();
        if (warp == 0) {  // left-looking in-place Cholesky by one warp
            for (int j = 0; j < R; ++j) {
                double d = 0.0;
                for (int k = lane; k < j; k += 32) d += L[j * R + k] * L[j * R + k];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                const double gjj = L[j * R + j];
                d = gjj - d;
                if (!(d > tau * gjj)) {
                    if (lane == 0) bad = 1;
                    d = 1.0;
                }
                const double ljj = sqrt(d);
                __syncwarp();
                if (lane == 0) L[j * R + j] = ljj;
                for (int i = j + 1 + lane; i < R; i += 32) {
                    double s2 = L[i * R + j];
                    for (int k = 0; k < j; ++k) s2 -= L[i * R + k] * L[j * R + k];
                    L[i * R + j] = s2 / ljj;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        const int failed = bad;
        __syncthreads();
        if (!failed) break;
        if (attempt == 0) {
            if (tid == 0) {
                double tr = 0.0;
                for (int j = 0; j < Rl; ++j) tr += gamma(j, j);
                ridge = 1e-12 * (tr / (double)Rl);
                bad = 0;
            }
            __syncthreads();
        } else if (tid == 0) {
            atomicOr(status, 1);
        }
    }
    // column j of L^{-1} (thread j): z_j = 1/L_jj, z_i = -sum_{k=j}^{i-1} L_ik z_k / L_ii;
    // z_i (i > j) stored at L[j][i] (strict upper triangle), z_j in dinv[j].
    for (int j = tid; j < R; j += blockDim.x) {
        const double zj = 1.0 / L[j * R + j];
        dinv[j] = zj;
        for (int i = j + 1; i < R; ++i) {
            double s2 = L[i * R + j] * zj;
            for (int k = j + 1; k < i; ++k) s2 += L[i * R + k] * L[j * R + k];
            L[j * R + i] = -s2 / L[i * R + i];
        }
    }
    __syncthreads();
    // Ginv[a][b] = sum_{k >= max(a,b)} Linv[k][a] Linv[k][b]
    for (int e = tid; e < R * R; e += blockDim.x) {
        const int a = e / R, b = e % R;
        const int k0 = a > b ? a : b;
        double s2 = 0.0;
        for (int k = k0; k < R; ++k) {
            const double la = (k == a) ? dinv[a] : L[a * R + k];
            const double lb = (k == b) ? dinv[b] : L[b * R + k];
            s2 += la * lb;
        }
        Ginv[e] = s2;
    }
}


// Gamma^{-1} by in-place Gauss-Jordan in shared memory, all threads per step
// (R steps x 3 barriers) -- the Cholesky above has a long dependent chain on
// one warp and sits on the critical path when the MTTKRP is short.  Without
// pivoting, the pivots of an SPD matrix are the squared Cholesky diagonal, so
// a non-positive pivot is exactly the Cholesky failure: same ridge retry.
// (block function: M = R x R and f = R doubles of shared memory; every thread
// of the block calls it; Ginv may be global or shared)
// Padded rank (R > Rl: columns Rl..R-1 of every factor are zero, DESIGN.md
// §4 "odd R"): Gamma's pad block is the identity, so Gamma^{-1} is
// diag(Gamma_Rl^{-1}, I) and the pad columns of V Gamma^{-1} stay zero.
__device__ void gj_inv_block(const double *G, int N, int n, int R, int Rl,
                             double *__restrict__ Ginv, int *__restrict__ status,
                             double *__restrict__ M, double *__restrict__ f) {
    __shared__ double piv;
    __shared__ int bad;
    const int tid = threadIdx.x, RR = R * R;
    for (int attempt = 0; attempt < 2; ++attempt) {
        double ridge = 0.0;
        if (attempt) {
            double tr = 0.0;  // every thread: trace of Gamma (Rl products, tiny)
            for (int j = 0; j < Rl; ++j) {
                double h = 1.0;
                for (int m = 0; m < N; ++m)
                    if (m != n) h *= G[(int64_t)m * RR + j * R + j];
                tr += h;
            }
            ridge = 1e-12 * (tr / (double)Rl);
        }
        for (int e = tid; e < RR; e += blockDim.x) {
            const int i = e / R, k = e % R;
            double h = 1.0;
            if (i >= Rl || k >= Rl) {
                h = i == k ? 1.0 : 0.0;
            } else {
                for (int m = 0; m < N; ++m)
                    if (m != n) h *= G[(int64_t)m * RR + e];
                if (i == k) h += ridge;
            }
            M[e] = h;
        }
        if (tid == 0) bad = 0;
        __syncthreads();
        for (int j = 0; j < R; ++j) {
            if (tid == 0) {
                double p = M[j * R + j];
                double gjj = 0.0;  // relative pivot test (first attempt): Gamma_jj
                if (!attempt) {
                    gjj = 1.0;
                    if (j < Rl)
                        for (int m = 0; m < N; ++m)
                            if (m != n) gjj *= G[(int64_t)m * RR + j * R + j];
                }
                if (!(p > kPivotRel * gjj)) bad = 1;
                if (!(p > 0.0)) p = 1.0;
                piv = 1.0 / p;
            }
            for (int i = tid; i < R; i += blockDim.x) f[i] = M[i * R + j];
            __syncthreads();
            const double rp = piv;
            for (int k = tid; k < R; k += blockDim.x)
                M[j * R + k] = (k == j ? 1.0 : M[j * R + k]) * rp;
            __syncthreads();
            for (int e = tid; e < RR; e += blockDim.x) {
                const int i = e / R, k = e % R;
                if (i != j) M[e] = (k == j ? 0.0 : M[e]) - f[i] * M[j * R + k];
            }
            __syncthreads();
        }
        const int failed = bad;
        __syncthreads();
        if (!failed) break;
        if (attempt == 1 && tid == 0) atomicOr(status, 1);
    }
    for (int e = tid; e < RR; e += blockDim.x) Ginv[e] = M[e];
    __syncthreads();
}

__global__ void __launch_bounds__(256)
    gj_inv_kernel(const double *__restrict__ G, int N, int n, int R, int Rl,
                  double *__restrict__ Ginv, int *__restrict__ status) {
    extern __shared__ double sm[];
    gj_inv_block(G, N, n, R, Rl, Ginv, status, sm, sm + R * R);
}

// The same unpivoted Gauss-Jordan (same ridge retry, padded-rank identity
// block) by ONE warp for R <= 32: lane i holds row i of Gamma in registers;
// each pivot step broadcasts the pivot row by shuffles and updates every row
// in parallel -- no block barriers, one FP64 division per step per lane.  The
// 256-thread kernel above spends 3 block barriers and a serial thread-0
// division per step: 10-16 us for R = 16 in the LBNL timeline
// (profiles/r02/s2/timeline_lbnl.log), longer than a short MTTKRP.
template <int LR>
__global__ void __launch_bounds__(32)
    gj_inv_warp_kernel(const double *__restrict__ G, int N, int n, int R, int Rl,
                       double *__restrict__ Ginv, int *__restrict__ status) {
    const int i = threadIdx.x;  // row
    const int RR = R * R;
    double m[LR];
    for (int attempt = 0; attempt < 2; ++attempt) {
        double ridge = 0.0;
        if (attempt) {  // 1e-12 tr(Gamma_Rl) / Rl, as the oracle
            double d = 1.0;
            if (i < Rl) {
                for (int q = 0; q < N; ++q)
                    if (q != n) d *= G[(int64_t)q * RR + i * R + i];
            } else {
                d = 0.0;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            ridge = 1e-12 * (d / (double)Rl);
        }
        // Gamma row i: the loads of every mode issued together (unrolled over
        // kMaxModes), then the Hadamard products
#pragma unroll
        for (int k = 0; k < LR; ++k) m[k] = 1.0;
#pragma unroll
        for (int q = 0; q < kMaxModes; ++q) {
            if (q >= N || q == n) continue;
            double gq[LR];
#pragma unroll
            for (int k = 0; k < LR; ++k)
                gq[k] = (i < Rl && k < Rl) ? __ldcg(G + (int64_t)q * RR + i * R + k) : 1.0;
#pragma unroll
            for (int k = 0; k < LR; ++k) m[k] *= gq[k];
        }
#pragma unroll
        for (int k = 0; k < LR; ++k) {
            if (i >= R || k >= R) m[k] = 0.0;
            else if (i >= Rl || k >= Rl) m[k] = i == k ? 1.0 : 0.0;
            else if (i == k) m[k] += ridge;
        }
        double dii = 0.0;  // Gamma_ii (relative pivot test, first attempt only)
#pragma unroll
        for (int k = 0; k < LR; ++k)
            if (k == i && !attempt) dii = m[k];
        bool bad = false;
#pragma unroll
        for (int j = 0; j < LR; ++j) {  // unrolled: m[] stays in registers
            if (j >= R) break;
            const double p = __shfl_sync(0xffffffffu, m[j], j);
            bad |= !(p > kPivotRel * __shfl_sync(0xffffffffu, dii, j));
            const double rp = 1.0 / (p > 0.0 ? p : 1.0);
            const double f = m[j];  // this row's multiplier (row j: the pivot itself)
#pragma unroll
            for (int k = 0; k < LR; ++k) {
                const double rk = __shfl_sync(0xffffffffu, m[k], j) * rp;  // new pivot row
                const double rkj = (k == j) ? rp : rk;
                m[k] = (i == j) ? rkj : ((k == j) ? 0.0 : m[k]) - f * rkj;
            }
        }
        if (!bad) break;
        if (attempt == 1 && i == 0) atomicOr(status, 1);
    }
    if (i < R)
#pragma unroll
        for (int k = 0; k < LR; ++k)
            if (k < R) Ginv[i * R + k] = m[k];
}

// Gamma^{-1} for mode n (SPTK_GAMMA_INV=chol forces the Cholesky kernel);
// R = the padded rank (row stride), Rl <= R the rank of the decomposition
static void launch_ginv(const double *G, int N, int n, int R, int Rl, double *Ginv, int *status,
                        cudaStream_t s) {
    if (opt(OPT_GAMMA_INV_CHOL))
        chol_inv_kernel<<<1, 256, sizeof(double) * (R * R + R), s>>>(G, N, n, R, Rl, Ginv, status);
    else if (opt(OPT_GJ_WARP) && R <= 8)
        gj_inv_warp_kernel<8><<<1, 32, 0, s>>>(G, N, n, R, Rl, Ginv, status);
    else if (opt(OPT_GJ_WARP) && R <= 16)
        gj_inv_warp_kernel<16><<<1, 32, 0, s>>>(G, N, n, R, Rl, Ginv, status);
    else if (opt(OPT_GJ_WARP) && R <= 32)
        gj_inv_warp_kernel<32><<<1, 32, 0, s>>>(G, N, n, R, Rl, Ginv, status);
    else
        gj_inv_kernel<<<1, 256, sizeof(double) * (R * R + R), s>>>(G, N, n, R, Rl, Ginv, status);
}

// A_raw(k,:) = V(k,:) Gamma^{-1} for rows [r0, r1); per-block partial column
// sums of squares of A_raw (-> lambda) and, for the fit, of A_raw(k,j) V(k,j).
// Thread t: column j = t % R, row lane t / R (R <= 256).
template <typename T>
__global__ void __launch_bounds__(256)
    apply_inv_kernel(const T *__restrict__ V, int64_t r0, int64_t r1, int R,
                     int64_t rows_per_block, const double *__restrict__ Ginv, T *__restrict__ A,
                     double *__restrict__ part_sq, double *__restrict__ part_dot) {
    extern __shared__ double sm[];
    double *Gi = sm;           // R x R
    double *red = sm + R * R;  // 2 x 256
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gi[e] = Ginv[e];
    __syncthreads();
    const int lanes = 256 / R;
    const int j = threadIdx.x % R, l = threadIdx.x / R;
    const int64_t b0 = r0 + blockIdx.x * rows_per_block;
    const int64_t b1 = min(r1, b0 + rows_per_block);
    const bool vec4 = (R % 4 == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0);
    double sq = 0.0, dot = 0.0;
    if (l < lanes) {
#pragma unroll 2
        for (int64_t k = b0 + l; k < b1; k += lanes) {
            const T *v = V + k * R;
            double x = 0.0;
            if (vec4) {  // 4 values per load: one LDG per 4 columns of the row
                for (int i = 0; i < R; i += 4) {
                    T q[4];
                    if constexpr (sizeof(T) == 8) {
                        const double2 a0 = __ldg(reinterpret_cast<const double2 *>(v + i));
                        const double2 a1 = __ldg(reinterpret_cast<const double2 *>(v + i + 2));
                        q[0] = a0.x; q[1] = a0.y; q[2] = a1.x; q[3] = a1.y;
                    } else {
                        const float4 a0 = __ldg(reinterpret_cast<const float4 *>(v + i));
                        q[0] = a0.x; q[1] = a0.y; q[2] = a0.z; q[3] = a0.w;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) x += (double)q[u] * Gi[(i + u) * R + j];
                }
            } else {
                for (int i = 0; i < R; ++i) x += (double)v[i] * Gi[i * R + j];
            }
            const T xt = (T)x;
            A[k * R + j] = xt;
            sq += (double)xt * (double)xt;
            dot += (double)xt * (double)v[j];
        }
    }
    red[threadIdx.x] = sq;
    red[256 + threadIdx.x] = dot;
    __syncthreads();
    if (threadIdx.x < R) {
        double a = 0.0, d = 0.0;
        for (int q = 0; q < lanes; ++q) {
            a += red[q * R + threadIdx.x];
            d += red[256 + q * R + threadIdx.x];
        }
        part_sq[(int64_t)blockIdx.x * R + threadIdx.x] = a;
        if (part_dot) part_dot[(int64_t)blockIdx.x * R + threadIdx.x] = d;
    }
}

// lambda_j = ||A_raw(:,j)||_2 from colsq; A(:,j) /= lambda_j; a zero column
// becomes e_1 with lambda_j = 0.  Block 0 also writes lambda.
// Pad columns (j >= Rl, padded rank) stay zero with lambda_j = 0.
template <typename T>
__global__ void normalize_kernel(T *__restrict__ A, int64_t r0, int64_t r1, int R, int Rl,
                                 const double *__restrict__ colsq, double *__restrict__ lam) {
    if (blockIdx.x == 0)
        for (int j = threadIdx.x; j < R; j += blockDim.x) lam[j] = sqrt(colsq[j]);
    const int64_t n = (r1 - r0) * R;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = r0 + i / R;
        const int j = (int)(i % R);
        const double l = sqrt(colsq[j]);
        T *a = A + k * R + j;
        if (j >= Rl) *a = T(0);
        else if (l == 0.0) *a = (T)(k == 0 ? 1.0 : 0.0);
        else *a = (T)((double)*a / l);
    }
}

// fit from dot_j = sum_k A_raw(k,j) V(k,j) (= lambda_j sum_k A(k,j) V(k,j)),
// lambda and the Gram matrices -> out[0] = fit, out[1] = <X,M>, out[2] = ||M||^2.
// Called by all 256 threads of one block.
// trace (nullable): the fit is also appended at trace[(*trace_n)++] (device-side
// fit history, so iterations can be replayed back to back without a host sync)
__device__ void fit_block(const double *dot, const double *lam,
                          const double *G, int N, int R, double normX2,
                          double *__restrict__ out, double *__restrict__ trace = nullptr,
                          int *__restrict__ trace_n = nullptr) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int a = e / R, b = e % R;
        double h = 1.0;
        for (int m = 0; m < N; ++m) h *= G[(int64_t)m * R * R + e];
        acc += lam[a] * h * lam[b];
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double normM2 = sh[0];
        double inner = 0.0;
        for (int j = 0; j < R; ++j) inner += dot[j];
        double res2 = normX2 + normM2 - 2.0 * inner;
        if (res2 < 0.0) res2 = 0.0;
        out[0] = 1.0 - sqrt(res2) / sqrt(normX2);
        out[1] = inner;
        out[2] = normM2;
        if (trace) trace[(*trace_n)++] = out[0];
    }
}

__global__ void __launch_bounds__(256)
    fit_kernel(const double *__restrict__ dot, const double *__restrict__ lam,
               const double *__restrict__ G, int N, int R, double normX2,
               double *__restrict__ out, double *__restrict__ trace = nullptr,
               int *__restrict__ trace_n = nullptr) {
    pdl_wait();
    fit_block(dot, lam, G, N, R, normX2, out, trace, trace_n);
}

// Tail of a mode update (single GPU), one grid: every block
//   (a) takes lambda_j = sqrt(colsq_j) (colsq reduced once beforehand),
//   (b) normalises its row chunk of A_n (zero column -> e_1),
//   (c) writes the partial Gram matrix of its normalised rows (reduced in block
//       order by reduce_partials_kernel); block 0 writes lambda.
template <typename T, int KE>
__global__ void __launch_bounds__(256)
    finish_kernel(T *__restrict__ A, int64_t I, int R, int Rl, int64_t rows_per_block,
                  const double *__restrict__ colsq, double *__restrict__ gpart,
                  double *__restrict__ lam) {
    constexpr int TR = kGramTileRows;
    extern __shared__ double sm[];
    double *lam_s = sm;     // R
    double *tile = sm + R;  // TR x R
    const int tid = threadIdx.x;
    const int RR = R * R;
    for (int j = tid; j < R; j += blockDim.x) lam_s[j] = sqrt(colsq[j]);
    __syncthreads();
    if (blockIdx.x == 0)
        for (int j = tid; j < R; j += blockDim.x) lam[j] = lam_s[j];
    const int64_t r0 = blockIdx.x * rows_per_block;
    const int64_t r1 = min(I, r0 + rows_per_block);
    for (int e0 = 0; e0 < RR; e0 += 256 * KE) {
        double acc[KE];
#pragma unroll
        for (int k = 0; k < KE; ++k) acc[k] = 0.0;
        for (int64_t rt = r0; rt < r1; rt += TR) {
            const int nr = (int)min((int64_t)TR, r1 - rt);
            __syncthreads();
#pragma unroll 4
            for (int x = tid; x < nr * R; x += blockDim.x) {
                T *a = A + rt * R + x;
                T v = *a;
                if (e0 == 0) {  // normalise once (first entry chunk); later chunks re-read
                    const double l = lam_s[x % R];
                    if (x % R >= Rl) v = T(0);  // pad column (padded rank)
                    else v = (l == 0.0) ? (T)(rt + x / R == 0 ? 1.0 : 0.0) : (T)((double)v / l);
                    *a = v;
                }
                tile[x] = (double)v;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < KE; ++k) {
                const int e = e0 + k * 256 + tid;
                if (e < RR) {
                    const int a = e / R, b = e % R;
                    double s = acc[k];
                    for (int r = 0; r < nr; ++r) s += tile[r * R + a] * tile[r * R + b];
                    acc[k] = s;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < KE; ++k) {
            const int e = e0 + k * 256 + tid;
            if (e < RR) gpart[(int64_t)blockIdx.x * RR + e] = acc[k];
        }
    }
}


// ------------------------------------------------- fused glue, R <= 32 (single GPU)
// Deferred normalisation: A_n is kept as A_raw = V Gamma^{-1}; its column
// scales s_n = 1/lambda_n are applied where the normalised factor is consumed
// -- the next MTTKRPs take prod_{m != n} s_m as their column weights (applied
// at the row flush, Eq. (2)'s lambda), the Gram matrix is D_s G_raw D_s -- and
// once to every factor after the last iteration.  The tail of a mode update is
// then one pass over V (A_raw, its Gram partials, the column partials) plus an
// R x R finalisation, instead of apply + normalise + Gram (two passes over A).
constexpr int kApplyTileDefault = 64;
// V elements per thread per tile of apply_gram<T, RM> (its register prefetch)
#ifndef SPTK_APPLY_PF_DIV  // A/B builds only
#define SPTK_APPLY_PF_DIV 4
#endif
__host__ __device__ constexpr int apply_pf(int RM) { return RM / SPTK_APPLY_PF_DIV; }
#ifndef SPTK_TAIL_BLOCKS  // A/B builds only
#define SPTK_TAIL_BLOCKS 32
#endif
constexpr int kTailBlocks = SPTK_TAIL_BLOCKS;  // apply_gram grids up to this size finalise in their last block
static int apply_tile_rows() {  // option apply_tile (rows of V per tile, tuning)
    const int64_t v = opt(OPT_APPLY_TILE);
    return v >= 16 ? (int)v : kApplyTileDefault;
}

// option apply_nb_mult: apply_gram block cap = mult x 8 x SMs (tuning)
static int apply_nb_mult() {
    const int64_t v = opt(OPT_APPLY_NB_MULT);
    return v > 0 ? (int)v : 1;
}

static int64_t tail_rows() {  // option tail_rows (tuning); 0 = grid by tile only
    return opt(OPT_TAIL_ROWS);
}

static bool deferred_norm(int64_t R) {  // read per call: tests switch it per case
    return opt(OPT_DEFERRED_NORM) != 0 && R <= 32;
}

// Rows [b0, b1) of the block: V tile -> shared memory (coalesced), A_raw tile =
// V_tile Ginv (thread (j, l): column j, rows l, l + 256/R, ...), written to A
// and to shared memory; Gram partials of the tile in 2 x 2 register blocks
// (256 / ceil(R/2)^2 row groups); per-block partials: psq/pdot [blk][R],
// gpart [blk][R*R].
// One block.  lambda_n = sqrt(colsq); s_n = 1/lambda_n; the normalised Gram
// G_n = D_s G_raw D_s.  A zero column j (lambda_j = 0) becomes e_1 as in the
// oracle: A_raw(0, j) := 1 with s_j = 1, and its Gram entries are
// e_1 . A_norm(:, b) = A_raw(0, b) s_b (1 against another zero column).  Then
// the column scale of the next mode's MTTKRP: prod_{m != next} s_m.
template <typename T>
__device__ void finalize_mode_block(const double *__restrict__ colsq,
                                    const double *__restrict__ graw, T *__restrict__ A, int N,
                                    int n, int R, int Rl, int next, double *__restrict__ s_all,
                                    double *__restrict__ lam, double *__restrict__ G,
                                    T *__restrict__ scale_next) {
    __shared__ double sn[128];
    __shared__ double row0[128];
    __shared__ int zero[128];
    const int tid = threadIdx.x;
    for (int j = tid; j < R; j += blockDim.x) {
        // pad column of a padded rank (j >= Rl): zero, lambda 0, scale 0 --
        // its Gram entries and the next MTTKRP's weight stay 0
        const bool pad = j >= Rl;
        const double l = pad ? 0.0 : sqrt(colsq[j]);
        lam[j] = l;
        zero[j] = !pad && !(l > 0.0);
        sn[j] = pad ? 0.0 : (l > 0.0 ? 1.0 / l : 1.0);
        row0[j] = (double)A[j];
    }
    __syncthreads();
    double *Gn = G + (int64_t)n * R * R;
    for (int e = tid; e < R * R; e += blockDim.x) {
        const int a = e / R, b = e % R;
        double g;
        if (!zero[a] && !zero[b]) g = graw[e] * sn[a] * sn[b];
        else if (zero[a] && zero[b]) g = 1.0;
        else if (zero[a]) g = row0[b] * sn[b];
        else g = row0[a] * sn[a];
        Gn[e] = g;
    }
    for (int j = tid; j < R; j += blockDim.x) {
        if (zero[j]) A[j] = (T)1.0;
        s_all[(int64_t)n * R + j] = sn[j];
    }
    __syncthreads();
    for (int j = tid; j < R; j += blockDim.x) {
        double p = 1.0;
        for (int m = 0; m < N; ++m)
            if (m != next) p *= (m == n) ? sn[j] : s_all[(int64_t)m * R + j];
        scale_next[j] = (T)p;
    }
    __syncthreads();
}

template <typename T>
__global__ void __launch_bounds__(256)
    finalize_mode_kernel(const double *__restrict__ colsq, const double *__restrict__ graw,
                         T *__restrict__ A, int N, int n, int R, int Rl, int next,
                         double *__restrict__ s_all, double *__restrict__ lam,
                         double *__restrict__ G, T *__restrict__ scale_next) {
    pdl_wait();
    finalize_mode_block<T>(colsq, graw, A, N, n, R, Rl, next, s_all, lam, G, scale_next);
}

// A large mode's tail in one launch: block g reduces four consecutive
// entries of one of [colsq | graw | dot] over the nb apply blocks' partials,
// then the last block to arrive finalises the mode (and, after the last mode,
// the fit).  Replaces 3 (5) dependent launches: reduce colsq, reduce graw,
// finalise (reduce dot, fit).
// Reduction layout: lane (s, q) = (lane >> 2, lane & 3) of warp w reads entry
// k0 + q of blocks b = 8w + s + 64i -- four adjacent entries of a block's
// partial row are one 32-byte sector, so every sector fetched is used (the
// previous one-warp-per-entry layout read a sector per element: 4x the L2
// traffic at R = 16, 15 us for LBNL's 1184 partial rows); four accumulators
// per thread, then a fixed shuffle tree over s and a fixed sum over the 8
// warps: deterministic.
constexpr int kRedQ = 4;  // entries per reduction block
__host__ __device__ inline int reduce_groups(int R, bool dot) {
    const int gs = (R + kRedQ - 1) / kRedQ;
    return gs + (R * R + kRedQ - 1) / kRedQ + (dot ? gs : 0);
}
template <typename T>
__global__ void __launch_bounds__(256)
    reduce_finalize_kernel(const double *__restrict__ psq, const double *__restrict__ gpart,
                           const double *__restrict__ pdot, int nb, int R, int Rl,
                           double *__restrict__ colsq, double *__restrict__ graw, T *__restrict__ A,
                           int N, int n, int next, double *__restrict__ s_all,
                           double *__restrict__ lam, double *__restrict__ G,
                           T *__restrict__ scale_next, int *__restrict__ counter, double normX2,
                           double *__restrict__ fit, double *__restrict__ trace,
                           int *__restrict__ trace_n) {
    pdl_wait();
    __shared__ double wsum[8][kRedQ];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int RR = R * R, gs = (R + kRedQ - 1) / kRedQ, gg = (RR + kRedQ - 1) / kRedQ;
    int g = blockIdx.x;
    const double *part;
    int stride;
    double *dst;
    if (g < gs) {
        part = psq, stride = R, dst = colsq;
    } else if ((g -= gs) < gg) {
        part = gpart, stride = RR, dst = graw;
    } else {
        g -= gg;
        part = pdot, stride = R, dst = colsq + R;
    }
    const int k = g * kRedQ + (lane & 3);
    const bool on = k < stride;  // stride = the array's entry count
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
    if (on) {
        const double *p = part + k;
        int b = 8 * w + (lane >> 2);
        for (; b + 192 < nb; b += 256) {
            x0 += p[(int64_t)b * stride];
            x1 += p[(int64_t)(b + 64) * stride];
            x2 += p[(int64_t)(b + 128) * stride];
            x3 += p[(int64_t)(b + 192) * stride];
        }
        for (; b < nb; b += 64) x0 += p[(int64_t)b * stride];
    }
    double x = (x0 + x1) + (x2 + x3);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane < kRedQ) wsum[w][lane] = x;
    __syncthreads();
    if (threadIdx.x < kRedQ && g * kRedQ + (int)threadIdx.x < stride) {
        double t = 0.0;
#pragma unroll
        for (int v = 0; v < 8; ++v) t += wsum[v][threadIdx.x];
        dst[g * kRedQ + threadIdx.x] = t;
    }
    __shared__ int last_block;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last_block = atomicAdd(counter, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last_block) return;
    __threadfence();
    finalize_mode_block<T>(colsq, graw, A, N, n, R, Rl, next, s_all, lam, G, scale_next);
    if (pdot) fit_block(colsq + R, lam, G, N, R, normX2, fit, trace, trace_n);
    if (threadIdx.x == 0) *counter = 0;  // ready for the next launch (graph replays)
}

// Where the last block of apply_gram leaves the mode's results (counter NULL:
// the partials are reduced by separate kernels instead).
struct ModeTail {
    int *counter;          // zero-initialised; reset by the last block
    double *colsq;         // [0,R) sum A_raw^2, [R,2R) sum A_raw V (last mode)
    double *graw;          // R x R
    double *s_all, *lam, *G, *fit;
    double *trace;         // device fit history (see fit_block)
    int *trace_n;
    void *scale_next;      // R values of the tensor dtype
    double normX2;
    int N, n, next;
    int Rl;                // rank of the decomposition (< R: padded rank)
};

// Where apply_gram also stores the rows it computes (sharded CP-ALS with the
// fused exchange): every rank's replica of A_n by NVLink peer
// stores (np > 0), or one NVLS multicast store that reaches every rank (mc).
struct ExchOut {
    int np = 0;
    char *peer[kMaxPeers] = {};  // A_n on rank p (byte address in this process)
    char *mc = nullptr;          // multicast address of A_n
    // option zero_in_apply: the last zb blocks of the launch only zero the
    // next mode's MTTKRP output (zw 16-byte words at zp) and exit
    int zb = 0;
    int64_t zw = 0;
    uint4 *zp = nullptr;
};

// The zeroing blocks of an apply launch (ExchOut::zb > 0): blocks
// [gridDim.x - zb, gridDim.x) store zeros over the next mode's output buffer
// (a buffer of its own) and return; the rest of the kernel
// sees nb = gridDim.x - zb blocks.  True for a zeroing block.
__device__ __forceinline__ bool apply_zero_blocks(const ExchOut &ex) {
    if (!ex.zb) return false;
    const int z = (int)blockIdx.x - ((int)gridDim.x - ex.zb);
    if (z < 0) return false;
    const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = (int64_t)z * blockDim.x + threadIdx.x; i < ex.zw;
         i += (int64_t)ex.zb * blockDim.x)
        ex.zp[i] = zero;
    return true;
}

__device__ __forceinline__ void mm_store(double *p, double v) {
    asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void mm_store(float *p, float v) {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// The tail of a mode update in the LAST block of an apply kernel to finish
// (tail.counter != NULL): reduce every block's partials in block order (eight
// interleaved sums combined in a fixed order: deterministic), finalise the
// mode (lambda, scales, normalised Gram, the next MTTKRP's weights) and, after
// the last mode, the fit.  Called by every thread of every block.
template <typename T>
__device__ void apply_tail(const ModeTail &tail, T *__restrict__ A, int R,
                           const double *part_sq, const double *part_dot, const double *gpart,
                           int zb = 0) {
    if (!tail.counter) return;
    const int tid = threadIdx.x;
    const int nb = (int)gridDim.x - zb, RR = R * R;  // apply blocks (zeroing blocks excluded)
    __shared__ int last_block;
    __threadfence();
    __syncthreads();
    if (tid == 0) last_block = atomicAdd(tail.counter, 1) == nb - 1;
    __syncthreads();
    if (!last_block) return;
    __threadfence();
    auto sum_parts = [&](const double *part, int stride, int e) {
        double acc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = 0.0;
        int b = 0;
        for (; b + 7 < nb; b += 8) {  // 8 independent loads in flight per thread
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldcg(part + (int64_t)(b + k) * stride + e);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] += v[k];
        }
        for (; b < nb; ++b) acc[0] += __ldcg(part + (int64_t)b * stride + e);
        return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    };
    for (int e = tid; e < R; e += blockDim.x) {
        tail.colsq[e] = sum_parts(part_sq, R, e);
        if (part_dot) tail.colsq[R + e] = sum_parts(part_dot, R, e);
    }
    for (int e = tid; e < RR; e += blockDim.x) tail.graw[e] = sum_parts(gpart, RR, e);
    __threadfence_block();
    __syncthreads();
    finalize_mode_block<T>(tail.colsq, tail.graw, A, tail.N, tail.n, R, tail.Rl, tail.next,
                           tail.s_all,
                           tail.lam, tail.G, static_cast<T *>(tail.scale_next));
    if (part_dot)
        fit_block(tail.colsq + R, tail.lam, tail.G, tail.N, R, tail.normX2, tail.fit, tail.trace,
                  tail.trace_n);
    if (tid == 0) *tail.counter = 0;  // ready for the next launch (graph replays)
}

#ifndef SPTK_APPLY_MINB  // A/B builds only
#define SPTK_APPLY_MINB 2
#endif
template <typename T, int RM>  // RM >= R: Gamma^{-1} column length held in registers
__global__ void __launch_bounds__(256, SPTK_APPLY_MINB)
    apply_gram_kernel(const T *__restrict__ V, int64_t r_begin, int64_t I, int R,
                      int64_t rows_per_block, int kApplyTile,
                      const double *__restrict__ Ginv, T *__restrict__ A,
                      double *__restrict__ part_sq, double *__restrict__ part_dot,
                      double *__restrict__ gpart, const ModeTail tail, const ExchOut ex) {
    pdl_wait();
    if (apply_zero_blocks(ex)) return;
    extern __shared__ __align__(16) double sm[];
    const int RP = (R + 3) & ~3;              // padded row stride (whole 4-column blocks)
    double *Vt = sm;                          // kApplyTile x RP
    double *At = Vt + kApplyTile * RP;        // kApplyTile x RP
    double *red = At + kApplyTile * RP;       // 4 x 256
    const int tid = threadIdx.x;
    const int lanes = 256 / R, j = tid % R, l = tid / R;
    double gi[RM];  // column j of Gamma^{-1}
#pragma unroll
    for (int i = 0; i < RM; ++i) gi[i] = (i < R && l < lanes) ? Ginv[i * R + j] : 0.0;
    // Gram partials in 4 x 4 register blocks of the upper triangle (4 shared
    // loads per 16 FMAs; mirrored on output); the group count is what the
    // V/A tiles can hold when they are reused to stage the partials
    const int hb = RP / 4, nblk = hb * (hb + 1) / 2;
    const int groups = max(1, min(256 / nblk, (2 * kApplyTile * RP) / (nblk * 16)));
    const int bi = tid % nblk, grp = tid / nblk;
    auto block_of = [hb](int b, int &a0, int &c0) {
        int ba = 0;
        while (b >= hb - ba) b -= hb - ba, ++ba;
        a0 = 4 * ba, c0 = 4 * (ba + b);
    };
    int a0, c0;
    block_of(bi, a0, c0);
    double g[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) g[q] = 0.0;
    double sq = 0.0, dot = 0.0;
    const int64_t b0 = r_begin + (int64_t)blockIdx.x * rows_per_block;  // rows [r_begin, I)
    const int64_t b1 = min(I, b0 + rows_per_block);
    // the next tile of V is loaded into registers while this one is computed
    // (kApplyTile * R <= kApplyPf * 256, clamped by the host): without it each
    // block waits for its 8 KB tile, and a tall mode's pass is latency-bound
    constexpr int kApplyPf = apply_pf(RM);
    T pf[kApplyPf];
    auto fetch = [&](int64_t rt) {
        const int n = (int)(min((int64_t)kApplyTile, b1 - rt) * R);
#pragma unroll
        for (int k = 0; k < kApplyPf; ++k) {
            const int x = tid + k * 256;
            pf[k] = x < n ? V[rt * R + x] : T(0);
        }
    };
    if (b0 < b1) fetch(b0);
    for (int64_t rt = b0; rt < b1; rt += kApplyTile) {
        const int nr = (int)min((int64_t)kApplyTile, b1 - rt);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kApplyPf; ++k) {
            const int x = tid + k * 256;
            if (x < nr * R) {
                const int r = x / R, c = x - r * R;
                Vt[r * RP + c] = (double)pf[k];
            }
        }
        if (rt + kApplyTile < b1) fetch(rt + kApplyTile);
        if (RP != R)
            for (int x = tid; x < nr * (RP - R); x += blockDim.x) {
                const int r = x / (RP - R), c = R + x - r * (RP - R);
                Vt[r * RP + c] = 0.0, At[r * RP + c] = 0.0;
            }
        __syncthreads();
        if (l < lanes) {
            auto emit = [&](int r, double x) {
                const T xt = (T)x;
                const int64_t ix = (rt + r) * R + j;
                if (ex.mc) {
                    mm_store(reinterpret_cast<T *>(ex.mc) + ix, xt);
                } else if (ex.np) {
                    for (int p = 0; p < ex.np; ++p) reinterpret_cast<T *>(ex.peer[p])[ix] = xt;
                } else {
                    A[ix] = xt;
                }
                const double xd = (double)xt;
                At[r * RP + j] = xd;
                sq += xd * xd;
                dot += xd * Vt[r * RP + j];
            };
            // two partial sums per row: FMA chains of R/2 (one chain of R is
            // latency-bound, ncu "wait" stalls); one row per pass keeps the
            // register count (two rows per pass: 158 registers, one block per
            // SM, measured slower)
            for (int r = l; r < nr; r += lanes) {
                const double2 *v2 = reinterpret_cast<const double2 *>(Vt + r * RP);
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int i = 0; i < RM; i += 2) {
                    if (i < R) {
                        const double2 q = v2[i >> 1];
                        a0 += q.x * gi[i];
                        a1 += q.y * gi[i + 1];
                    }
                }
                emit(r, a0 + a1);
            }
        }
        __syncthreads();
        if (grp < groups) {
            for (int r = grp; r < nr; r += groups) {
                const double2 x01 = *reinterpret_cast<const double2 *>(At + r * RP + a0);
                const double2 x23 = *reinterpret_cast<const double2 *>(At + r * RP + a0 + 2);
                const double2 y01 = *reinterpret_cast<const double2 *>(At + r * RP + c0);
                const double2 y23 = *reinterpret_cast<const double2 *>(At + r * RP + c0 + 2);
                const double x[4] = {x01.x, x01.y, x23.x, x23.y};
                const double y[4] = {y01.x, y01.y, y23.x, y23.y};
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int q = 0; q < 4; ++q) g[p * 4 + q] += x[p] * y[q];
            }
        }
    }
    // the stores to the other ranks' replicas are visible before this rank's
    // next collective (the all-reduce of the partials) is issued
    if (ex.np || ex.mc) __threadfence_system();
    __syncthreads();
    red[tid] = sq;
    red[256 + tid] = dot;
    __syncthreads();
    if (tid < R) {
        double a = 0.0, d = 0.0;
        for (int q = 0; q < lanes; ++q) {
            a += red[q * R + tid];
            d += red[256 + q * R + tid];
        }
        part_sq[(int64_t)blockIdx.x * R + tid] = a;
        if (part_dot) part_dot[(int64_t)blockIdx.x * R + tid] = d;
    }
    __syncthreads();
    // Gram partials: sum the row groups of each 4 x 4 block in group order
    double *gs = sm;  // [groups][nblk][16] in the V/A tiles (no longer read)
    if (grp < groups) {
        double *o = gs + ((size_t)grp * nblk + bi) * 16;
#pragma unroll
        for (int q = 0; q < 16; ++q) o[q] = g[q];
    }
    __syncthreads();
    double *gp = gpart + (int64_t)blockIdx.x * R * R;
    for (int e = tid; e < nblk * 16; e += blockDim.x) {
        const int b = e >> 4, q = e & 15;
        int ba0, bc0;
        block_of(b, ba0, bc0);
        const int a = ba0 + (q >> 2), c = bc0 + (q & 3);
        double acc = 0.0;
        for (int gg = 0; gg < groups; ++gg) acc += gs[((size_t)gg * nblk + b) * 16 + q];
        if (a < R && c < R) gp[a * R + c] = gp[c * R + a] = acc;
    }
    apply_tail<T>(tail, A, R, part_sq, part_dot, gpart, ex.zb);
}

// Warp-private variant of apply_gram (round 2; option apply_warp): no block-wide
// barrier inside the row loop.  A warp takes groups of 32/LR consecutive rows
// (LR = R rounded up to 8/16/32 lanes, lane = (row slot, column j)), stages the
// V rows and the A_raw rows it computes in its own shared-memory tile, reads
// them back as broadcasts (two columns per 128-bit load), and keeps column j
// of Gamma^{-1} and row j of the Gram partial in registers: A_raw(r, j) =
// sum_i V(r, i) Gamma^{-1}(i, j) in two partial sums, G_raw(j, b) += A(r, j)
// A(r, b) for every b.  The next group's V is loaded before the current one is
// used.  Partials are reduced across row slots (shuffles) and warps (shared
// memory) in a fixed order, then the same per-block partials / last-block tail
// as apply_gram.  The smem-tile kernel above synchronises the block three
// times per 64-row tile; on LBNL's 868K-row mode it ran at 2.1 TB/s (ncu:
// 16 warps/SM, "wait" and barrier stalls).
template <int LR>
__host__ __device__ constexpr size_t apply_warp_smem_doubles() {
    return (size_t)8 * 2 * 32 + (size_t)8 * LR * LR + (size_t)2 * 8 * LR;
}

template <typename T, int LR>
__global__ void __launch_bounds__(256, 2)
    apply_gram_warp_kernel(const T *__restrict__ V, int64_t r_begin, int64_t r_end, int R,
                           const double *__restrict__ Ginv, T *__restrict__ A,
                           double *__restrict__ part_sq, double *__restrict__ part_dot,
                           double *__restrict__ gpart, const ModeTail tail, const ExchOut ex) {
    pdl_wait();
    if (apply_zero_blocks(ex)) return;
    constexpr int RPW = 32 / LR;
    extern __shared__ __align__(16) double wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int rs = lane / LR, j = lane % LR;
    double *Vw = wsm + warp * 64;            // [RPW][LR] V rows of the group
    double *Aw = Vw + 32;                    // [RPW][LR] A_raw rows of the group
    double *gs = wsm + 8 * 64;               // [8][LR][LR] per-warp Gram sums
    double *ss = gs + 8 * LR * LR;           // [8][LR] column sums of squares
    double *ds = ss + 8 * LR;                // [8][LR] column dots with V
    double gi[LR], g[LR];
#pragma unroll
    for (int i = 0; i < LR; ++i) {
        gi[i] = (i < R && j < R) ? Ginv[i * R + j] : 0.0;
        g[i] = 0.0;
    }
    double sq = 0.0, dot = 0.0;
    const int64_t ngroups = (r_end - r_begin + RPW - 1) / RPW;
    const int64_t wstride = (int64_t)(gridDim.x - ex.zb) * 8;
    auto load_v = [&](int64_t grp) {
        const int64_t r = r_begin + grp * RPW + rs;
        return (grp < ngroups && r < r_end && j < R) ? (double)V[r * R + j] : 0.0;
    };
    int64_t grp = blockIdx.x * (int64_t)8 + warp;
    double vnext = load_v(grp);
    for (; grp < ngroups; grp += wstride) {
        const double v = vnext;
        vnext = load_v(grp + wstride);
        const int64_t r = r_begin + grp * RPW + rs;
        const bool on = r < r_end && j < R;
        Vw[rs * LR + j] = v;
        __syncwarp();
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int i = 0; i < LR; i += 2) {
            const double2 q = *reinterpret_cast<const double2 *>(Vw + rs * LR + i);
            x0 += q.x * gi[i];
            x1 += q.y * gi[i + 1];
        }
        double xd = 0.0;
        if (on) {
            const T xt = (T)(x0 + x1);
            const int64_t ix = r * R + j;
            if (ex.mc) {
                mm_store(reinterpret_cast<T *>(ex.mc) + ix, xt);
            } else if (ex.np) {
                for (int p = 0; p < ex.np; ++p) reinterpret_cast<T *>(ex.peer[p])[ix] = xt;
            } else {
                A[ix] = xt;
            }
            xd = (double)xt;
        }
        Aw[rs * LR + j] = xd;
        __syncwarp();
        sq += xd * xd;
        dot += xd * v;
#pragma unroll
        for (int b = 0; b < LR; b += 2) {
            const double2 q = *reinterpret_cast<const double2 *>(Aw + rs * LR + b);
            g[b] += xd * q.x;
            g[b + 1] += xd * q.y;
        }
        __syncwarp();
    }
    if (ex.np || ex.mc) __threadfence_system();  // replicas written before the all-reduce
    // fixed-order reduction: row slots (shuffles), then warps (shared memory)
#pragma unroll
    for (int o = LR; o < 32; o <<= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        dot += __shfl_xor_sync(0xffffffffu, dot, o);
#pragma unroll
        for (int b = 0; b < LR; ++b) g[b] += __shfl_xor_sync(0xffffffffu, g[b], o);
    }
    if (rs == 0) {
#pragma unroll
        for (int b = 0; b < LR; ++b) gs[(warp * LR + j) * LR + b] = g[b];
        ss[warp * LR + j] = sq;
        ds[warp * LR + j] = dot;
    }
    __syncthreads();
    const int RR = R * R;
    for (int e = tid; e < RR; e += blockDim.x) {
        const int a = e / R, b = e % R;
        double acc = 0.0;
        for (int w = 0; w < 8; ++w) acc += gs[(w * LR + a) * LR + b];
        gpart[(int64_t)blockIdx.x * RR + e] = acc;
    }
    for (int c = tid; c < R; c += blockDim.x) {
        double a2 = 0.0, d2 = 0.0;
        for (int w = 0; w < 8; ++w) {
            a2 += ss[w * LR + c];
            d2 += ds[w * LR + c];
        }
        part_sq[(int64_t)blockIdx.x * R + c] = a2;
        if (part_dot) part_dot[(int64_t)blockIdx.x * R + c] = d2;
    }
    apply_tail<T>(tail, A, R, part_sq, part_dot, gpart, ex.zb);
}

// ------------------------------------------ apply_gram on the FP64 tensor cores
// R = 8 RB (8 or 16).  The warp-private kernel above issues 16 + 16 DFMA per
// row in dependent chains and holds Gamma^{-1} and the Gram row in 64
// registers (2 blocks/SM): on LBNL's 868K-row mode it ran at 22 % of the FP64
// pipe and 1.8 TB/s (110-117 us for 222 MB).  Here a warp takes 8 rows at a
// time and both products are DMMA (mma.sync m8n8k4 f64; the fp64 path of the
// B200 tensor cores -- tcgen05 has no f64 kind):
//   A_raw(8 x R) = V(8 x R) Gamma^{-1}(R x R): RB n-blocks x 2RB k-steps,
//     Gamma^{-1} held as B fragments (2 RB^2 doubles per lane);
//   G_raw += A_raw^T A_raw over the 8 rows: the RB(RB+1)/2 upper 8x8 blocks
//     x 2 k-steps, A_raw re-read from shared memory in operand layout;
// colsq = diag(G_raw); dot(A_raw, V) from the result fragments.  The V tile
// (8 rows, contiguous since the row stride is R) is one coalesced load per
// lane, prefetched a tile ahead.  Same per-block partials / tail / exchange
// stores as the kernels above; a fixed summation order (deterministic).
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// shared-memory row stride of the V / A_raw tiles: 8RB + 4 doubles, so that
// the fragment loads (8 rows x 4 columns) and stores hit distinct banks per
// half-warp (a 128-byte row stride put all 8 rows of a column in one bank:
// 8-way conflicts on every fragment access)
template <int RB>
__host__ __device__ constexpr int mma_tile_stride() { return 8 * RB + 4; }
template <int RB>
__host__ __device__ constexpr size_t apply_mma_smem_doubles() {
    // per warp: V tile + A_raw tile (8 rows each); per block: 8 Gram partials
    // (8RB)^2 + colsq / dot partials 2 x 8 x 8RB
    return (size_t)8 * 2 * 8 * mma_tile_stride<RB>() + (size_t)8 * (8 * RB) * (8 * RB) +
           (size_t)2 * 8 * (8 * RB);
}

#ifndef SPTK_APPLY_MMA_PF  // A/B builds only
#define SPTK_APPLY_MMA_PF 1
#endif
#ifndef SPTK_APPLY_MMA_MINB
#define SPTK_APPLY_MMA_MINB 3
#endif
constexpr int kApplyMmaPf = SPTK_APPLY_MMA_PF;

template <typename T, int RB>
__global__ void __launch_bounds__(256, SPTK_APPLY_MMA_MINB)
    apply_gram_mma_kernel(const T *__restrict__ V, int64_t r_begin, int64_t r_end, int R,
                          const double *__restrict__ Ginv, T *__restrict__ A,
                          double *__restrict__ part_sq, double *__restrict__ part_dot,
                          double *__restrict__ gpart, const ModeTail tail, const ExchOut ex) {
    pdl_wait();
    if (apply_zero_blocks(ex)) return;
    constexpr int RR = 8 * RB;       // == R
    constexpr int PL = RR * 8 / 32;  // V / A_raw tile doubles per lane (2 RB)
    constexpr int NB = RB * (RB + 1) / 2;
    extern __shared__ __align__(16) double msm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int g = lane >> 2, q = lane & 3;
    constexpr int S = mma_tile_stride<RB>();
    double *vt = msm + warp * 2 * 8 * S;    // [8][S]
    double *at = vt + 8 * S;                // [8][S]
    double *gs = msm + 8 * 2 * 8 * S;       // [8 warps][RR][RR]
    double *ss = gs + 8 * RR * RR;          // [8][RR] colsq partials
    double *ds = ss + 8 * RR;               // [8][RR] dot partials
    // Gamma^{-1} as B fragments: gib[ks][nb] = Ginv[4ks + q][8nb + g]
    double gib[2 * RB][RB];
#pragma unroll
    for (int ks = 0; ks < 2 * RB; ++ks)
#pragma unroll
        for (int nb = 0; nb < RB; ++nb) gib[ks][nb] = Ginv[(4 * ks + q) * RR + 8 * nb + g];
    double gacc[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) gacc[b][0] = gacc[b][1] = 0.0;
    double dacc[RB][2];
#pragma unroll
    for (int nb = 0; nb < RB; ++nb) dacc[nb][0] = dacc[nb][1] = 0.0;
    const int64_t ntile = (r_end - r_begin + 7) / 8;
    const int64_t wstride = (int64_t)(gridDim.x - ex.zb) * 8;
    // lane's slice of a V tile: row lane / (32/8... ) -- tile doubles [PL*lane, PL*lane + PL)
    auto load_tile = [&](int64_t ti, double (&v)[PL]) {
        const int64_t e0 = (r_begin + ti * 8) * RR + (int64_t)lane * PL;  // element index
        const int64_t lim = r_end * RR;
        if (ti < ntile && e0 + PL <= lim) {
            if constexpr (sizeof(T) == 8 && PL == 4) {
                const double4 x = *reinterpret_cast<const double4 *>(V + e0);
                v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
            } else if constexpr (sizeof(T) == 8 && PL == 2) {
                const double2 x = *reinterpret_cast<const double2 *>(V + e0);
                v[0] = x.x; v[1] = x.y;
            } else {
#pragma unroll
                for (int k = 0; k < PL; ++k) v[k] = (double)V[e0 + k];
            }
        } else {
#pragma unroll
            for (int k = 0; k < PL; ++k) v[k] = (ti < ntile && e0 + k < lim) ? (double)V[e0 + k] : 0.0;
        }
    };
    // V tiles kApplyMmaPf ahead (1 KB per warp each; 4 ahead at 2 blocks/SM
    // measured 2 % slower on LBNL than 1 ahead at 3 blocks/SM once the tile
    // strides were conflict-free, profiles/r02/s2/ab_apply_mma_variants.log)
    int64_t ti0 = blockIdx.x * (int64_t)8 + warp;
    double vn[kApplyMmaPf][PL];
#pragma unroll
    for (int u = 0; u < kApplyMmaPf; ++u) load_tile(ti0 + u * wstride, vn[u]);
    for (; ti0 < ntile; ti0 += kApplyMmaPf * wstride)
#pragma unroll
    for (int u = 0; u < kApplyMmaPf; ++u) {
        const int64_t ti = ti0 + u * wstride;
        if (ti >= ntile) break;
        {   // the lane's PL consecutive doubles: row lane / (RR / PL), padded stride
            const int e = lane * PL, row = e / RR, col = e % RR;
#pragma unroll
            for (int k = 0; k < PL; ++k) vt[row * S + col + k] = vn[u][k];
        }
        load_tile(ti + kApplyMmaPf * wstride, vn[u]);
        __syncwarp();
        // A_raw = V Gamma^{-1}: D fragment (row g, cols 8nb + 2q + {0,1})
        double d[RB][2];
#pragma unroll
        for (int nb = 0; nb < RB; ++nb) d[nb][0] = d[nb][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2 * RB; ++ks) {
            const double a = vt[g * S + 4 * ks + q];
#pragma unroll
            for (int nb = 0; nb < RB; ++nb) dmma(d[nb][0], d[nb][1], a, gib[ks][nb]);
        }
        const int64_t r = r_begin + ti * 8 + g;
        const bool on = r < r_end;
#pragma unroll
        for (int nb = 0; nb < RB; ++nb) {
            const int c = 8 * nb + 2 * q;
            const T x0 = (T)d[nb][0], x1 = (T)d[nb][1];
            double y0 = 0.0, y1 = 0.0;
            if (on) {
                const int64_t ix = r * RR + c;
                if (ex.mc) {
                    mm_store(reinterpret_cast<T *>(ex.mc) + ix, x0);
                    mm_store(reinterpret_cast<T *>(ex.mc) + ix + 1, x1);
                } else if (ex.np) {
                    for (int p = 0; p < ex.np; ++p) {
                        reinterpret_cast<T *>(ex.peer[p])[ix] = x0;
                        reinterpret_cast<T *>(ex.peer[p])[ix + 1] = x1;
                    }
                } else if constexpr (sizeof(T) == 8) {
                    *reinterpret_cast<double2 *>(A + ix) = make_double2(x0, x1);
                } else {
                    *reinterpret_cast<float2 *>(A + ix) = make_float2(x0, x1);
                }
                y0 = (double)x0;
                y1 = (double)x1;
            }
            // the Gram and the fit use the stored (T-rounded) values
            *reinterpret_cast<double2 *>(at + g * S + c) = make_double2(y0, y1);
            dacc[nb][0] += y0 * vt[g * S + c];
            dacc[nb][1] += y1 * vt[g * S + c + 1];
        }
        __syncwarp();
        // G_raw += A_raw^T A_raw: operand fragments f[ks][b] = A_raw[4ks + q][8b + g]
        double f[2][RB];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int b = 0; b < RB; ++b) f[ks][b] = at[(4 * ks + q) * S + 8 * b + g];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            int bi = 0;
#pragma unroll
            for (int mb = 0; mb < RB; ++mb)
#pragma unroll
                for (int nb = mb; nb < RB; ++nb, ++bi) dmma(gacc[bi][0], gacc[bi][1], f[ks][mb], f[ks][nb]);
        }
        __syncwarp();
    }
    if (ex.np || ex.mc) __threadfence_system();  // replicas written before the all-reduce
    // per-warp Gram (both triangles) and column partials to shared memory
    {
        double *gw = gs + warp * RR * RR;
        int bi = 0;
#pragma unroll
        for (int mb = 0; mb < RB; ++mb)
#pragma unroll
            for (int nb = mb; nb < RB; ++nb, ++bi)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int a = 8 * mb + g, b = 8 * nb + 2 * q + e;
                    gw[a * RR + b] = gacc[bi][e];
                    if (mb != nb) gw[b * RR + a] = gacc[bi][e];
                }
        // dot: sum the 8 row slots (lanes of equal q) in a fixed shuffle order
#pragma unroll
        for (int nb = 0; nb < RB; ++nb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double x = dacc[nb][e];
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                if (g == 0) ds[warp * RR + 8 * nb + 2 * q + e] = x;
            }
    }
    __syncthreads();
    for (int c = tid; c < RR; c += blockDim.x)
        for (int w = 0; w < 8; ++w) ss[w * RR + c] = gs[(w * RR + c) * RR + c];  // colsq = diag
    __syncthreads();
    const int RRR = RR * RR;
    for (int e = tid; e < RRR; e += blockDim.x) {
        double acc = 0.0;
        for (int w = 0; w < 8; ++w) acc += gs[w * RRR + e];
        gpart[(int64_t)blockIdx.x * RRR + e] = acc;
    }
    for (int c = tid; c < RR; c += blockDim.x) {
        double a2 = 0.0, d2 = 0.0;
        for (int w = 0; w < 8; ++w) {
            a2 += ss[w * RR + c];
            d2 += ds[w * RR + c];
        }
        part_sq[(int64_t)blockIdx.x * RR + c] = a2;
        if (part_dot) part_dot[(int64_t)blockIdx.x * RR + c] = d2;
    }
    apply_tail<T>(tail, A, RR, part_sq, part_dot, gpart, ex.zb);
}

// apply_gram grid cap: one full wave of resident blocks (SPTK_APPLY_WAVE=0: the
// 8-per-SM cap alone, for A/B) -- a tall mode's pass otherwise runs ~2.7 waves
template <typename T>
static int apply_block_cap(int cap, int R, size_t smb) {
    const bool wave = opt(OPT_APPLY_WAVE) != 0;
    if (!wave) return cap;
    int occ = 0;
    if (R <= 16)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, apply_gram_kernel<T, 16>, 256, smb);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, apply_gram_kernel<T, 32>, 256, smb);
    return occ > 0 ? std::min(cap, occ * dev_sms()) : cap;
}

// A(:, j) *= s_j (the deferred normalisation, once after the last iteration)
template <typename T>
__global__ void scale_columns_kernel(T *__restrict__ A, int64_t I, int R,
                                     const double *__restrict__ s) {
    const int64_t n = I * R;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        A[i] = (T)((double)A[i] * s[i % R]);
}

template <typename T>
__global__ void fill_kernel(T *__restrict__ out, int n, T v) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = v;
}

__global__ void fill_f64_kernel(double *__restrict__ out, int n, double v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = v;
}

// ---------------------------------------------------------- tiled glue (R > 32)
// Register-blocked fp64 tiles for the two dense products of the glue when R
// is large (the paper's R = 128 CP-ALS workload): A_raw = V Gamma^{-1} and the
// Gram matrix A^T A.  64 x 64 output tiles, 256 threads x (4 x 4) outputs,
// k-chunks of 32 staged in shared memory.
constexpr int kTB = 64, kTK = 32;

// A_raw(k,:) = V(k,:) Ginv for rows [r0, r1); grid (row tiles, col tiles).
// part_sq / part_dot: [row tile][R] column partials of A_raw^2 and A_raw .* V.
template <typename T>
__global__ void __launch_bounds__(256)
    apply_inv_tiled_kernel(const T *__restrict__ V, int64_t r0, int64_t r1, int R,
                           const double *__restrict__ Ginv, T *__restrict__ A,
                           double *__restrict__ part_sq, double *__restrict__ part_dot) {
    __shared__ double sV[kTB][kTK + 1];             // [row][k] (padded: conflict-free)
    __shared__ __align__(16) double sG[kTK][kTB];   // [k][col] (vector reads)
    // after the main loop sV is reused for the column partials: red[2][16][kTB]
    double(*red)[16][kTB] = reinterpret_cast<double(*)[16][kTB]>(&sV[0][0]);
    static_assert(2 * 16 * kTB <= kTB * (kTK + 1), "partials must fit in sV");
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t row0 = r0 + (int64_t)blockIdx.x * kTB;
    const int col0 = blockIdx.y * kTB;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < R; k0 += kTK) {
        for (int x = threadIdx.x; x < kTB * kTK; x += 256) {
            const int r = x / kTK, k = x % kTK;  // V tile: coalesced along k
            const int64_t row = row0 + r;
            sV[r][k] = (row < r1 && k0 + k < R) ? (double)V[row * R + k0 + k] : 0.0;
            const int kk = x / kTB, c = x % kTB;  // Ginv tile: coalesced along cols
            sG[kk][c] = (k0 + kk < R && col0 + c < R) ? Ginv[(int64_t)(k0 + kk) * R + col0 + c] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < kTK; ++k) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sV[ty * 4 + i][k];
            const double2 g01 = *reinterpret_cast<const double2 *>(&sG[k][tx * 4]);
            const double2 g23 = *reinterpret_cast<const double2 *>(&sG[k][tx * 4 + 2]);
            b[0] = g01.x; b[1] = g01.y; b[2] = g23.x; b[3] = g23.y;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
        }
        __syncthreads();
    }
    double sq[4] = {0, 0, 0, 0}, dt[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t row = row0 + ty * 4 + i;
        if (row >= r1) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = col0 + tx * 4 + j;
            if (col >= R) continue;
            const T v = (T)acc[i][j];
            A[row * R + col] = v;
            sq[j] += (double)v * (double)v;
            dt[j] += (double)v * (double)V[row * R + col];
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        red[0][ty][tx * 4 + j] = sq[j];
        red[1][ty][tx * 4 + j] = dt[j];
    }
    __syncthreads();
    if (threadIdx.x < kTB) {
        const int col = col0 + threadIdx.x;
        if (col < R) {
            double a = 0.0, d = 0.0;
            for (int q = 0; q < 16; ++q) {
                a += red[0][q][threadIdx.x];
                d += red[1][q][threadIdx.x];
            }
            part_sq[(int64_t)blockIdx.x * R + col] = a;
            if (part_dot) part_dot[(int64_t)blockIdx.x * R + col] = d;
        }
    }
}

// partial[b][a*R + c] = sum over rows of block b of A(k,a) A(k,c);
// grid (row chunks, (R/64)^2 output tiles)
template <typename T>
__global__ void __launch_bounds__(256)
    gram_tiled_kernel(const T *__restrict__ A, int64_t I, int R, int64_t rows_per_block,
                      double *__restrict__ partial) {
    __shared__ __align__(16) double sa[kTK][kTB];
    __shared__ __align__(16) double sb[kTK][kTB];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int nt = (R + kTB - 1) / kTB;
    const int ta = blockIdx.y / nt, tb = blockIdx.y % nt;
    const int64_t b0 = (int64_t)blockIdx.x * rows_per_block;
    const int64_t b1 = min(I, b0 + rows_per_block);
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t k0 = b0; k0 < b1; k0 += kTK) {
        for (int x = threadIdx.x; x < kTB * kTK; x += 256) {
            const int k = x / kTB, c = x % kTB;
            const int64_t row = k0 + k;
            const int ca = ta * kTB + c, cb = tb * kTB + c;
            sa[k][c] = (row < b1 && ca < R) ? (double)A[row * R + ca] : 0.0;
            sb[k][c] = (row < b1 && cb < R) ? (double)A[row * R + cb] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < kTK; ++k) {
            double a[4], b[4];
            const double2 a01 = *reinterpret_cast<const double2 *>(&sa[k][ty * 4]);
            const double2 a23 = *reinterpret_cast<const double2 *>(&sa[k][ty * 4 + 2]);
            const double2 b01 = *reinterpret_cast<const double2 *>(&sb[k][tx * 4]);
            const double2 b23 = *reinterpret_cast<const double2 *>(&sb[k][tx * 4 + 2]);
            a[0] = a01.x; a[1] = a01.y; a[2] = a23.x; a[3] = a23.y;
            b[0] = b01.x; b[1] = b01.y; b[2] = b23.x; b[3] = b23.y;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int ra = ta * kTB + ty * 4 + i;
        if (ra >= R) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cb = tb * kTB + tx * 4 + j;
            if (cb < R) partial[(int64_t)blockIdx.x * R * R + (int64_t)ra * R + cb] = acc[i][j];
        }
    }
}

template <typename T>
__global__ void cast_kernel(const double *__restrict__ in, int n, T *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (T)in[i];
}

// ---------------------------------------------------------------- host
static int grid_for(int64_t n, int per = 256) {
    int64_t b = (n + per - 1) / per;
    const int64_t cap = (int64_t)dev_sms() * 8;
    if (b > cap) b = cap;
    return b < 1 ? 1 : (int)b;
}

struct AlsCtx {
    sptk_tensor t;
    int64_t R;                             // row stride of the factors: the padded rank
    int64_t Rl;                            // rank of the decomposition (<= R)
    cudaStream_t s;
    sptk_comm comm;
    std::vector<void *> A;                 // device factor pointers
    std::vector<std::vector<int64_t>> b;   // per-mode row bounds (comm)
    int nblocks;                           // blocks of the R x R partial-sum kernels
    int nb_row;                            // blocks of the R-vector partial-sum kernels
    size_t part_stride;                    // doubles between the psq and pdot partials
    int nb_apply = 0;                      // block cap of apply_gram
    // sharded deferred path: factor replicas in the comm's symmetric buffer
    bool sym_iter = false;
    // pre-zeroed MTTKRP outputs (single GPU): mode n writes V buffer vb[n];
    // consecutive modes use different buffers, and the buffer a mode's apply
    // has just released is zeroed on the side stream for its next user while
    // the next MTTKRP runs -- the zeroing (LBNL's 868K-row mode: 111 MB,
    // 17 us) leaves the critical path.  zsame[m]: mode m's buffer is zeroed
    // earlier in the same iteration (its MTTKRP waits for ev_zero[m]);
    // otherwise in the previous iteration (graph launches are serialised).
    bool prezero = false;
    bool zapply = false;   // option zero_in_apply: pre-zeroing by the previous mode's apply launch
    bool copy_fit = true;  // per-iteration D2H of (fit, status) inside the iteration
    void *vbuf[3] = {};
    int vb[kMaxModes] = {};
    int znext[kMaxModes] = {};  // the mode whose buffer is zeroed when mode n starts
    bool zsame[kMaxModes] = {};
    bool pz[kMaxModes] = {};    // mode m's output is pre-zeroed (>= 256 MB; smaller ones zero in-launch)
    std::vector<size_t> off;               // byte offset of A_m in c.comm->sym
};

// Plan and launch of the apply pass over rows [r0, r1): the warp-private kernel
// (option apply_warp, default) or the shared-memory tile kernel.  small: the
// caller wants at most kTailBlocks blocks (the last one finalises the mode).
struct ApplyPlan {
    bool mma = false;   // apply_gram_mma_kernel (R = 8 or 16)
    bool warp = false;
    int LR = 16, tile = 0, nb = 1;
    int64_t rpb = 0;
    size_t smb = 0;
};

template <typename T, int LR>
static int warp_apply_cap(size_t smb) {
    // per device: the attribute and the occupancy are properties of the
    // device's context (a process may drive several GPUs)
    static std::atomic<int> occ[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (occ[dev].load() < 1) {
        cudaFuncSetAttribute(apply_gram_warp_kernel<T, LR>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, apply_gram_warp_kernel<T, LR>, 256,
                                                          smb) != cudaSuccess || o < 1) {
            cudaGetLastError();
            o = 1;
        }
        occ[dev].store(o);
    }
    return occ[dev].load() * dev_sms();
}

template <typename T, int RB>
static int mma_apply_cap(size_t smb) {
    static std::atomic<int> occ[64];  // per device (see warp_apply_cap)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (occ[dev].load() < 1) {
        cudaFuncSetAttribute(apply_gram_mma_kernel<T, RB>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, apply_gram_mma_kernel<T, RB>, 256,
                                                          smb) != cudaSuccess || o < 1) {
            cudaGetLastError();
            o = 1;
        }
        occ[dev].store(o);
    }
    return occ[dev].load() * dev_sms();
}

template <typename T>
static ApplyPlan plan_apply(AlsCtx &c, int64_t rows, int R, bool small) {
    ApplyPlan p;
    // FP64 tensor-core apply for R = 8 / 16 (R is the padded rank here)
    p.mma = opt(OPT_APPLY_MMA) != 0 && (R == 8 || R == 16);
    if (p.mma) {
        p.LR = R;
        p.smb = sizeof(double) * (R == 8 ? apply_mma_smem_doubles<1>() : apply_mma_smem_doubles<2>());
        const int cap = R == 8 ? mma_apply_cap<T, 1>(p.smb) : mma_apply_cap<T, 2>(p.smb);
        const int64_t tiles = (rows + 7) / 8;
        int64_t nb = std::min<int64_t>(cap, (tiles + 7) / 8);
        if (small) nb = std::min<int64_t>(nb, kTailBlocks);
        if (tiles <= 64) nb = 1;  // <= 8 tiles per warp: one block, no cross-block reduction
        p.nb = (int)std::max<int64_t>(nb, 1);
        return p;
    }
    // the warp kernel for R <= 16 (LBNL -0.6 %, C1 -1.7 %, NELL-2 and Delicious
    // neutral); at R = 32 its 64 register-held doubles spill (+2.8 %)
    p.warp = opt(OPT_APPLY_WARP) != 0 && R <= 16;
    if (p.warp) {
        p.LR = R <= 8 ? 8 : R <= 16 ? 16 : 32;
        int cap = 0;
        if (p.LR == 8) {
            p.smb = sizeof(double) * apply_warp_smem_doubles<8>();
            cap = warp_apply_cap<T, 8>(p.smb);
        } else if (p.LR == 16) {
            p.smb = sizeof(double) * apply_warp_smem_doubles<16>();
            cap = warp_apply_cap<T, 16>(p.smb);
        } else {
            p.smb = sizeof(double) * apply_warp_smem_doubles<32>();
            cap = warp_apply_cap<T, 32>(p.smb);
        }
        const int64_t groups = (rows + 32 / p.LR - 1) / (32 / p.LR);
        int64_t nb = std::min<int64_t>(cap, (groups + 7) / 8);
        if (small) nb = std::min<int64_t>(nb, kTailBlocks);
        p.nb = (int)std::max<int64_t>(nb, 1);
        return p;
    }
    p.tile = std::min(apply_tile_rows(), apply_pf(R <= 16 ? 16 : 32) * 256 / R);
    p.smb = sizeof(double) * (2 * p.tile * ((R + 3) & ~3) + 4 * 256);
    int nb = (int)std::min<int64_t>(apply_block_cap<T>(c.nb_apply, R, p.smb),
                                    (rows + p.tile - 1) / p.tile);
    if (small) nb = std::min(nb, kTailBlocks);
    if (nb < 1) nb = 1;
    p.rpb = (rows + nb - 1) / nb;
    p.nb = (int)((rows + p.rpb - 1) / p.rpb);
    return p;
}

template <typename T>
static cudaError_t run_apply(const ApplyPlan &p, cudaStream_t s, const T *V, int64_t r0,
                             int64_t r1, int R, const double *Ginv, T *An, double *psq,
                             double *pdot, double *gpart, const ModeTail &tail,
                             const ExchOut &ex) {
    if (p.mma) {
        if (p.LR == 8)
            return launch_pdl(apply_gram_mma_kernel<T, 1>, p.nb + ex.zb, 256, p.smb, s, V, r0, r1, R, Ginv,
                              An, psq, pdot, gpart, tail, ex);
        return launch_pdl(apply_gram_mma_kernel<T, 2>, p.nb + ex.zb, 256, p.smb, s, V, r0, r1, R, Ginv, An,
                          psq, pdot, gpart, tail, ex);
    }
    if (p.warp) {
        if (p.LR == 8)
            return launch_pdl(apply_gram_warp_kernel<T, 8>, p.nb + ex.zb, 256, p.smb, s, V, r0, r1, R, Ginv,
                              An, psq, pdot, gpart, tail, ex);
        if (p.LR == 16)
            return launch_pdl(apply_gram_warp_kernel<T, 16>, p.nb + ex.zb, 256, p.smb, s, V, r0, r1, R, Ginv,
                              An, psq, pdot, gpart, tail, ex);
        return launch_pdl(apply_gram_warp_kernel<T, 32>, p.nb + ex.zb, 256, p.smb, s, V, r0, r1, R, Ginv,
                          An, psq, pdot, gpart, tail, ex);
    }
    if (R <= 16)
        return launch_pdl(apply_gram_kernel<T, 16>, p.nb + ex.zb, 256, p.smb, s, V, r0, r1, R, p.rpb,
                          p.tile, Ginv, An, psq, pdot, gpart, tail, ex);
    return launch_pdl(apply_gram_kernel<T, 32>, p.nb + ex.zb, 256, p.smb, s, V, r0, r1, R, p.rpb, p.tile,
                      Ginv, An, psq, pdot, gpart, tail, ex);
}

// G_m = A_m^T A_m (fixed-order reduction of per-block partials in `part`,
// default w.partial; the fused path passes w.gpart so w.partial keeps the
// fit's column partials)
// rows [r0, r1) only when r1 >= 0 (a rank's own rows; an empty range gives 0)
template <typename T>
static sptk_status gram(AlsCtx &c, int m, double *part = nullptr, int64_t r0 = 0,
                        int64_t r1 = -1) {
    sptk_tensor t = c.t;
    ALSWork &w = t->als;
    const int R = (int)c.R;
    if (r1 < 0) r1 = t->dims[m];
    const int64_t I = r1 - r0;
    if (I <= 0) {
        SPTK_CUDA(cudaMemsetAsync(w.G.as<double>() + (int64_t)m * R * R, 0,
                                  sizeof(double) * R * R, c.s));
        return SPTK_OK;
    }
    const T *Am = static_cast<const T *>(c.A[m]) + r0 * R;
    int nb = (int)std::min<int64_t>(c.nblocks, (I + kGramTileRows - 1) / kGramTileRows);
    const int64_t rpb = (I + nb - 1) / nb;
    nb = (int)((I + rpb - 1) / rpb);
    if (!part) part = w.partial.as<double>();
    if (R > 32) {
        const int nt = (R + kTB - 1) / kTB;
        gram_tiled_kernel<T><<<dim3((unsigned)nb, (unsigned)(nt * nt)), 256, 0, c.s>>>(
            Am, I, R, rpb, part);
    } else {
        const size_t sm = sizeof(double) * kGramTileRows * R;
        if (R <= 16)
            gram_partial_kernel<T, 1><<<nb, 256, sm, c.s>>>(Am, I, R, rpb, part);
        else
            gram_partial_kernel<T, 4><<<nb, 256, sm, c.s>>>(Am, I, R, rpb, part);
    }
    reduce_partials_kernel<<<(R * R + 7) / 8, 256, 0, c.s>>>(
        part, nb, R * R, w.G.as<double>() + (int64_t)m * R * R);
    count_launch(2);
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

// A_raw = V Gamma^{-1} on rows [r0, r1) with per-partition column partials
// of A_raw^2 (psq) and A_raw .* V (pdot, may be NULL); returns the number of
// partials.  R <= 32: row-parallel kernel; R > 32: register-blocked tiles.
template <typename T>
static sptk_status apply_inverse(AlsCtx &c, const T *V, int64_t r0, int64_t r1, T *An,
                                 double *psq, double *pdot, int *nparts) {
    const int R = (int)c.R;
    const double *Ginv = c.t->als.L.as<double>();
    const int64_t rows = r1 - r0;
    if (R > 32) {  // (measured: the 64x64 tiles lose 2.7x at R = 16)
        const int nrt = (int)((rows + kTB - 1) / kTB);
        const dim3 grid((unsigned)nrt, (unsigned)((R + kTB - 1) / kTB));
        apply_inv_tiled_kernel<T><<<grid, 256, 0, c.s>>>(V, r0, r1, R, Ginv, An, psq, pdot);
        *nparts = nrt;
    } else {
        const int lanes = 256 / R;
        int nb = (int)std::min<int64_t>(c.nb_row, (rows + 4 * lanes - 1) / (4 * lanes));
        if (nb < 1) nb = 1;
        const int64_t rpb = (rows + nb - 1) / nb;
        nb = (int)((rows + rpb - 1) / rpb);
        apply_inv_kernel<T><<<nb, 256, sizeof(double) * (R * R + 512), c.s>>>(
            V, r0, r1, R, rpb, Ginv, An, psq, pdot);
        *nparts = nb;
    }
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

// Single-GPU iteration: per mode the Cholesky/inverse runs on a side stream
// while the MTTKRP runs (it only needs the Gram matrices of the other
// modes), then apply_inv and one finish kernel (lambda, normalise, Gram, fit).
template <typename T>
static sptk_status enqueue_iteration_fused(AlsCtx &c) {
    sptk_tensor t = c.t;
    ALSWork &w = t->als;
    const int N = t->N, R = (int)c.R;
    double *lam = w.lam.as<double>();
    double *scal = w.scal.as<double>();
    int *status = reinterpret_cast<int *>(scal + 8);
    double *Ginv = w.L.as<double>();
    double *s_all = w.scl.as<double>();                      // N x R column scales
    double *graw = s_all + (size_t)N * R;                    // R x R Gram of A_raw
    T *scale = reinterpret_cast<T *>(graw + (size_t)R * R);  // R: next MTTKRP's weights
    double *trace = w.trace.as<double>();                     // device fit history
    int *trace_n = reinterpret_cast<int *>(scal + 12);
    const bool deferred = deferred_norm(R);
    for (int n = 0; n < N; ++n) {
        const bool last = n == N - 1;
        const int64_t I = t->dims[n];
        T *V = c.prezero ? static_cast<T *>(c.vbuf[c.vb[n]]) : w.V.as<T>();
        // side stream: Gamma^{-1} for mode n once G_{n-1} is final
        SPTK_CUDA(cudaEventRecord(w.ev_gram, c.s));
        SPTK_CUDA(cudaStreamWaitEvent(w.side, w.ev_gram, 0));
        launch_ginv(w.G.as<double>(), N, n, R, (int)c.Rl, Ginv, status, w.side);
        count_launch();
        SPTK_CUDA(cudaGetLastError());
        SPTK_CUDA(cudaEventRecord(w.ev_inv, w.side));
        if (c.prezero && !c.zapply) {  // the buffer mode n-1's apply released, for its next user
            const int m = c.znext[n];
            if (c.pz[m]) {
                SPTK_CUDA(cudaMemsetAsync(c.vbuf[c.vb[m]], 0, sizeof(T) * (size_t)t->dims[m] * R,
                                          w.side));
                if (c.zsame[m]) SPTK_CUDA(cudaEventRecord(w.ev_zero[m], w.side));
            }
            if (c.pz[n] && c.zsame[n]) SPTK_CUDA(cudaStreamWaitEvent(c.s, w.ev_zero[n], 0));
        }
        // V = MTTKRP with the normalised factors: raw factors, column scales at the flush
        SPTK_TRY(mttkrp_launch(t, n, c.R, c.A.data(), deferred ? scale : nullptr, V, 0, I, c.s,
                               c.prezero && c.pz[n]));
        SPTK_CUDA(cudaStreamWaitEvent(c.s, w.ev_inv, 0));
        T *An = static_cast<T *>(c.A[n]);
        double *psq = w.partial.as<double>();
        double *pdot = psq + c.part_stride;
        double *colsq = w.colsq.as<double>();
        if (deferred) {  // one pass: A_raw, its Gram partials, column partials; R x R finalise
            // modes up to tail_rows() rows: few fat blocks, so the mode tail
            // (reductions, finalise, fit) runs in the last block, no extra launches
            const ApplyPlan ap = plan_apply<T>(c, I, R, I <= tail_rows());
            const int nb = ap.nb;
            // few blocks (small modes): the last block reduces and finalises
            // in place; many blocks: a single block's reduction is latency-
            // bound (measured slower than the parallel reduction kernels)
            ModeTail tail{};
            tail.counter = nb <= kTailBlocks ? reinterpret_cast<int *>(scale + R) : nullptr;
            tail.colsq = colsq;
            tail.graw = graw;
            tail.s_all = s_all;
            tail.lam = lam;
            tail.G = w.G.as<double>();
            tail.fit = scal;
            tail.trace = trace;
            tail.trace_n = trace_n;
            tail.scale_next = scale;
            tail.normX2 = t->normX2;
            tail.N = N;
            tail.n = n;
            tail.next = (n + 1) % N;
            tail.Rl = (int)c.Rl;
            ExchOut zex{};
            const int nx = (n + 1) % N;
            if (c.zapply && c.pz[nx]) {  // zero the next mode's output from extra blocks
                const size_t bytes = sizeof(T) * (size_t)t->dims[nx] * R;
                zex.zp = static_cast<uint4 *>(c.vbuf[c.vb[nx]]);
                zex.zw = (int64_t)(bytes / 16);
                zex.zb = dev_sms() * 2;
            }
            SPTK_CUDA(run_apply<T>(ap, c.s, V, 0, I, R, Ginv, An, psq, last ? pdot : nullptr,
                                   w.gpart.as<double>(), tail, zex));
            count_launch();
            SPTK_CUDA(cudaGetLastError());
            if (!tail.counter && opt(OPT_FUSED_REDUCE)) {  // one launch: reductions + finalise
                SPTK_CUDA(launch_pdl(reduce_finalize_kernel<T>, reduce_groups(R, last), 256, 0, c.s,
                                     (const double *)psq, (const double *)w.gpart.as<double>(),
                                     (const double *)(last ? pdot : nullptr), nb, R, (int)c.Rl,
                                     colsq, graw, An, N, n, (n + 1) % N, s_all, lam,
                                     w.G.as<double>(), scale, reinterpret_cast<int *>(scale + R),
                                     t->normX2, scal, trace, trace_n));
                count_launch();
                SPTK_CUDA(cudaGetLastError());
            } else if (!tail.counter) {  // many blocks: parallel reductions, then one finalise block
                SPTK_CUDA(launch_pdl(reduce_partials_kernel, (R + 7) / 8, 256, 0, c.s,
                                     (const double *)psq, nb, R, colsq));
                SPTK_CUDA(launch_pdl(reduce_partials_kernel, (R * R + 7) / 8, 256, 0, c.s,
                                     (const double *)w.gpart.as<double>(), nb, R * R, graw));
                SPTK_CUDA(launch_pdl(finalize_mode_kernel<T>, 1, 256, 0, c.s, (const double *)colsq,
                                     (const double *)graw, An, N, n, R, (int)c.Rl, (n + 1) % N,
                                     s_all, lam,
                                     w.G.as<double>(), scale));
                count_launch(3);
                if (last) {
                    double *dot = colsq + R;
                    SPTK_CUDA(launch_pdl(reduce_partials_kernel, (R + 7) / 8, 256, 0, c.s,
                                         (const double *)pdot, nb, R, dot));
                    SPTK_CUDA(launch_pdl(fit_kernel, 1, 256, 0, c.s, (const double *)dot,
                                         (const double *)lam, (const double *)w.G.as<double>(), N,
                                         R, t->normX2, scal, trace, trace_n));
                    count_launch(2);
                }
                SPTK_CUDA(cudaGetLastError());
            }
        } else {  // explicit normalisation: apply, reduce, normalise + Gram
            int nb = 0;
            SPTK_TRY(apply_inverse<T>(c, V, 0, I, An, psq, last ? pdot : nullptr, &nb));
            reduce_partials_kernel<<<(R + 7) / 8, 256, 0, c.s>>>(psq, nb, R, colsq);
            count_launch();
            if (R <= 32) {  // one fused tail: lambda, normalise, Gram partials
                int nf = (int)std::min<int64_t>(c.nblocks, (I + kGramTileRows - 1) / kGramTileRows);
                const int64_t fpb = (I + nf - 1) / nf;
                nf = (int)((I + fpb - 1) / fpb);
                const size_t fsm = sizeof(double) * (R + kGramTileRows * R);
                if (R <= 16)
                    finish_kernel<T, 1><<<nf, 256, fsm, c.s>>>(An, I, R, (int)c.Rl, fpb, colsq,
                                                               w.gpart.as<double>(), lam);
                else
                    finish_kernel<T, 4><<<nf, 256, fsm, c.s>>>(An, I, R, (int)c.Rl, fpb, colsq,
                                                               w.gpart.as<double>(), lam);
                reduce_partials_kernel<<<(R * R + 7) / 8, 256, 0, c.s>>>(
                    w.gpart.as<double>(), nf, R * R, w.G.as<double>() + (int64_t)n * R * R);
                count_launch(2);
            } else {        // large R: normalise, tiled Gram
                normalize_kernel<T><<<grid_for(std::max<int64_t>(I, 1) * R), 256, 0, c.s>>>(
                    An, 0, I, R, (int)c.Rl, colsq, lam);
                count_launch();
                SPTK_CUDA(cudaGetLastError());
                SPTK_TRY(gram<T>(c, n, w.gpart.as<double>()));
            }
            SPTK_CUDA(cudaGetLastError());
            if (last) {
                double *dot = colsq + R;
                reduce_partials_kernel<<<(R + 7) / 8, 256, 0, c.s>>>(pdot, nb, R, dot);
                fit_kernel<<<1, 256, 0, c.s>>>(dot, lam, w.G.as<double>(), N, R, t->normX2, scal,
                                               trace, trace_n);
                count_launch(2);
            }
        }
        SPTK_CUDA(cudaGetLastError());
    }
    if (c.prezero) {  // join the side stream's last zeroing (graph capture needs every fork joined)
        SPTK_CUDA(cudaEventRecord(w.ev_join, w.side));
        SPTK_CUDA(cudaStreamWaitEvent(c.s, w.ev_join, 0));
    }
    // fit and status to pinned host memory (a graph-capturable copy); the
    // no-convergence-test path reads the device fit history instead and copies
    // the (sticky) status once after the last replay
    if (c.copy_fit)
        SPTK_CUDA(cudaMemcpyAsync(w.hres, scal, sizeof(double) * 9, cudaMemcpyDeviceToHost, c.s));
    return SPTK_OK;
}

// Sharded iteration (R <= 32, deferred normalisation): rank g
// owns rows [b_g, b_{g+1}) of every mode.  Per mode: Gamma^{-1} on the side
// stream; the rank's MTTKRP rows (other factors' column scales at the flush);
// apply_gram on its rows, which writes A_raw = V Gamma^{-1} straight into
// every rank's replica of A_n (NVLS multimem or NVLink peer stores: the
// exchange is fused into the kernel that computes the rows) and leaves the
// column / Gram / fit partials; one all-reduce of [colsq, dot, G_raw]
// (2R + R^2 doubles) -- which also orders every rank's stores before anyone
// reads A_n; then the same finalisation as one GPU on every rank.  Without
// peer access the rows go out by grouped NCCL broadcasts instead.
template <typename T>
static sptk_status enqueue_iteration_sharded(AlsCtx &c) {
    sptk_tensor t = c.t;
    ALSWork &w = t->als;
    const int N = t->N, R = (int)c.R;
    SymMem &sm = c.comm->sym;
    double *lam = w.lam.as<double>();
    double *scal = w.scal.as<double>();
    int *status = reinterpret_cast<int *>(scal + 8);
    double *Ginv = w.L.as<double>();
    T *V = w.V.as<T>();
    double *s_all = w.scl.as<double>();
    double *graw_unused = s_all + (size_t)N * R;
    (void)graw_unused;
    T *scale = reinterpret_cast<T *>(s_all + (size_t)N * R + (size_t)R * R);
    double *trace = w.trace.as<double>();
    int *trace_n = reinterpret_cast<int *>(scal + 12);
    double *ared = w.colsq.as<double>();   // [colsq R][dot R][G_raw R^2], all-reduced
    double *psq = w.partial.as<double>();
    double *pdot = psq + c.part_stride;
    const int rank = c.comm->rank;
    for (int n = 0; n < N; ++n) {
        const bool last = n == N - 1;
        const int64_t r0 = c.b[n][rank], r1 = c.b[n][rank + 1], rows = r1 - r0;
        SPTK_CUDA(cudaEventRecord(w.ev_gram, c.s));
        SPTK_CUDA(cudaStreamWaitEvent(w.side, w.ev_gram, 0));
        launch_ginv(w.G.as<double>(), N, n, R, (int)c.Rl, Ginv, status, w.side);
        count_launch();
        SPTK_CUDA(cudaGetLastError());
        SPTK_CUDA(cudaEventRecord(w.ev_inv, w.side));
        SPTK_TRY(mttkrp_launch(t, n, c.R, c.A.data(), scale, V, r0, r1, c.s));
        SPTK_CUDA(cudaStreamWaitEvent(c.s, w.ev_inv, 0));
        T *An = static_cast<T *>(c.A[n]);
        if (rows > 0) {
            const ApplyPlan ap = plan_apply<T>(c, rows, R, false);
            const int nb = ap.nb;
            ExchOut ex{};
            if (sm.exchange == 2) {
                ex.mc = sm.mc + c.off[n];
            } else if (sm.exchange == 1) {
                ex.np = sm.npeer;
                for (int p = 0; p < sm.npeer; ++p) ex.peer[p] = sm.peer[p] + c.off[n];
            }
            ModeTail tail{};  // counter NULL: partials reduced below, across ranks
            SPTK_CUDA(run_apply<T>(ap, c.s, V, r0, r1, R, Ginv, An, psq, last ? pdot : nullptr,
                                   w.gpart.as<double>(), tail, ex));
            reduce_partials_kernel<<<(R + 7) / 8, 256, 0, c.s>>>(psq, nb, R, ared);
            reduce_partials_kernel<<<(R * R + 7) / 8, 256, 0, c.s>>>(w.gpart.as<double>(), nb,
                                                                    R * R, ared + 2 * R);
            count_launch(3);
            if (last) {
                reduce_partials_kernel<<<(R + 7) / 8, 256, 0, c.s>>>(pdot, nb, R, ared + R);
                count_launch();
            }
            SPTK_CUDA(cudaGetLastError());
        } else {
            SPTK_CUDA(cudaMemsetAsync(ared, 0, sizeof(double) * (2 * R + R * R), c.s));
        }
        SPTK_TRY(comm_allreduce_f64(c.comm, ared, 2 * R + (int64_t)R * R, c.s));
        if (sm.exchange == 0)
            SPTK_TRY(comm_bcast_rows(c.comm, An, c.R, t->dtype, c.b[n].data(), c.s));
        finalize_mode_kernel<T><<<1, 256, 0, c.s>>>(ared, ared + 2 * R, An, N, n, R, (int)c.Rl, (n + 1) % N,
                                                     s_all, lam, w.G.as<double>(), scale);
        count_launch();
        if (last) {
            fit_kernel<<<1, 256, 0, c.s>>>(ared + R, lam, w.G.as<double>(), N, R, t->normX2, scal,
                                           trace, trace_n);
            count_launch();
        }
        SPTK_CUDA(cudaGetLastError());
    }
    SPTK_CUDA(cudaMemcpyAsync(w.hres, scal, sizeof(double) * 9, cudaMemcpyDeviceToHost, c.s));
    return SPTK_OK;
}

// wait for the iteration and read (fit, status) from the pinned buffer
static sptk_status complete_iteration(AlsCtx &c, double *fit_host, int *status_host) {
    SPTK_CUDA(cudaStreamSynchronize(c.s));
    const double *h = c.t->als.hres;
    *fit_host = h[0];
    int st;
    memcpy(&st, &h[8], sizeof(int));
    *status_host = st;
    return SPTK_OK;
}

template <typename T>
static sptk_status enqueue_iteration(AlsCtx &c) {
    return c.sym_iter ? enqueue_iteration_sharded<T>(c) : enqueue_iteration_fused<T>(c);
}

template <typename T>
static sptk_status als_iteration(AlsCtx &c, double *fit_host, int *status_host) {
    if (!sharded(c.comm) || c.sym_iter) {
        SPTK_TRY(enqueue_iteration<T>(c));
        return complete_iteration(c, fit_host, status_host);
    }
    sptk_tensor t = c.t;
    ALSWork &w = t->als;
    const int N = t->N, R = (int)c.R;
    const bool multi = sharded(c.comm);
    double *colsq = w.colsq.as<double>();  // [0,R): sum A_raw^2; [R,2R): sum A_raw V
    double *lam = w.lam.as<double>();
    double *scal = w.scal.as<double>();
    int *status = reinterpret_cast<int *>(scal + 8);
    double *Ginv = w.L.as<double>();
    T *V = w.V.as<T>();
    for (int n = 0; n < N; ++n) {
        const bool last = n == N - 1;
        const int64_t r0 = multi ? c.b[n][c.comm->rank] : 0;
        const int64_t r1 = multi ? c.b[n][c.comm->rank + 1] : t->dims[n];
        // Gamma^{-1} on the side stream while this rank's MTTKRP rows run; it
        // needs only the Gram matrices, final once G_{n-1} was all-reduced
        // (the event was recorded there, before the row broadcast)
        if (n == 0) SPTK_CUDA(cudaEventRecord(w.ev_gram, c.s));
        SPTK_CUDA(cudaStreamWaitEvent(w.side, w.ev_gram, 0));
        launch_ginv(w.G.as<double>(), N, n, R, (int)c.Rl, Ginv, status, w.side);
        count_launch();
        SPTK_CUDA(cudaGetLastError());
        SPTK_CUDA(cudaEventRecord(w.ev_inv, w.side));
        SPTK_TRY(mttkrp_launch(t, n, c.R, c.A.data(), nullptr, V, r0, r1, c.s));
        SPTK_CUDA(cudaStreamWaitEvent(c.s, w.ev_inv, 0));
        T *An = static_cast<T *>(c.A[n]);
        const int64_t rows = r1 - r0;
        if (rows > 0) {
            double *pdot = w.partial.as<double>() + c.part_stride;
            int nb = 0;
            SPTK_TRY(apply_inverse<T>(c, V, r0, r1, An, w.partial.as<double>(),
                                      last ? pdot : nullptr, &nb));
            reduce_partials_kernel<<<(R + 7) / 8, 256, 0, c.s>>>(w.partial.as<double>(), nb, R,
                                                                colsq);
            count_launch();
            if (last) {
                reduce_partials_kernel<<<(R + 7) / 8, 256, 0, c.s>>>(pdot, nb, R, colsq + R);
                count_launch();
            }
            SPTK_CUDA(cudaGetLastError());
        } else {
            SPTK_CUDA(cudaMemsetAsync(colsq, 0, sizeof(double) * 2 * R, c.s));
        }
        if (multi) SPTK_TRY(comm_allreduce_f64(c.comm, colsq, last ? 2 * R : R, c.s));
        normalize_kernel<T><<<grid_for(std::max<int64_t>(rows, 1) * R), 256, 0, c.s>>>(
            An, r0, r1, R, (int)c.Rl, colsq, lam);
        count_launch();
        SPTK_CUDA(cudaGetLastError());
        // G_n = sum over ranks of the Gram matrix of each rank's own normalised
        // rows (R x R all-reduce), so the next mode's Cholesky can run on the
        // side stream while the rows are being broadcast
        SPTK_TRY(gram<T>(c, n, nullptr, r0, r1));
        if (multi) SPTK_TRY(comm_allreduce_f64(c.comm, w.G.as<double>() + (int64_t)n * R * R,
                                               (int64_t)R * R, c.s));
        SPTK_CUDA(cudaEventRecord(w.ev_gram, c.s));
        if (multi) SPTK_TRY(comm_bcast_rows(c.comm, An, c.R, t->dtype, c.b[n].data(), c.s));
    }
    fit_kernel<<<1, 256, 0, c.s>>>(colsq + R, lam, w.G.as<double>(), N, R, t->normX2, scal);
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    double h[9];
    SPTK_CUDA(cudaMemcpyAsync(h, scal, sizeof(double) * 9, cudaMemcpyDeviceToHost, c.s));
    SPTK_CUDA(cudaStreamSynchronize(c.s));
    *fit_host = h[0];
    int st;
    memcpy(&st, &h[8], sizeof(int));
    *status_host = st;
    return SPTK_OK;
}

// Everything a captured iteration graph reads (kernel arguments are baked into
// the graph): buffer addresses, cache keys, the stream, the options generation.
static std::vector<uint64_t> graph_key(AlsCtx &c, cudaStream_t s) {
    sptk_tensor t = c.t;
    ALSWork &w = t->als;
    std::vector<uint64_t> k;
    auto add = [&](uint64_t v) { k.push_back(v); };
    auto addp = [&](const void *p) { k.push_back((uint64_t)(uintptr_t)p); };
    add((uint64_t)c.R);
    add((uint64_t)c.Rl);
    add((uint64_t)t->N);
    add((uint64_t)t->dtype);
    addp(s);
    addp(c.comm);
    add(options_generation());
    add(c.sym_iter);
    add(c.prezero);
    for (int n = 0; n < t->N; ++n) add(c.pz[n]);
    add(c.copy_fit);
    for (const void *p : c.vbuf) addp(p);
    add((uint64_t)c.part_stride);
    add((uint64_t)c.nb_apply);
    add((uint64_t)c.nblocks);
    add((uint64_t)c.nb_row);
    for (void *p : c.A) addp(p);
    const void *bufs[] = {w.V.p, w.G.p, w.L.p, w.partial.p, w.colsq.p, w.lam.p, w.scal.p,
                          w.trace.p, w.gpart.p, w.scl.p, (const void *)w.side,
                          (const void *)w.ev_gram, (const void *)w.ev_inv, (const void *)w.hres,
                          t->rec.p, t->det_row.p, t->det_part.p, t->rowmax_dev.p};
    for (const void *p : bufs) addp(p);
    for (int m = 0; m < t->N; ++m) {
        addp(t->perm[m].p);
        addp(t->rowptr[m].p);
        addp(t->srec[m].p);
        addp(t->wrow[m].p);
        addp(t->soff[m].p);
        add(t->has_srec[m]);
        add((uint64_t)t->copy_sec[m]);
        add((uint64_t)t->copy_p0[m]);
        add((uint64_t)t->copy_p1[m]);
        add(t->copy_rowrec[m]);
        add((uint64_t)t->row_max[m]);
        for (int i = 0; i < 3; ++i) add((uint64_t)t->wrow_key[m][i]);
        for (int i = 0; i < 4; ++i) add((uint64_t)t->soff_key[m][i]);
    }
    if (c.comm) {
        addp(c.comm->sym.local);
        add((uint64_t)c.comm->sym.exchange);
        for (size_t o : c.off) add(o);
        for (const auto &b : c.b)
            for (int64_t x : b) add((uint64_t)x);
    }
    return k;
}

// Row stride of CP-ALS's factors for rank Rl (DESIGN.md §4 "odd R"): the
// MTTKRP's lanes load 32-byte vectors (V = 32 / sizeof(T) columns), which a
// row of Rl columns cannot use unless Rl is a multiple of V (or a power of two
// below it) -- R = 17 in fp64 ran 4.8x slower than R = 16 on 8-byte lanes.
// Other ranks run on factors padded with zero columns to the next multiple of
// min(V, pow2ceil(Rl)); the pad columns stay exactly zero through every step
// (Gamma's pad block is the identity, lambda_pad = 0, scale_pad = 0), so the
// decomposition is the rank-Rl one.  Option pad_rank = 0: stride Rl.
template <typename T>
static int64_t padded_rank(int64_t Rl) {
    const int64_t V = 32 / (int64_t)sizeof(T);
    int64_t p2 = 1;
    while (p2 < Rl) p2 <<= 1;
    if (!opt(OPT_PAD_RANK) || Rl % V == 0 || p2 == Rl) return Rl;
    // pad_rank > 1: pad to a multiple of that many columns instead (A/B)
    const int64_t q = std::max<int64_t>(std::min(V, p2), opt(OPT_PAD_RANK));
    return std::min<int64_t>((Rl + q - 1) / q * q, kMaxAlsRank);
}

template <typename T>
static sptk_status cp_als_impl(sptk_tensor t, int64_t Rl, int max_iters, double tol, uint64_t seed,
                               const void *const *init, void *const *factors_out,
                               void *lambda_out, double *fit_out, int *iters_out,
                               double *fit_trace, sptk_comm comm, cudaStream_t s) {
    const int N = t->N;
    const size_t es = sizeof(T);
    // R: the factors' row stride inside the iteration (padded rank), Rl the rank
    const int64_t R = padded_rank<T>(Rl);
    const bool padded = R != Rl;
    ALSWork &w = t->als;
    int64_t Imax = 0, Isum = 0;
    for (int m = 0; m < N; ++m) {
        Imax = std::max(Imax, t->dims[m]);
        Isum += t->dims[m];
    }
    AlsCtx c;
    c.t = t;
    c.R = R;
    c.Rl = Rl;
    c.s = s;
    c.comm = comm;
    // enough blocks to cover tall factors (LBNL's 868K-row mode) in one wave
    // set; R x R partials are capped harder at large R
    c.nblocks = dev_sms() * (R <= 32 ? 8 : 2);
    c.nb_row = dev_sms() * 8;
    SPTK_TRY(w.V.reserve(es * Imax * R));
    SPTK_TRY(w.G.reserve(sizeof(double) * N * R * R));
    SPTK_TRY(w.L.reserve(sizeof(double) * R * R));  // Gamma^{-1}
    // R-vector partials: one per block (row-parallel kernel) or per 64-row tile
    const int64_t nparts_max = std::max<int64_t>((Imax + kTB - 1) / kTB, c.nb_row);
    c.part_stride = (size_t)nparts_max * R;
    SPTK_TRY(w.partial.reserve(sizeof(double) * std::max<size_t>((size_t)c.nblocks * R * R,
                                                                2 * c.part_stride)));
    SPTK_TRY(w.colsq.reserve(sizeof(double) * (2 * R + R * R)));
    SPTK_TRY(w.lam.reserve(sizeof(double) * R));
    SPTK_TRY(w.scal.reserve(sizeof(double) * 16));
    SPTK_TRY(w.trace.reserve(sizeof(double) * (size_t)std::max(max_iters, 1)));
    SPTK_TRY(w.lamT.reserve(es * R));
    c.nb_apply = c.nblocks * apply_nb_mult();
    SPTK_TRY(w.gpart.reserve(sizeof(double) * (size_t)c.nb_apply * R * R));
    SPTK_TRY(w.scl.reserve(sizeof(double) * ((size_t)N * R + (size_t)R * R + R + 1)));
    if (!w.hres) SPTK_CUDA(cudaMallocHost(&w.hres, sizeof(double) * 16));
    if (!w.side) {
        // highest priority on tensors with long MTTKRPs: the one-block inverse
        // is then scheduled at the next block retirement of the MTTKRP it
        // overlaps (at default priority it waited for the MTTKRP's last wave:
        // LBNL 0.583 -> 0.516 ms/iter); on tiny tensors, where every kernel is
        // a few us, the prioritised stream measured slower (C1 0.075 -> 0.113)
        int lo = 0, hi = 0;
        SPTK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        const int64_t sp = opt(OPT_SIDE_PRIO);
        const bool prio = sp == 1 || (sp < 0 && t->P >= ((int64_t)1 << 20));
        SPTK_CUDA(cudaStreamCreateWithPriority(&w.side, cudaStreamNonBlocking, prio ? hi : 0));
        SPTK_CUDA(cudaEventCreateWithFlags(&w.ev_gram, cudaEventDisableTiming));
        SPTK_CUDA(cudaEventCreateWithFlags(&w.ev_inv, cudaEventDisableTiming));
        SPTK_CUDA(cudaEventCreateWithFlags(&w.ev_join, cudaEventDisableTiming));
        for (cudaEvent_t &e : w.ev_zero) SPTK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    SPTK_CUDA(cudaMemsetAsync(w.scal.p, 0, sizeof(double) * 16, s));
    w.R = R;

    // factor storage: caller's device buffers, or staging for host buffers;
    // the sharded deferred path keeps the replicas in the communicator's
    // symmetric buffer (other ranks store rows into it) and copies out at the end
    const bool multi = sharded(comm);
    c.sym_iter = multi && deferred_norm(R);
    std::vector<bool> host_out(N);
    bool any_host = false;
    for (int m = 0; m < N; ++m) {  // padded: staged, copied out with stride Rl
        host_out[m] = c.sym_iter || padded || !is_device_ptr(factors_out[m]);
        any_host = any_host || padded || !is_device_ptr(factors_out[m]);
    }
    c.A.resize(N);
    if (c.sym_iter) {
        c.off.assign(N, 0);
        size_t bytes = 0;
        for (int m = 0; m < N; ++m) {
            c.off[m] = bytes;
            bytes += (es * t->dims[m] * R + 255) / 256 * 256;
        }
        SPTK_TRY(comm_sym_reserve(comm, bytes, s));
        for (int m = 0; m < N; ++m) c.A[m] = static_cast<char *>(comm->sym.local) + c.off[m];
    } else {
        if (any_host) SPTK_TRY(w.stage.reserve(es * Isum * R));
        char *st = w.stage.as<char>();
        for (int m = 0; m < N; ++m) {
            if (host_out[m]) {
                c.A[m] = st;
                st += es * t->dims[m] * R;
            } else {
                c.A[m] = factors_out[m];
            }
        }
    }
    for (int m = 0; m < N; ++m) {
        const size_t bytes = es * t->dims[m] * R;
        if (!init || !init[m]) {
            init_factor_kernel<T><<<grid_for(t->dims[m] * R), 256, 0, s>>>(
                seed, (uint64_t)(N + 1 + m), t->dims[m], (int)Rl, (int)R,
                static_cast<T *>(c.A[m]));
            count_launch();
            SPTK_CUDA(cudaGetLastError());
        } else if (padded) {  // rows of Rl into rows of R, pad columns zero
            SPTK_CUDA(cudaMemsetAsync(c.A[m], 0, bytes, s));
            if (t->dims[m] > 0)
                SPTK_CUDA(cudaMemcpy2DAsync(c.A[m], es * R, init[m], es * Rl, es * Rl, t->dims[m],
                                            cudaMemcpyDefault, s));
        } else if (init[m] != c.A[m]) {
            SPTK_CUDA(cudaMemcpyAsync(c.A[m], init[m], bytes, cudaMemcpyDefault, s));
        }
    }
    for (int m = 0; m < N; ++m)
        if (!t->has_perm[m]) SPTK_TRY(build_perm_mode(t, m, s));
    if (multi) {
        c.b.assign(N, std::vector<int64_t>(comm->nranks + 1));
        for (int m = 0; m < N; ++m) {
            SPTK_TRY(host_rowptr(t, m, s));
            SPTK_TRY(sptk_partition_rows(t->host_rowptr[m].data(), t->dims[m], comm->nranks,
                                         c.b[m].data()));
        }
    }
    for (int m = 0; m < N; ++m) SPTK_TRY(gram<T>(c, m));
    // pre-zeroed MTTKRP output buffers (AlsCtx::prezero): 2 for even N, a third
    // for the last mode of odd N; buffer b holds the longest of its modes
    c.prezero = !multi && opt(OPT_PREZERO) != 0;
    if (c.prezero) {
        int64_t rows[3] = {0, 0, 0};
        for (int n = 0; n < N; ++n) {
            c.vb[n] = (N % 2 == 1 && n == N - 1) ? 2 : n % 2;
            rows[c.vb[n]] = std::max(rows[c.vb[n]], t->dims[n]);
        }
        c.vbuf[0] = w.V.p;
        if (w.V2.reserve(es * std::max<int64_t>(rows[1], 1) * R) != SPTK_OK ||
            (rows[2] && w.V3.reserve(es * rows[2] * R) != SPTK_OK)) {
            set_error("");  // no room: zero inside each MTTKRP launch instead
            c.prezero = false;
        }
        c.vbuf[1] = w.V2.p;
        c.vbuf[2] = rows[2] ? w.V3.p : nullptr;
        for (int n = 0; n < N && c.prezero; ++n) {
            const int p = (n + N - 1) % N;  // its apply has released buffer vb[p]
            int k = 1;
            while (c.vb[(p + k) % N] != c.vb[p]) ++k;
            const int m = (p + k) % N;      // the next mode writing that buffer
            c.znext[n] = m;
            c.zsame[m] = p == N - 1 || p + k <= N - 1;
        }
        // only outputs of >= 256 MB (Delicious' 17M- and 2.5M-row modes: -1 %);
        // below that an in-launch zero costs less than a side-stream memset
        // and its dependency (LBNL's 111 MB mode: +1.2 % pre-zeroed, C1 +4 %,
        // profiles/r02/s2/ab_glue_s13.log)
        bool any = false;
        for (int n = 0; n < N; ++n) {
            c.pz[n] = opt(OPT_PREZERO) == 2 ||
                      es * (size_t)t->dims[n] * R >= ((size_t)std::max<int64_t>(opt(OPT_PREZERO_MB), 0) << 20);
            any = any || c.pz[n];
        }
        c.prezero = c.prezero && any;
        for (int b = 0; b < 3 && c.prezero; ++b)
            if (rows[b]) SPTK_CUDA(cudaMemsetAsync(c.vbuf[b], 0, es * rows[b] * R, s));
    }
    // deferred normalisation state (single GPU, R <= 32): all scales 1, and the
    // first MTTKRP's column weights 1
    const bool deferred = (!multi || c.sym_iter) && deferred_norm(R);
    // the fused deferred iteration zeroes a pre-zeroed output from extra
    // blocks of the previous mode's apply instead of a side-stream memset
    c.zapply = c.prezero && deferred && !multi && opt(OPT_ZERO_IN_APPLY) != 0;
    if (deferred) {
        double *s_all = w.scl.as<double>();
        fill_f64_kernel<<<(unsigned)((N * R + 255) / 256), 256, 0, s>>>(s_all, N * (int)R, 1.0);
        T *scale = reinterpret_cast<T *>(s_all + (size_t)N * R + (size_t)R * R);
        fill_kernel<T><<<1, 128, 0, s>>>(scale, (int)R, T(1));  // no host staging, no sync
        SPTK_CUDA(cudaMemsetAsync(scale + R, 0, sizeof(int), s));  // apply_gram's block counter
        count_launch(2);
        SPTK_CUDA(cudaGetLastError());
    }

    double fit = 0.0, fit_prev = 0.0;
    int it = 0;
    sptk_status st = SPTK_OK;
    // Single GPU: after one eager iteration (which builds every cache the
    // launches read), capture one iteration -- both streams, ~4N+2 kernels and
    // the fit copy -- into a CUDA graph and replay it.  Not while profiling
    // (kernel-span events cannot be timed inside graphs) or for < 4 iterations.
    bool use_graph = (!multi || c.sym_iter) && !profile().on && max_iters >= 4 && !opt(OPT_NO_GRAPH);
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t launches_per_iter = 0;
    bool fast_done = false;
    if (use_graph && tol <= 0.0) {
        c.copy_fit = c.sym_iter;  // single GPU: no per-iteration copy (the sharded one keeps its own)
        // No convergence test.  If the previous call captured this same
        // iteration (same buffers, caches, stream and options: graph_key), its
        // graph is replayed from iteration 0.  Otherwise iteration 0 runs
        // eagerly (its host side builds every cache the launches read) WITHOUT
        // waiting for it, iteration 1 is captured while the GPU runs it, and the
        // graph is replayed for the rest back to back.  One host
        // synchronisation per call; the fits come from the device-side history.
        // (C1 at 20 iterations per call: 0.084 -> 0.069 ms/iter for the
        // overlapped capture.)
        int k0 = 0;
        if (!(w.exec && w.graph_key == graph_key(c, s))) {
            w.drop_graph();
            st = enqueue_iteration<T>(c);
            const int64_t l1 = profile().launches;
            bool ok = st == SPTK_OK &&
                      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            sptk_status est = ok ? enqueue_iteration<T>(c) : SPTK_ECUDA;
            if (st == SPTK_OK) {
                cudaGraph_t g = nullptr;
                const bool ended = ok && cudaStreamEndCapture(s, &g) == cudaSuccess;
                ok = ok && est == SPTK_OK && ended && g &&
                     cudaGraphInstantiate(&w.exec, g, 0) == cudaSuccess;
                w.graph = g;
                w.launches_per_iter = profile().launches - l1;
                if (ok) {
                    w.graph_key = graph_key(c, s);
                } else {  // eager launches for the rest of the call
                    cudaGetLastError();
                    set_error("");
                    w.drop_graph();
                    profile().launches = l1;
                }
            }
            k0 = 1;
        }
        for (int k = k0; k < max_iters && st == SPTK_OK; ++k) {
            if (w.exec) {
                profile().launches += w.launches_per_iter;
                if (cudaGraphLaunch(w.exec, s) != cudaSuccess)
                    st = cuda_fail(cudaGetLastError(), "cudaGraphLaunch(ALS iteration)");
            } else {
                st = enqueue_iteration<T>(c);
            }
        }
        if (st == SPTK_OK && !c.copy_fit &&
            cudaMemcpyAsync(w.hres, w.scal.p, sizeof(double) * 9, cudaMemcpyDeviceToHost, s) !=
                cudaSuccess)
            st = cuda_fail(cudaGetLastError(), "fit/status copy");
        int bad = 0;
        if (st == SPTK_OK) st = complete_iteration(c, &fit, &bad);
        if (st == SPTK_OK) {
            std::vector<double> hist((size_t)max_iters);
            SPTK_CUDA(cudaMemcpy(hist.data(), w.trace.p, sizeof(double) * max_iters,
                                 cudaMemcpyDeviceToHost));
            if (bad) st = fail(SPTK_ESINGULAR, "Gamma is singular after the ridge retry");
            for (int k = 0; k < max_iters && st == SPTK_OK; ++k)
                if (!std::isfinite(hist[k]))
                    st = fail(SPTK_ESINGULAR, "non-finite fit: Gamma numerically singular");
            if (fit_trace)
                for (int k = 0; k < max_iters; ++k) fit_trace[k] = hist[k];
            fit = hist[max_iters - 1];
        }
        it = max_iters;
        fast_done = true;  // the loop below has nothing left to run
    }
    for (it = fast_done ? max_iters : 0; it < max_iters; ++it) {
        int bad = 0;
        if (use_graph && it >= 1) {
            if (!exec) {
                const int64_t l0 = profile().launches;
                bool ok = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
                sptk_status est = ok ? enqueue_iteration<T>(c) : SPTK_ECUDA;
                cudaGraph_t g = nullptr;
                const bool ended = cudaStreamEndCapture(s, &g) == cudaSuccess;
                ok = ok && est == SPTK_OK && ended && g &&
                     cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
                graph = g;
                launches_per_iter = profile().launches - l0;
                if (!ok) {  // fall back to eager launches for the rest of the call
                    cudaGetLastError();
                    set_error("");
                    if (exec) cudaGraphExecDestroy(exec);
                    exec = nullptr;
                    use_graph = false;
                    profile().launches = l0;
                    st = enqueue_iteration<T>(c);
                    if (st == SPTK_OK) st = complete_iteration(c, &fit, &bad);
                    if (st != SPTK_OK) break;
                    goto have_fit;
                }
            } else {
                profile().launches += launches_per_iter;
            }
            if (cudaGraphLaunch(exec, s) != cudaSuccess) {
                st = cuda_fail(cudaGetLastError(), "cudaGraphLaunch(ALS iteration)");
                break;
            }
            if (tol <= 0.0 && it >= 2) {
                // no convergence test: replay the remaining iterations back to
                // back (no host round trip per iteration); the fits are taken
                // from the device-side history afterwards, the Cholesky status
                // (sticky) once at the end
                for (int k = it + 1; k < max_iters; ++k) {
                    profile().launches += launches_per_iter;
                    if (cudaGraphLaunch(exec, s) != cudaSuccess) {
                        st = cuda_fail(cudaGetLastError(), "cudaGraphLaunch(ALS iteration)");
                        break;
                    }
                }
                if (st != SPTK_OK) break;
                st = complete_iteration(c, &fit, &bad);
                if (st != SPTK_OK) break;
                std::vector<double> hist((size_t)max_iters);
                SPTK_CUDA(cudaMemcpy(hist.data(), w.trace.p, sizeof(double) * max_iters,
                                     cudaMemcpyDeviceToHost));
                if (bad) {
                    st = fail(SPTK_ESINGULAR, "Gamma is singular after the ridge retry");
                    break;
                }
                if (fit_trace)
                    for (int k = it; k < max_iters; ++k) fit_trace[k] = hist[k];
                fit = hist[max_iters - 1];
                it = max_iters;
                for (int k = 0; k < max_iters; ++k)
                    if (!std::isfinite(hist[k])) {
                        st = fail(SPTK_ESINGULAR, "non-finite fit: Gamma numerically singular");
                        break;
                    }
                break;
            }
            st = complete_iteration(c, &fit, &bad);
        } else {
            st = als_iteration<T>(c, &fit, &bad);
        }
        if (st != SPTK_OK) break;
    have_fit:
        if (bad) {
            st = fail(SPTK_ESINGULAR, "Gamma is singular after the ridge retry");
            break;
        }
        if (!std::isfinite(fit)) {  // a tiny positive pivot can still overflow Gamma^{-1}
            st = fail(SPTK_ESINGULAR, "non-finite fit: Gamma numerically singular");
            break;
        }
        if (fit_trace) fit_trace[it] = fit;
        if (tol > 0.0 && fabs(fit - fit_prev) < tol) {
            ++it;
            break;
        }
        fit_prev = fit;
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (deferred && it > 0) {  // apply the deferred column normalisation once
        for (int m = 0; m < N; ++m) {
            scale_columns_kernel<T><<<grid_for(t->dims[m] * R), 256, 0, s>>>(
                static_cast<T *>(c.A[m]), t->dims[m], (int)R, w.scl.as<double>() + (size_t)m * R);
            count_launch();
        }
        SPTK_CUDA(cudaGetLastError());
    }
    if (fit_out) *fit_out = fit;
    if (iters_out) *iters_out = it;
    if (st != SPTK_OK) return st;
    if (max_iters == 0) {  // lambda = ones
        SPTK_CUDA(cudaMemsetAsync(w.lam.p, 0, sizeof(double) * R, s));
        std::vector<double> ones(R, 1.0);
        SPTK_CUDA(cudaMemcpyAsync(w.lam.p, ones.data(), sizeof(double) * R,
                                  cudaMemcpyHostToDevice, s));
        SPTK_CUDA(cudaStreamSynchronize(s));
    }
    for (int m = 0; m < N; ++m)
        if (host_out[m] && padded && t->dims[m] > 0)  // drop the pad columns
            SPTK_CUDA(cudaMemcpy2DAsync(factors_out[m], es * Rl, c.A[m], es * R, es * Rl,
                                        t->dims[m], cudaMemcpyDefault, s));
        else if (host_out[m])
            SPTK_CUDA(cudaMemcpyAsync(factors_out[m], c.A[m], es * t->dims[m] * R,
                                      cudaMemcpyDefault, s));
    if (lambda_out) {
        cast_kernel<T><<<(unsigned)((Rl + 127) / 128), 128, 0, s>>>(w.lam.as<double>(), (int)Rl,
                                                                   w.lamT.as<T>());
        count_launch();
        SPTK_CUDA(cudaGetLastError());
        SPTK_CUDA(cudaMemcpyAsync(lambda_out, w.lamT.p, es * Rl, cudaMemcpyDefault, s));
    }
    if (any_host || (lambda_out && !is_device_ptr(lambda_out)))
        SPTK_CUDA(cudaStreamSynchronize(s));
    return SPTK_OK;
}

}  // namespace sptk

using namespace sptk;

extern "C" sptk_status sptk_cp_als(sptk_tensor t, int64_t R, int max_iters, double tol,
                                   uint64_t seed, const void *const *init,
                                   void *const *factors_out, void *lambda_out, double *fit_out,
                                   int *iters_out, double *fit_trace, sptk_comm comm,
                                   void *stream) {
    if (!t) return fail(SPTK_EINVAL, "null tensor handle");
    if (t->poisoned) return fail(SPTK_ECUDA, "tensor handle poisoned by an earlier CUDA error");
    if (t->N < 2) return fail(SPTK_EUNSUPPORTED, "cp_als needs nmodes >= 2");
    if (R < 1) return fail(SPTK_EINVAL, "R must be >= 1");
    if (R > kMaxAlsRank) return fail(SPTK_EUNSUPPORTED, "cp_als supports R <= 128");
    if (max_iters < 0) return fail(SPTK_EINVAL, "max_iters < 0");
    if (!factors_out) return fail(SPTK_EINVAL, "factors_out is NULL");
    for (int m = 0; m < t->N; ++m)
        if (!factors_out[m]) return fail(SPTK_EINVAL, "factors_out[m] is NULL");
    if (!(t->normX2 > 0.0)) return fail(SPTK_EZERONORM, "||X|| = 0");
    cudaStream_t s = (cudaStream_t)stream;
    // Gamma^{-1} staging can exceed the 48 KB default shared memory for R > 64
    // the attribute is per device (context): set it once for each device used,
    // under a mutex (several host threads may drive several GPUs)
    static std::mutex attr_mu;
    static bool attr_done[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64)
        return fail(SPTK_ECUDA, "cudaGetDevice failed");
    {
    std::lock_guard<std::mutex> attr_lk(attr_mu);
    if (!attr_done[dev]) {
        cudaFuncSetAttribute(apply_inv_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(apply_inv_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(gj_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(apply_gram_kernel<double, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(apply_gram_kernel<double, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(apply_gram_kernel<float, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(apply_gram_kernel<float, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(finish_kernel<double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(finish_kernel<double, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(finish_kernel<float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(finish_kernel<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_done[dev] = true;
    }
    }
    sptk_status st =
        t->dtype == SPTK_F64
            ? cp_als_impl<double>(t, R, max_iters, tol, seed, init, factors_out, lambda_out,
                                  fit_out, iters_out, fit_trace, comm, s)
            : cp_als_impl<float>(t, R, max_iters, tol, seed, init, factors_out, lambda_out,
                                 fit_out, iters_out, fit_trace, comm, s);
    if (st == SPTK_ECUDA) t->poisoned = true;
    return st;
}
