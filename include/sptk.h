/*
 * sptk.h -- C ABI of the B200-native sparse MTTKRP / CP-ALS library
 * (libsptk.so), the hot path of arXiv 1809.09175 (GenTen, "Sparse Tensor
 * Decomposition Algorithms for Performance Portability").
 *
 * Citations: P:NNN = line of the paper text (reference PAPER.md), with the
 * section / equation / figure named; S:NNN = line of the CPU-program SPEC.md
 * (interfaces only).  Design and readings: DESIGN.md.
 *
 * Conventions (all calls):
 *  - Every call returns sptk_status (0 = SPTK_OK).  On error a thread-local
 *    message is available from sptk_last_error().  Precondition violations
 *    never abort.  After SPTK_ECUDA the handle is poisoned (every later call
 *    on it returns SPTK_ECUDA).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Device work is stream-ordered on it; calls return without
 *    synchronising unless stated.
 *  - "device or host" pointers are classified with cudaPointerGetAttributes:
 *    host (pageable or pinned) memory is staged through device buffers inside
 *    the call (that call then synchronises `stream`).
 *  - Factor matrices are row-major I_m x R ("row-wise memory
 *    layout"), element type = the tensor's dtype, caller-owned.
 *  - Limits: 1 <= nmodes <= 6 (cp_als: >= 2); 1 <= dims[m] < 2^32;
 *    0 <= nnz <= 2^32 - 4096 (32-bit positions); R >= 1 (cp_als: R <= 128).
 *    Indices are 0-based (Z2).
 *  - Concurrency: the tensor's values never change after create, but a
 *    handle keeps per-handle caches (permuted copies, worker start rows,
 *    scratch, ALS workspace) that MTTKRP / CP-ALS calls may (re)build, so
 *    calls on ONE handle must be serialised (one host thread at a time; any
 *    streams).  Different handles are independent.
 */
#ifndef SPTK_H
#define SPTK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { SPTK_F32 = 1, SPTK_F64 = 2 } sptk_dtype;

/* sptk_sptensor_create flags */
enum {
    SPTK_CREATE_DEFAULT = 0,
    /* Keep the paper's traversal literally: MTTKRP reads perm_n[i] and then
     * gathers record perm_n[i] (§5, Fig. mttkrp_perm).  Without
     * this flag build_perm(n) also materialises the records in perm_n order
     * (one gather at build time) and MTTKRP streams that copy instead of
     * gathering through the permutation -- same visiting order, same write
     * discipline, same result; DESIGN.md §4 gives the measured reason (a
     * random 32 B record read costs a 128 B HBM line on B200).  If the copy
     * cannot be allocated the mode silently uses the perm-gather traversal. */
    SPTK_CREATE_PERM_GATHER = 2,
    /* Bit-reproducible MTTKRP (and hence CP-ALS): the rows a worker shares
     * with its neighbours are not flushed with atomics but written to a
     * scratch slot and summed in worker order by a fix-up kernel (SURVEY
     * §8(f) NEXT-3).  Supported on the permuted-copy fast path (N in 3..5,
     * any R, element-aligned factors; not with SPTK_CREATE_PERM_GATHER);
     * other calls on such a tensor return SPTK_EUNSUPPORTED. */
    SPTK_CREATE_DETERMINISTIC = 4,
    /* Duplicate-coordinate policy (default: duplicates kept, MTTKRP
     * is linear in X).  DUP_SUM merges equal coordinates into one nonzero at
     * the position of the first occurrence with the values summed in storage
     * order (the tensor's nnz shrinks accordingly); DUP_ERROR fails with
     * SPTK_EDUP if any coordinate repeats.  Both use an on-GPU lexicographic
     * stable sort (one radix sort per mode, last mode first). */
    SPTK_CREATE_DUP_SUM = 8,
    SPTK_CREATE_DUP_ERROR = 16
};
typedef enum { SPTK_IDX_I64 = 1, SPTK_IDX_U32 = 2 } sptk_idx_type;

typedef enum {
    SPTK_OK = 0,
    SPTK_EINVAL = 1,       /* bad argument (null pointer, dtype mismatch, shape) */
    SPTK_ERANGE = 2,       /* a coordinate >= dims[m] (or < 0) */
    SPTK_EDUP = 3,         /* duplicate coordinate under SPTK_CREATE_DUP_ERROR */
    SPTK_ENOPERM = 4,      /* sptk_build_perm(mode) has not been run */
    SPTK_ENOMEM = 5,       /* device allocation failed */
    SPTK_ECUDA = 6,        /* CUDA runtime error (handle poisoned) */
    SPTK_ENCCL = 7,        /* NCCL missing or failed */
    SPTK_ESINGULAR = 8,    /* Gamma not positive definite after the ridge retry */
    SPTK_EZERONORM = 9,    /* ||X|| = 0 in cp_als */
    SPTK_EUNSUPPORTED = 10 /* outside the limits above */
} sptk_status;

typedef struct sptk_tensor_s *sptk_tensor; /* opaque; owns device records, perms, rowptrs */
typedef struct sptk_comm_s *sptk_comm;     /* opaque; owns an ncclComm_t */

/* Library version string, e.g. "sptk 0.1 sm_100a". */
const char *sptk_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char *sptk_last_error(void);

/* ---------------------------------------------------------------- tensor */

/* Create a COO sparse tensor ("a P-vector of real values and a
 * P x d vector of coordinates"; COO).
 *   nmodes   d (1..6)
 *   dims     host int64[nmodes], I_m >= 1
 *   nnz      P >= 0 (0 = empty tensor)
 *   idx      device or host, nnz x nmodes row-major, 0-based; element type
 *            itype (int64 or uint32).  May be NULL iff nnz == 0.
 *   vals     device or host, nnz values of `dtype`.  NULL iff nnz == 0.
 *   flags    SPTK_CREATE_DEFAULT, or SPTK_CREATE_PERM_GATHER or
 *            SPTK_CREATE_DETERMINISTIC (mutually exclusive), optionally OR-ed
 *            with one of SPTK_CREATE_DUP_SUM / SPTK_CREATE_DUP_ERROR.
 *            Duplicate coordinates are always allowed (MTTKRP is linear in X;
 *            DESIGN.md Z3).
 *   out      receives the handle
 * Copies the input into packed device records {value, idx[d]} (16 or 32 B)
 * after validating 0 <= idx < dims (SPTK_ERANGE otherwise) -- the caller may
 * free its buffers when the call returns.  Also caches ||X||^2.  Synchronises
 * `stream` once (reading the validation flag). */
sptk_status sptk_sptensor_create(int nmodes, const int64_t *dims, int64_t nnz,
                                 const void *idx, sptk_idx_type itype, const void *vals,
                                 sptk_dtype dtype, unsigned flags, void *stream,
                                 sptk_tensor *out);

/* Free all device memory owned by the handle (NULL is a no-op). */
sptk_status sptk_sptensor_destroy(sptk_tensor t);

/* Shape query: any output pointer may be NULL; dims receives nmodes values. */
sptk_status sptk_sptensor_info(sptk_tensor t, int *nmodes, int64_t *dims, int64_t *nnz,
                               sptk_dtype *dtype);

/* Device bytes owned by the handle (records + perms + rowptrs + permuted
 * copies + workspace). */
sptk_status sptk_sptensor_device_bytes(sptk_tensor t, int64_t *bytes);

/* Declare that this handle serves rank `rank` of `nranks` row-range shards
 * (rank g owns rows [b_g, b_{g+1}) of every mode, b =
 * sptk_partition_rows over rowptr_n).  The permuted copies built afterwards
 * (build_perm, or lazily by the first MTTKRP of a mode) then hold only this
 * rank's positions: 1/nranks of the copy memory per rank.  MTTKRP calls whose
 * rows fall outside the shard stay correct (they gather through perm_n, the
 * paper's traversal).  Existing copies are dropped.  nranks = 1 restores the
 * whole-tensor copies.  Errors: SPTK_EINVAL for rank outside [0, nranks). */
sptk_status sptk_sptensor_set_shard(sptk_tensor t, int nranks, int rank);

/* Build the mode-`mode` permutation (mode = -1: all modes).  P:513-515 (§5
 * "Permutation approach"): "a permutation array for each mode that sorts the
 * tensor nonzeros in increasing index along that mode"; the sort is STABLE
 * (ties keep storage order), so the permutation is unique.
 * Also builds rowptr_n[I_n+1] (start of each mode-n row in permuted order)
 * and, unless the tensor was created with SPTK_CREATE_PERM_GATHER, the
 * records in perm_n order (rec_bytes x nnz).  On-GPU LSD radix sort;
 * temporary device memory ~16 B x nnz. */
sptk_status sptk_build_perm(sptk_tensor t, int mode, void *stream);

/* Copy perm_n (uint32[nnz]) / rowptr_n (uint32[I_n + 1]) to `out` (device or
 * host).  SPTK_ENOPERM if build_perm(mode) has not run. */
sptk_status sptk_get_perm(sptk_tensor t, int mode, uint32_t *out, void *stream);
sptk_status sptk_get_rowptr(sptk_tensor t, int mode, uint32_t *out, void *stream);

/* ---------------------------------------------------------------- MTTKRP */

/* Mode-n MTTKRP, Eq. (2):
 *   out(k, j) = lambda_j * sum_{i : l_in = k} x_i * prod_{m != n} A_m(l_im, j)
 * computed by permuted traversal (§5, Fig. mttkrp_perm): nonzeros
 * are visited in perm_n order (through perm_n, or streaming the permuted copy
 * of the records), a row is accumulated in registers and written
 * when the mode-n index changes -- plain store for rows interior to a
 * worker's block, atomic add for a block's first/last row.  On
 * long balanced rows the B200 slice traversal splits each row's run by the
 * copy's secondary index and adds one partial per (row, slice) atomically
 * (DESIGN.md §4); the result is the same sum.  The first call for a mode may
 * synchronise `stream` once (host copy of rowptr_n for launch decisions);
 * later calls do not, so they can be captured in a CUDA graph.
 *   mode     n in [0, nmodes)
 *   R        rank (columns), >= 1
 *   factors  HOST array of nmodes DEVICE pointers, factors[m] is I_m x R
 *            row-major of the tensor's dtype; factors[mode] is ignored (may
 *            be NULL)
 *   lambda   device R-vector or NULL (= all ones; Z1)
 *   out      device I_n x R, overwritten (rows without nonzeros are exactly 0;
 *            S:239)
 *   comm     NULL: single GPU.  Otherwise each rank computes the rows of its
 *            contiguous row range (sptk_partition_rows over rowptr_n) and the
 *            full `out` is replicated on every rank by NCCL broadcasts.
 * Result equals Eq. (2) up to floating-point summation order (atomics).
 * SPTK_ENOPERM if build_perm(mode) has not run. */
sptk_status sptk_mttkrp(sptk_tensor t, int mode, int64_t R, const void *const *factors,
                        const void *lambda, void *out, sptk_comm comm, void *stream);

/* The paper's atomic-per-nonzero MTTKRP (VerA/VerB, Figs. mttkrp_alg and
 * mttkrp_array): nonzeros in storage order, every
 * contribution added to `out` with atomics.  Same arguments and result as
 * sptk_mttkrp (up to summation order); needs no permutation.
 * Provided for the paper's VerB-vs-VerC comparison. */
sptk_status sptk_mttkrp_atomic(sptk_tensor t, int mode, int64_t R, const void *const *factors,
                               const void *lambda, void *out, void *stream);

/* The per-shard unit of the multi-GPU path: the same computation restricted
 * to output rows [row_begin, row_end) of mode n, i.e. to the permuted
 * positions [rowptr_n[row_begin], rowptr_n[row_end]).  Rows
 * outside the range are not touched; rows inside are overwritten.  Several
 * calls over a partition of [0, I_n) (e.g. sptk_partition_rows) reproduce
 * sptk_mttkrp. */
sptk_status sptk_mttkrp_rows(sptk_tensor t, int mode, int64_t R, const void *const *factors,
                             const void *lambda, void *out, int64_t row_begin, int64_t row_end,
                             void *stream);

/* ---------------------------------------------------------------- CP-ALS */

/* CP-ALS (the paper omits the algorithm and defers to Kolda &
 * Bader): textbook alternating least squares, readings in DESIGN.md §2.
 * For it < max_iters, for n = 0..N-1: V = MTTKRP(n); Gamma = Hadamard of
 * A_m^T A_m (m != n); A_n = V Gamma^{-1} (Gamma SPD: inverse by unpivoted
 * Gauss-Jordan, whose pivots are the squared Cholesky diagonal; a pivot
 * d_j <= 1e-12 Gamma_jj is a failure (numerically singular Gamma, e.g.
 * duplicate components: DESIGN.md §2 Z23); one ridge retry with
 * 1e-12 tr(Gamma)/R, which needs only d_j > 0); lambda = column 2-norms;
 * normalise.  fit = 1 - ||X - M||
 * / ||X|| after each iteration; stop when tol > 0 and |fit - fit_prev| < tol.
 *   init        HOST array of nmodes pointers (device or host) with the
 *               initial factors, or NULL: A_m(r, c) = U[0,1) drawn from the
 *               counter generator of DESIGN.md §3 with seed `seed`
 *               (stream nmodes+1+m, counter r*R+c).  init[m] may equal
 *               factors_out[m] (in place).
 *   factors_out HOST array of nmodes pointers (device or host), I_m x R each
 *   lambda_out  R values (device or host) or NULL
 *   fit_out, iters_out   host scalars or NULL
 *   fit_trace   host double[max_iters] or NULL
 *   comm        NULL or a communicator (row-range sharding of every mode;
 *               factors replicated on all ranks)
 * Any R in 1..128: when R is not a multiple of the 32-byte lane vector the
 * iteration runs on internally zero-padded factors (option pad_rank) and the
 * outputs are the rank-R ones, stride R.  Synchronises `stream` once per
 * iteration (the fit) when tol > 0, once per call otherwise (the fits then
 * come from a device-side history).  Builds missing perms.  Requires nmodes
 * >= 2.  SPTK_EZERONORM if ||X|| = 0; SPTK_ESINGULAR if Gamma stays singular
 * or the fit is not finite. */
sptk_status sptk_cp_als(sptk_tensor t, int64_t R, int max_iters, double tol, uint64_t seed,
                        const void *const *init, void *const *factors_out, void *lambda_out,
                        double *fit_out, int *iters_out, double *fit_trace, sptk_comm comm,
                        void *stream);

/* --------------------------------------------------------- multi-GPU */

/* Fill `id128` (128 bytes, host) with a new NCCL unique id (rank 0 only;
 * broadcast it to the other ranks out of band, e.g. torch.distributed). */
sptk_status sptk_comm_unique_id(void *id128);

/* Create / destroy a communicator over `nranks` processes (one GPU each;
 * the current CUDA device is used).  Collective: every rank must call it.
 * With SPTK_FORCE_SHARDED=1 in the environment a 1-rank communicator still
 * takes the sharded code path (partition, per-rank kernels, NCCL exchange) --
 * used to test that path on a single GPU. */
sptk_status sptk_comm_create(const void *id128, int nranks, int rank, sptk_comm *out);
sptk_status sptk_comm_destroy(sptk_comm c);

/* How a sharded sptk_cp_als (R <= 32) replicates each updated factor's rows
 * (DESIGN.md §7): 2 = NVLS multimem stores and 1 = NVLink peer stores, both
 * issued by the kernel that computes the rows into the communicator's
 * symmetric buffer (ncclMemAlloc + ncclCommWindowRegister); 0 = grouped NCCL
 * broadcasts after it; -1 = not decided yet (no sharded cp_als has run on
 * this communicator).  The mode is the best one every rank supports, capped
 * by the `exchange` option (sptk_set_option). */
sptk_status sptk_comm_exchange(sptk_comm c, int *mode);

/* Host-only (no GPU needed): split rows [0, In) into nranks contiguous ranges
 * of near-equal nonzero counts.  rowptr (host, In+1 entries, non-decreasing,
 * rowptr[0] = 0, rowptr[In] = nnz).  bounds (host, nranks+1): rank g owns rows
 * [bounds[g], bounds[g+1]) and positions [rowptr[bounds[g]],
 * rowptr[bounds[g+1]]).  bounds[g] = min{ r : rowptr[r] >= ceil(g*nnz/nranks) }
 * for 0 < g < nranks, bounds[0] = 0, bounds[nranks] = In. */
sptk_status sptk_partition_rows(const uint32_t *rowptr, int64_t In, int nranks,
                                int64_t *bounds);

/* ---------------------------------------------------------- measurement */

/* When enabled, the library brackets every MTTKRP kernel launch with CUDA
 * events on its launch stream and accumulates the elapsed time (read after
 * the stream is synchronised).  Launch counters count every kernel the
 * library launches.  Not thread-safe; for benchmarking. */
sptk_status sptk_profile_enable(int on);
sptk_status sptk_profile_reset(void);
sptk_status sptk_profile_read(double *mttkrp_ms, int64_t *mttkrp_launches,
                              int64_t *kernel_launches);

/* Tuning knobs of the MTTKRP launch (process-wide; for sweeps): `variant`
 * selects the fast kernel's worker shape on the permuted copy (0 = per-group
 * runs, 1 = warp-cooperative steps; -1 = keep; -2 = automatic, the default:
 * warp-cooperative when rows average >= 64 nonzeros and a warp holds >= 4
 * groups), `run` the nonzeros per
 * worker group (the paper's NZPTM, P:220;
 * rounded up to a multiple of 4; 0 = keep; -2 = adaptive, the default:
 * clamp(positions / (4 waves of workers), 16, 256)).  Initial values come
 * from SPTK_VARIANT / SPTK_RUN. */
sptk_status sptk_set_tuning(int variant, int64_t run);

/* Process-wide options (traversal selection and tuning).
 * Each starts from its default, or from the environment variable SPTK_<NAME>
 * (upper case, integer) if set.  Names and defaults:
 *   run 0 (positions per worker, 0 = adaptive), variant -1 (auto; 0 per-group,
 *   1 warp-cooperative), slice 1 (0 disables the slice traversal, 2 forces
 *   it wherever the permuted copy has a secondary mode),
 *   slice_l2_kb 32768 (L2 window of the slice traversal when the secondary
 *   factor exceeds it), slice_rows 0 (auto), slice_other_first -1 (auto),
 *   rowrec 1, force_v 0 (cap of the lane vector width in elements),
 *   generic 0 (1 forces the generic scalar kernel), debug_dispatch 0,
 *   copy_order 1 (secondary order of the permuted copies: 1 by balance --
 *   the largest other factor for power-law modes, else the shortest one
 *   >= 2048 rows; 2 always the shortest; 0 none, perm_n order), deferred_norm 1,
 *   no_graph 0, gamma_inv_chol 0, use_copy 1 (0: gather the records through
 *   perm_n, the paper's traversal, even where a permuted copy exists),
 *   apply_tile 64, apply_nb_mult 1, tail_rows 8192, apply_wave 1, apply_warp 1
 *   (CP-ALS glue tuning), keep_keys 1 (the sort keys emitted at ingest stay resident after
 *   build_perm while memory allows; 0 releases them), pdl 1 (programmatic dependent launch of the MTTKRP and CP-ALS
 *   kernels: a kernel's launch overlaps its predecessor's tail), exchange -1 (sharded CP-ALS row exchange: -1 best available,
 *   0 NCCL broadcast, 1 peer stores, 2 NVLS multimem; sptk_comm_exchange),
 *   pad_rank 1 (CP-ALS with R not a multiple of the 32-byte lane vector runs
 *   on internally padded factors whose pad columns stay zero -- the output is
 *   the rank-R result; 0: stride R; > 1: pad to a multiple of that many
 *   columns), sort_v1 0 (1: the round-1 radix downsweep, A/B),
 *   prezero 1 (CP-ALS: MTTKRP outputs of >= 256 MB zeroed on a side stream
 *   while the previous mode runs; 2: every output), apply_mma 1 (CP-ALS V Gamma^{-1} and Gram update on the
 *   FP64 tensor cores for R = 8 / 16), gj_warp 1 (one-warp Gauss-Jordan
 *   Gamma^{-1} for R <= 32), side_prio -1 (the CP-ALS side stream at the highest
 *   priority: -1 for >= 2^20 nonzeros, 1 always, 0 never; read when the handle's
 *   stream is created), win 0 (> 0: window-major permuted copies, built at
 *   build_perm, for modes with few rows whose secondary factor spans >= 2 x win
 *   L2 windows; served by the cooperative kernel), slice_fill 6 (the slice
 *   traversal halves its slices until its grid has this many blocks per SM; 0
 *   off), fused_reduce 1 (CP-ALS: a large mode's reductions, finalisation and
 *   fit in one launch), prezero_mb 256 (with prezero 1: the MTTKRP outputs of
 *   at least this many MB are zeroed on the side stream), zero_in_apply 0 (1:
 *   those outputs are zeroed by extra blocks of the previous mode's apply
 *   launch instead of a side-stream memset; deferred single-GPU CP-ALS).
 * Every choice gives the same result up to summation order; options change
 * which kernel computes it.  Not synchronised with calls in flight on other
 * threads.  SPTK_EINVAL for an unknown name. */
sptk_status sptk_set_option(const char *name, int64_t value);
sptk_status sptk_get_option(const char *name, int64_t *value);
/* back to the defaults / environment values */
sptk_status sptk_reset_options(void);
/* The traversal the last MTTKRP call on this thread ran, e.g. "slice V4",
 * "coop V4", "fast_rowrec V4", "perm_gather V4", "generic V1",
 * "slice_l2window V4", "fast+det V4", "atomic" ("" before the first call). */
const char *sptk_last_dispatch(void);

#ifdef __cplusplus
}
#endif
#endif /* SPTK_H */
