// mttkrp.cuh -- the hot-path kernel: permuted-traversal COO MTTKRP
// (SURVEY §8(a) rows a3-a7), Eq. (2) of the paper computed by the
// permutation approach of §5 (Fig. mttkrp_perm):
//
//   "Each thread within a team iterates over a given block size of tensor
//    nonzeros and writes its contribution to the resulting factor matrix only
//    when the mode-n coordinate changes.  This must be an atomic-write if the
//    mode-n index is equal to the first or last index of the block ...;
//    otherwise, it is a regular (non-atomic) write."
//
// B200 mapping:
//   * a "worker" is a group of G lanes (G = R*sizeof(T)/32 rounded up to a
//     power of two); its lanes span the R columns, each lane owning V = 32 B /
//     sizeof(T) consecutive columns, so one factor row is one coalesced run of
//     256-bit loads (LDG.E.ENL2.256) across the group;
//   * each worker owns a contiguous run of `run` permuted positions (the
//     paper's NZPTM block);
//   * per position i: p = perm_n[i] (sequential), the 16/32-byte record
//     {x_p, l_p*} (one random aligned load, L1::no_allocate), then the N-1
//     factor rows A_m(l_pm, cols) (random 256-bit gathers: the dominant
//     traffic), Hadamard product times x_p in registers, accumulated while
//     the row is unchanged;
//   * on a row change the register row is flushed: plain vector store for a
//     row interior to the run (owned by this worker alone), red.global.add
//     (fp64 scalar / fp32 .v4) for the run's first and last rows;
//   * lambda (NULL = ones) is applied once per flush (Z1);
//   * U positions are processed per step with the perm entries for the next
//     step prefetched, so several records and 2U factor rows are in flight.
// The generic kernel (any N <= 6, any R) gathers through perm_n with scalar
// loads, runtime record offsets and column tiles; same write discipline.
#pragma once
#include "common.cuh"

namespace sptk {

constexpr uint32_t kNoRow = 0xffffffffu;

struct MttkrpArgs {
    const uint8_t *rec;
    const uint32_t *perm;        // NULL: `rec` is the compact permuted copy of `mode`
    const uint32_t *rowptr;      // rowptr_n (permuted copy only)
    const uint32_t *wrow;        // start row of every worker (permuted copy only)
    int64_t pos_begin, pos_end;  // permuted positions handled by this launch
    int64_t run;                 // positions per worker
    int64_t ld;                  // row stride of factors and out (= R)
    int col0, ncols;             // column tile
    int mode, N, rb;             // runtime mode / order / record bytes
    const void *A[kMaxModes];    // factor matrices (A[mode] unused)
    const void *lambda;          // NULL = ones
    void *out;
    // deterministic mode (permuted copy only): boundary-row partials go to
    // dpart[(2 w + slot) * ld + col] / drow[2 w + slot] instead of red.add
    // (slot 0: the worker's first row if it ends inside the block, slot 1: its
    // last row) and are summed in worker order by det_fixup_kernel
    uint32_t *drow;
    void *dpart;
    // slice traversal (mttkrp_slice_kernel): rows [row0, row1), row r's part
    // of slice k is [soff[(r-row0)(nslice+1)+k], soff[...+k+1]); sec = the
    // copy's secondary mode (its factor rows are L1-allocated, others not)
    const uint32_t *soff;
    int64_t row0, row1;
    int nslice, sec;
    int other_first;             // slice kernel: non-secondary gathers L2 evict_first
    int rowrec;                  // per-group kernel: row index stored in the copy's spare word
    // coop kernel over a window-major copy (order: window of l_sec, l_n,
    // l_sec; sort.cu): rows from the records' spare word, not monotonic, so
    // every flush is a red.add
    int win = 0;
};

// ----------------------------------------------------------------- loads
// L2 eviction policies: the streamed records are read once (evict_first), the
// gathered factor rows are reused (evict_last) -- keeps the record stream from
// flushing factor lines out of L2 when the factors exceed it (C4/C5 shapes).
#ifndef SPTK_STREAM_POLICY
#define SPTK_STREAM_POLICY "evict_first"
#endif
#ifndef SPTK_FACTOR_POLICY
#define SPTK_FACTOR_POLICY "evict_last"
#endif
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::" SPTK_STREAM_POLICY ".b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::" SPTK_FACTOR_POLICY ".b64 %0, 1.0;" : "=l"(p));
    return p;
}
#ifndef SPTK_REC_PREFETCH
#define SPTK_REC_PREFETCH ""
#endif
#ifndef SPTK_ROW_L1
#define SPTK_ROW_L1 ""
#endif
__device__ __forceinline__ void ld_rec32_p(const void *p, uint32_t (&r)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" SPTK_REC_PREFETCH ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_rec16_p(const void *p, uint32_t (&r)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint" SPTK_REC_PREFETCH ".v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "l"(p), "l"(pol));
    r[4] = r[5] = r[6] = r[7] = 0;
}
__device__ __forceinline__ void ld_row_p(const double *p, double (&r)[4], uint64_t pol) {
    asm volatile("ld.global.nc" SPTK_ROW_L1 ".L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                 : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_row_p(const float *p, float (&r)[8], uint64_t pol) {
    asm volatile("ld.global.nc" SPTK_ROW_L1 ".L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                   "=f"(r[6]), "=f"(r[7])
                 : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_rec32(const void *p, uint32_t (&r)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld_rec16(const void *p, uint32_t (&r)[8]) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "l"(p));
    r[4] = r[5] = r[6] = r[7] = 0;
}
__device__ __forceinline__ void ld_row(const double *p, double (&r)[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                 : "l"(p));
}
__device__ __forceinline__ void ld_row(const float *p, float (&r)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                   "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st_row(double *p, const double (&r)[4]) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r[0]), "d"(r[1]),
                 "d"(r[2]), "d"(r[3])
                 : "memory");
}
__device__ __forceinline__ void st_row(float *p, const float (&r)[8]) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]),
                 "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}
__device__ __forceinline__ void red_row(double *p, const double (&r)[4]) {
#pragma unroll
    for (int v = 0; v < 4; ++v)
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p + v), "d"(r[v]) : "memory");
}
__device__ __forceinline__ void red_row(float *p, const float (&r)[8]) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r[0]), "f"(r[1]),
                 "f"(r[2]), "f"(r[3])
                 : "memory");
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + 4), "f"(r[4]),
                 "f"(r[5]), "f"(r[6]), "f"(r[7])
                 : "memory");
}


// VW consecutive elements of T as one load/store (VW * sizeof(T) in {4..32}
// bytes, aligned): the lane's slice of a factor row.  vld carries the L2
// cache-hint policy; f64 reductions are scalar (red.global.add.v2.f64 is not
// accepted for sm_100a), f32 uses .v4 when it can.
template <typename T, int VW>
__device__ __forceinline__ void vld(const T *p, T (&r)[VW], uint64_t pol) {
    if constexpr (sizeof(T) * VW == 32) {
        ld_row_p(p, r, pol);
    } else if constexpr (sizeof(T) == 8 && VW == 2) {
        asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(r[0]), "=d"(r[1]) : "l"(p), "l"(pol));
    } else if constexpr (sizeof(T) == 8 && VW == 1) {
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r[0]) : "l"(p), "l"(pol));
    } else if constexpr (sizeof(T) == 4 && VW == 4) {
        asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "l"(p), "l"(pol));
    } else if constexpr (sizeof(T) == 4 && VW == 2) {
        asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                     : "=f"(r[0]), "=f"(r[1]) : "l"(p), "l"(pol));
    } else {
        asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r[0]) : "l"(p), "l"(pol));
    }
}
// gather that allocates in L1 only if `l1` (slice kernel: L1 is kept for the
// secondary factor's window); one predicated pair of loads, any vector width
template <typename T, int VW>
__device__ __forceinline__ void vld_sel(const T *p, T (&r)[VW], uint64_t pol, bool l1) {
    const unsigned f = l1;
    if constexpr (sizeof(T) == 8 && VW == 4) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %6;\n\t"
                     "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %6;\n\t}"
                     : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p), "r"(f), "l"(pol));
    } else if constexpr (sizeof(T) == 8 && VW == 2) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %4;\n\t"
                     "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %4;\n\t}"
                     : "=d"(r[0]), "=d"(r[1]) : "l"(p), "r"(f), "l"(pol));
    } else if constexpr (sizeof(T) == 8) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.f64 %0, [%1], %3;\n\t"
                     "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %3;\n\t}"
                     : "=d"(r[0]) : "l"(p), "r"(f), "l"(pol));
    } else if constexpr (VW == 8) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %9, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %10;\n\t"
                     "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %10;\n\t}"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                       "=f"(r[6]), "=f"(r[7])
                     : "l"(p), "r"(f), "l"(pol));
    } else if constexpr (VW == 4) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %6;\n\t"
                     "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %6;\n\t}"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "l"(p), "r"(f), "l"(pol));
    } else if constexpr (VW == 2) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %4;\n\t"
                     "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %4;\n\t}"
                     : "=f"(r[0]), "=f"(r[1]) : "l"(p), "r"(f), "l"(pol));
    } else {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                     "@q ld.global.nc.L2::cache_hint.f32 %0, [%1], %3;\n\t"
                     "@!q ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %3;\n\t}"
                     : "=f"(r[0]) : "l"(p), "r"(f), "l"(pol));
    }
}
template <typename T, int VW>
__device__ __forceinline__ void vld_plain(const T *p, T (&r)[VW]) {
#pragma unroll
    for (int v = 0; v < VW; ++v) r[v] = __ldg(p + v);
}
template <typename T, int VW>
__device__ __forceinline__ void vst(T *p, const T (&r)[VW]) {
    if constexpr (sizeof(T) * VW == 32) {
        st_row(p, r);
    } else if constexpr (sizeof(T) * VW == 16) {
        if constexpr (sizeof(T) == 8) *reinterpret_cast<double2 *>(p) = make_double2(r[0], r[1]);
        else *reinterpret_cast<float4 *>(p) = make_float4(r[0], r[1], r[2], r[3]);
    } else if constexpr (sizeof(T) * VW == 8 && sizeof(T) == 4) {
        *reinterpret_cast<float2 *>(p) = make_float2(r[0], r[1]);
    } else {
#pragma unroll
        for (int v = 0; v < VW; ++v) p[v] = r[v];
    }
}
template <typename T, int VW>
__device__ __forceinline__ void vred(T *p, const T (&r)[VW]) {
    if constexpr (sizeof(T) == 4 && VW % 4 == 0) {
#pragma unroll
        for (int v = 0; v < VW; v += 4)
            asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + v), "f"(r[v]),
                         "f"(r[v + 1]), "f"(r[v + 2]), "f"(r[v + 3])
                         : "memory");
    } else {
#pragma unroll
        for (int v = 0; v < VW; ++v) atomicAdd(p + v, r[v]);
    }
}

template <typename T> __device__ __forceinline__ T rec_val(const uint32_t (&w)[8]);
template <> __device__ __forceinline__ double rec_val<double>(const uint32_t (&w)[8]) {
    return __hiloint2double((int)w[1], (int)w[0]);
}
template <> __device__ __forceinline__ float rec_val<float>(const uint32_t (&w)[8]) {
    return __uint_as_float(w[0]);
}

// ------------------------------------------------------- fast kernel body
// T, N (3..5), MODE (< N) and G (lanes per worker) are compile-time; the
// column tile is [col0, col0 + ncols) with ncols <= G*V and ncols % V == 0.
// SORTED: `rec` is the compact permuted copy of mode MODE ({x, l_m for
// m != MODE}, RB bytes, position i = record i, streamed and prefetched one
// step ahead); the mode-n row of position i is tracked with rowptr_n from
// the worker's start row `wrow` (rows only grow along the permutation).
// Otherwise the paper's traversal: p = perm_n[i] (prefetched one step ahead),
// gather the full record p and read l_pn from it.
// ROWREC (permuted copy with a spare record word): the row is read from the
// record instead of advancing through rowptr_n -- no dependent rowptr load per
// row change (short rows) or per empty row (power-law modes)
template <typename T, int N, int MODE, int G, int U, int RB, bool SORTED, int V, bool ROWREC>
__device__ __forceinline__ void mttkrp_fast_body(const MttkrpArgs &a) {
    constexpr int OFF = sizeof(T) / 4;  // first index word in a record
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t worker = gtid / G;
    const int q = (int)(gtid % G);
    if (a.pos_begin + worker * a.run >= a.pos_end) return;
    // positions fit in 32 bits (P < 2^32): keeps the loop state small
    const uint32_t s = (uint32_t)(a.pos_begin + worker * a.run);
    const uint32_t e = (uint32_t)min(a.pos_begin + worker * a.run + a.run, a.pos_end);
    const bool lane_on = q * V < a.ncols;
    const int c = a.col0 + q * V;
    const uint8_t *__restrict__ rec = a.rec;
    const uint32_t *__restrict__ perm = a.perm;
    T *__restrict__ out = static_cast<T *>(a.out);

    T acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = T(0);
    uint32_t cur = kNoRow, first = kNoRow;

    bool wrote0 = false;  // deterministic mode: slot 0 used
    auto flush = [&](uint32_t row, bool atomic, int slot) {
        if (atomic && a.dpart && q == 0) a.drow[2 * worker + slot] = row;
        if (atomic && slot == 0) wrote0 = true;
        if (!lane_on) return;
        T o[V];
#pragma unroll
        for (int v = 0; v < V; ++v) o[v] = acc[v];
        if (a.lambda) {  // lambda applied once per flushed row (Z1)
            T lam[V];
            vld_plain<T, V>(static_cast<const T *>(a.lambda) + c, lam);
#pragma unroll
            for (int v = 0; v < V; ++v) o[v] *= lam[v];
        }
        if (atomic && a.dpart)
            vst<T, V>(static_cast<T *>(a.dpart) + (2 * worker + slot) * a.ld + c, o);
        else if (atomic)
            vred<T, V>(out + (int64_t)row * a.ld + c, o);
        else
            vst<T, V>(out + (int64_t)row * a.ld + c, o);
    };
    const uint64_t pol_stream = policy_evict_first(), pol_factor = policy_evict_last();
    auto load_rec = [&](uint32_t pos, uint32_t (&r)[8]) {
        if constexpr (SORTED) {
            if constexpr (RB == 32) ld_rec32_p(rec + (size_t)pos * 32, r, pol_stream);
            else ld_rec16_p(rec + (size_t)pos * 16, r, pol_stream);
        } else {
            if constexpr (RB == 32) ld_rec32(rec + (size_t)pos * 32, r);
            else ld_rec16(rec + (size_t)pos * 16, r);
        }
    };

    uint32_t row = 0;   // SORTED: row of the current position
    uint32_t nxt = 0;   // SORTED: first position of row + 1
    if constexpr (SORTED && !ROWREC) {
        row = __ldg(a.wrow + worker);
        nxt = __ldg(a.rowptr + row + 1);
    }
    uint32_t pn[U];
    uint32_t wn[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if constexpr (SORTED) {
            pn[u] = (s + u < e) ? 0u : kNoRow;
            if (s + u < e) load_rec(s + u, wn[u]);
        } else {
            pn[u] = (s + u < e) ? __ldg(perm + s + u) : kNoRow;
        }
    }

    for (uint32_t i = s; i < e; i += U) {
        uint32_t p[U];
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) p[u] = pn[u];
        if constexpr (SORTED) {
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < 8; ++k) w[u][k] = wn[u][k];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t qq = i + U + u;
                pn[u] = qq < e ? 0u : kNoRow;
                if (qq < e) load_rec(qq, wn[u]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u)
                pn[u] = (i + U + u < e) ? __ldg(perm + i + U + u) : kNoRow;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (p[u] != kNoRow) {
                    load_rec(p[u], w[u]);
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) w[u][k] = 0;
                }
            }
        }
        T f[U][N][V];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < N; ++m)
                if (m != MODE) {
                    const int word = SORTED ? OFF + (m < MODE ? m : m - 1) : OFF + m;
                    if (p[u] != kNoRow && lane_on)
                        vld<T, V>(static_cast<const T *>(a.A[m]) + (int64_t)w[u][word] * a.ld + c,
                                  f[u][m], pol_factor);
                    else
#pragma unroll
                        for (int v = 0; v < V; ++v) f[u][m][v] = T(0);
                }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (p[u] == kNoRow) continue;
            uint32_t r;
            if constexpr (SORTED && ROWREC) {
                r = w[u][OFF + N - 1];
            } else if constexpr (SORTED) {
                const uint32_t pos = i + u;
                while (pos >= nxt) {
                    ++row;
                    nxt = __ldg(a.rowptr + row + 1);
                }
                r = row;
            } else {
                r = w[u][OFF + MODE];
            }
            if (r != cur) {
                if (cur != kNoRow) flush(cur, cur == first, 0);
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = T(0);
                if (first == kNoRow) first = r;
                cur = r;
            }
            const T x = rec_val<T>(w[u]);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                T t = x;
#pragma unroll
                for (int m = 0; m < N; ++m)
                    if (m != MODE) t *= f[u][m][v];
                acc[v] += t;
            }
        }
    }
    if (cur != kNoRow) flush(cur, true, 1);
    if (a.dpart && !wrote0 && q == 0) a.drow[2 * worker] = kNoRow;
}

template <typename T, int N, int G, int U, int RB, bool SORTED, int MINB, int V, bool ROWREC>
__global__ void __launch_bounds__(256, MINB) mttkrp_fast_kernel(const MttkrpArgs a) {
    pdl_wait();
    if constexpr (N >= 1) if (a.mode == 0) { mttkrp_fast_body<T, N, 0, G, U, RB, SORTED, V, ROWREC>(a); return; }
    if constexpr (N >= 2) if (a.mode == 1) { mttkrp_fast_body<T, N, 1, G, U, RB, SORTED, V, ROWREC>(a); return; }
    if constexpr (N >= 3) if (a.mode == 2) { mttkrp_fast_body<T, N, 2, G, U, RB, SORTED, V, ROWREC>(a); return; }
    if constexpr (N >= 4) if (a.mode == 3) { mttkrp_fast_body<T, N, 3, G, U, RB, SORTED, V, ROWREC>(a); return; }
    if constexpr (N >= 5) if (a.mode == 4) { mttkrp_fast_body<T, N, 4, G, U, RB, SORTED, V, ROWREC>(a); return; }
}

// ------------------------------------------------- warp-cooperative body
// Permuted copy only, for modes with long rows.  A worker is a whole warp
// owning `run * NG` consecutive positions (NG = 32 / G lane groups); each
// step the NG groups take NG consecutive positions (u = 0..U-1), so one
// warp-wide load covers NG consecutive compact records (NG*RB contiguous
// bytes) instead of NG scattered ones.  While every position of a step lies
// in the current row (warp-uniform test against rowptr_n) each group just
// accumulates its own products.  A step that crosses a row boundary (or the
// chunk's tail) is resolved serially: the group accumulators are summed with
// shuffles, then the step's products are taken in position order (broadcast
// from the owning group) and every completed row is flushed -- atomically if
// it is the chunk's first row, otherwise with a plain store; the last row of
// the chunk is flushed atomically at the end (P:521-523 with worker = warp).
template <typename T, int N, int MODE, int G, int U, int RB, int V>
__device__ __forceinline__ void mttkrp_coop_body(const MttkrpArgs &a) {
    constexpr int OFF = sizeof(T) / 4;
    constexpr int NG = 32 / G;
    const int64_t warp_id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int g = lane / G, q = lane % G;
    const int64_t chunk = a.run * NG;
    if (a.pos_begin + warp_id * chunk >= a.pos_end) return;
    const uint32_t s = (uint32_t)(a.pos_begin + warp_id * chunk);
    const uint32_t e = (uint32_t)min(a.pos_begin + warp_id * chunk + chunk, a.pos_end);
    const bool lane_on = q * V < a.ncols;
    const int c = a.col0 + q * V;
    const uint8_t *__restrict__ rec = a.rec;
    T *__restrict__ out = static_cast<T *>(a.out);

    bool wrote0 = false;  // deterministic mode: slot 0 used
    auto flush = [&](uint32_t row, const T (&val)[V], bool atomic, int slot) {
        if (atomic && slot == 0) wrote0 = true;
        if (g != 0) return;
        if (atomic && a.dpart && q == 0) a.drow[2 * warp_id + slot] = row;
        if (!lane_on) return;
        T o[V];
#pragma unroll
        for (int v = 0; v < V; ++v) o[v] = val[v];
        if (a.lambda) {
            T lam[V];
            vld_plain<T, V>(static_cast<const T *>(a.lambda) + c, lam);
#pragma unroll
            for (int v = 0; v < V; ++v) o[v] *= lam[v];
        }
        if (atomic && a.dpart)
            vst<T, V>(static_cast<T *>(a.dpart) + (2 * warp_id + slot) * a.ld + c, o);
        else if (atomic)
            vred<T, V>(out + (int64_t)row * a.ld + c, o);
        else
            vst<T, V>(out + (int64_t)row * a.ld + c, o);
    };
    const uint64_t pol_stream = policy_evict_first(), pol_factor = policy_evict_last();
    auto load_rec = [&](uint32_t pos, uint32_t (&r)[8]) {
        if constexpr (RB == 32) ld_rec32_p(rec + (size_t)pos * 32, r, pol_stream);
        else ld_rec16_p(rec + (size_t)pos * 16, r, pol_stream);
    };

    constexpr int RW = OFF + N - 1;  // spare record word: the position's row (window-major copy)
    const bool win = a.win != 0;
    uint32_t row, nxt;
    if (win) {
        row = __ldg(reinterpret_cast<const uint32_t *>(rec + (size_t)s * RB) + RW);
        nxt = 0;
    } else {
        row = __ldg(a.wrow + warp_id);
        nxt = __ldg(a.rowptr + row + 1);
    }
    const uint32_t first = row;
    T acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = T(0);

    uint32_t wn[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t pos = s + u * NG + g;
        if (pos < e) load_rec(pos, wn[u]);
    }
    for (uint32_t base = s; base < e; base += U * NG) {
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) w[u][k] = wn[u][k];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t pos = base + U * NG + u * NG + g;
            if (pos < e) load_rec(pos, wn[u]);
        }
        T t[U][V];
        {
            T f[U][N][V];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int m = 0; m < N; ++m)
                    if (m != MODE) {
                        const int word = OFF + (m < MODE ? m : m - 1);
                        if (base + u * NG + g < e && lane_on)
                            vld<T, V>(static_cast<const T *>(a.A[m]) + (int64_t)w[u][word] * a.ld + c,
                                      f[u][m], pol_factor);
                        else
#pragma unroll
                            for (int v = 0; v < V; ++v) f[u][m][v] = T(0);
                    }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const T x = (base + u * NG + g < e) ? rec_val<T>(w[u]) : T(0);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    T p = x;
#pragma unroll
                    for (int m = 0; m < N; ++m)
                        if (m != MODE) p *= f[u][m][v];
                    t[u][v] = p;
                }
            }
        }
        const uint32_t last = base + U * NG - 1;
        bool inside;
        if (win) {  // every position of the step in the current row (rows from the records)
            bool ok = last < e;
#pragma unroll
            for (int u = 0; u < U; ++u) ok = ok && w[u][RW] == row;
            inside = __all_sync(0xffffffffu, ok);
        } else {
            inside = last < nxt && last < e;
        }
        if (inside) {  // whole step inside the current row
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] += t[u][v];
            continue;
        }
        // serial resolution of the step: tot = sum of the group accumulators
        T tot[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            T x = acc[v];
#pragma unroll
            for (int o = G; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            tot[v] = x;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t myrow = w[u][RW];
            for (int gg = 0; gg < NG; ++gg) {
                const uint32_t pos = base + u * NG + gg;
                if (pos >= e) break;
                if (win) {
                    const uint32_t prow = __shfl_sync(0xffffffffu, myrow, gg * G);
                    if (prow != row) {
                        flush(row, tot, true, 0);
#pragma unroll
                        for (int v = 0; v < V; ++v) tot[v] = T(0);
                        row = prow;
                    }
                } else if (pos >= nxt) {
                    flush(row, tot, row == first, 0);
#pragma unroll
                    for (int v = 0; v < V; ++v) tot[v] = T(0);
                    do {
                        ++row;
                        nxt = __ldg(a.rowptr + row + 1);
                    } while (pos >= nxt);
                }
#pragma unroll
                for (int v = 0; v < V; ++v)
                    tot[v] += __shfl_sync(0xffffffffu, t[u][v], gg * G + q);
            }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = (g == 0) ? tot[v] : T(0);
    }
    // the chunk's last row (possibly also its first): atomic
    T tot[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        T x = acc[v];
#pragma unroll
        for (int o = G; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        tot[v] = x;
    }
    flush(row, tot, true, 1);
    if (a.dpart && !wrote0 && lane == 0) a.drow[2 * warp_id] = kNoRow;
}

template <typename T, int N, int G, int U, int RB, int MINB, int V>
__global__ void __launch_bounds__(256, MINB) mttkrp_coop_kernel(const MttkrpArgs a) {
    pdl_wait();
    if constexpr (N >= 1) if (a.mode == 0) { mttkrp_coop_body<T, N, 0, G, U, RB, V>(a); return; }
    if constexpr (N >= 2) if (a.mode == 1) { mttkrp_coop_body<T, N, 1, G, U, RB, V>(a); return; }
    if constexpr (N >= 3) if (a.mode == 2) { mttkrp_coop_body<T, N, 2, G, U, RB, V>(a); return; }
    if constexpr (N >= 4) if (a.mode == 3) { mttkrp_coop_body<T, N, 3, G, U, RB, V>(a); return; }
    if constexpr (N >= 5) if (a.mode == 4) { mttkrp_coop_body<T, N, 4, G, U, RB, V>(a); return; }
}

// ---------------------------------------------------- slice kernel
// Row-sliced traversal of the permuted copy (copy order: l_n, then the
// secondary mode a's index).  A block of B = blockDim/32 warps takes B
// consecutive rows and one slice k of a's index range; warp w walks row
// (row0 + B*blockIdx.x + w)'s nonzeros whose l_a falls in slice k -- a
// contiguous run of its row segment -- in permuted order, NG groups x U
// positions per step like the cooperative kernel, with no row break inside
// the run.  The B warps sweep the same A_a slice (sized to stay L1-resident),
// so each A_a row is fetched from L2 about once per block instead of once per
// nonzero; the other factors are gathered without L1 allocation.  Every row
// receives one partial per slice, flushed with red.global.add (the row is
// shared by the nslice blocks of its row group).
template <typename T, int N, int MODE, int G, int U, int RB, int V>
__device__ __forceinline__ void mttkrp_slice_body(const MttkrpArgs &a) {
    constexpr int OFF = sizeof(T) / 4;
    constexpr int NG = 32 / G;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane / G, q = lane % G;
    const int64_t r = a.row0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (r >= a.row1) return;
    const uint32_t *so = a.soff + (r - a.row0) * (a.nslice + 1) + blockIdx.y;
    const uint32_t s = __ldg(so), e = __ldg(so + 1);
    if (s >= e) return;
    const bool lane_on = q * V < a.ncols;
    const int c = a.col0 + q * V;
    const uint8_t *__restrict__ rec = a.rec;
    const uint64_t pol_stream = policy_evict_first(), pol_factor = policy_evict_last();
    // the window of the secondary factor stays in L2 (evict_last); with
    // other_first the other factors' random rows are evicted first
    const uint64_t pol_other = a.other_first ? pol_stream : pol_factor;
    auto load_rec = [&](uint32_t pos, uint32_t (&w)[8]) {
        if constexpr (RB == 32) ld_rec32_p(rec + (size_t)pos * 32, w, pol_stream);
        else ld_rec16_p(rec + (size_t)pos * 16, w, pol_stream);
    };
    T acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = T(0);
    uint32_t wn[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint32_t pos = s + u * NG + g;
        if (pos < e) load_rec(pos, wn[u]);
    }
    for (uint32_t base = s; base < e; base += U * NG) {
        uint32_t w[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) w[u][k] = wn[u][k];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t pos = base + U * NG + u * NG + g;
            if (pos < e) load_rec(pos, wn[u]);
        }
        T f[U][N][V];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < N; ++m)
                if (m != MODE) {
                    const int word = OFF + (m < MODE ? m : m - 1);
                    const T *src = static_cast<const T *>(a.A[m]) + (int64_t)w[u][word] * a.ld + c;
                    if (base + u * NG + g < e && lane_on) {
                        vld_sel<T, V>(src, f[u][m], m == a.sec ? pol_factor : pol_other,
                                      m == a.sec);
                    } else {
#pragma unroll
                        for (int v = 0; v < V; ++v) f[u][m][v] = T(0);
                    }
                }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const T x = (base + u * NG + g < e) ? rec_val<T>(w[u]) : T(0);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                T p = x;
#pragma unroll
                for (int m = 0; m < N; ++m)
                    if (m != MODE) p *= f[u][m][v];
                acc[v] += p;
            }
        }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
#pragma unroll
        for (int o = G; o < 32; o <<= 1) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], o);
    }
    if (g != 0 || !lane_on) return;
    if (a.lambda) {
        T lam[V];
        vld_plain<T, V>(static_cast<const T *>(a.lambda) + c, lam);
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] *= lam[v];
    }
    vred<T, V>(static_cast<T *>(a.out) + r * a.ld + c, acc);
}

template <typename T, int N, int G, int U, int RB, int MINB, int V>
__global__ void __launch_bounds__(256, MINB) mttkrp_slice_kernel(const MttkrpArgs a) {
    pdl_wait();
    if constexpr (N >= 1) if (a.mode == 0) { mttkrp_slice_body<T, N, 0, G, U, RB, V>(a); return; }
    if constexpr (N >= 2) if (a.mode == 1) { mttkrp_slice_body<T, N, 1, G, U, RB, V>(a); return; }
    if constexpr (N >= 3) if (a.mode == 2) { mttkrp_slice_body<T, N, 2, G, U, RB, V>(a); return; }
    if constexpr (N >= 4) if (a.mode == 3) { mttkrp_slice_body<T, N, 3, G, U, RB, V>(a); return; }
    if constexpr (N >= 5) if (a.mode == 4) { mttkrp_slice_body<T, N, 4, G, U, RB, V>(a); return; }
}

// ---------------------------------------------------- generic kernel
// Any N <= 6, any mode, any column tile: lane q of a G-lane worker owns
// columns col0 + q + G*k (k < NV), scalar loads, runtime record offsets.
template <typename T, int G, int NV>
__global__ void __launch_bounds__(256) mttkrp_generic_kernel(const MttkrpArgs a) {
    pdl_wait();
    constexpr int U = 2;
    const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t worker = gtid / G;
    const int q = (int)(gtid % G);
    const int64_t s = a.pos_begin + worker * a.run;
    if (s >= a.pos_end) return;
    const int64_t e = min(s + a.run, a.pos_end);
    const int N = a.N, mode = a.mode, rb = a.rb;
    const int off = sizeof(T) / 4;
    const uint8_t *__restrict__ rec = a.rec;
    T *__restrict__ out = static_cast<T *>(a.out);
    bool on[NV];
    int col[NV];
    T lam[NV], acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        col[k] = a.col0 + q + G * k;
        on[k] = q + G * k < a.ncols;
        lam[k] = (a.lambda && on[k]) ? static_cast<const T *>(a.lambda)[col[k]] : T(1);
        acc[k] = T(0);
    }
    uint32_t cur = kNoRow, first = kNoRow;
    auto flush = [&](uint32_t row, bool atomic) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            if (!on[k]) continue;
            T *dst = out + (int64_t)row * a.ld + col[k];
            const T o = acc[k] * lam[k];
            if (atomic) atomicAdd(dst, o);
            else *dst = o;
        }
    };
    for (int64_t i = s; i < e; i += U) {
        uint32_t p[U], row[U];
        T x[U];
        T t[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            p[u] = (i + u < e) ? __ldg(a.perm + i + u) : kNoRow;
            if (p[u] == kNoRow) continue;
            const uint8_t *r = rec + (size_t)p[u] * rb;
            x[u] = __ldg(reinterpret_cast<const T *>(r));
            const uint32_t *ix = reinterpret_cast<const uint32_t *>(r) + off;
            row[u] = __ldg(ix + mode);
#pragma unroll
            for (int k = 0; k < NV; ++k) t[u][k] = x[u];
#pragma unroll
            for (int m = 0; m < kMaxModes; ++m) {
                if (m >= N || m == mode) continue;
                const T *Am = static_cast<const T *>(a.A[m]) + (int64_t)__ldg(ix + m) * a.ld;
#pragma unroll
                for (int k = 0; k < NV; ++k)
                    if (on[k]) t[u][k] *= __ldg(Am + col[k]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (p[u] == kNoRow) continue;
            if (row[u] != cur) {
                if (cur != kNoRow) flush(cur, cur == first);
#pragma unroll
                for (int k = 0; k < NV; ++k) acc[k] = T(0);
                if (first == kNoRow) first = row[u];
                cur = row[u];
            }
#pragma unroll
            for (int k = 0; k < NV; ++k) acc[k] += t[u][k];
        }
    }
    if (cur != kNoRow) flush(cur, true);
}

// Launch shapes: U positions per step per group; >= 3 resident 256-thread
// blocks per SM (register cap 80) for N = 3, >= 2 (cap 128) for N >= 4, whose
// U(N-1) gathered 32-byte slices spill under the 80-register cap (measured on
// the Delicious shape, N = 4: -9 % with 2 blocks; NELL-2, N = 3: +20 %
// with 2 blocks, profiles/r01/ab_minblocks.log).  Variant 0: per-group runs
// (mttkrp_fast_kernel); variant 1: warp-cooperative steps
// (mttkrp_coop_kernel, permuted copy only).
constexpr int kNumVariants = 2;
#ifndef SPTK_KU
#define SPTK_KU 2
#endif
#ifndef SPTK_KMINB
#define SPTK_KMINB 3
#endif
#ifndef SPTK_KMINB_WIDE
#define SPTK_KMINB_WIDE 2
#endif
#ifndef SPTK_KU_WIDE
#define SPTK_KU_WIDE SPTK_KU
#endif
#ifndef SPTK_KU_5  // N = 5 (LBNL) separately, for A/B builds
#define SPTK_KU_5 SPTK_KU_WIDE
#endif
#ifndef SPTK_KMINB_5
#define SPTK_KMINB_5 SPTK_KMINB_WIDE
#endif
template <int N> constexpr int kU = N <= 3 ? SPTK_KU : (N == 5 ? SPTK_KU_5 : SPTK_KU_WIDE);
template <int N> constexpr int kMinBlocks = N <= 3 ? SPTK_KMINB : (N == 5 ? SPTK_KMINB_5 : SPTK_KMINB_WIDE);

template <typename T, int N, int RB, bool SORTED, bool COOP, int V, bool ROWREC = false>
inline sptk_status fast_launch_g(int G, const MttkrpArgs &a, int64_t workers, cudaStream_t s) {
    const int64_t threads = COOP ? workers * 32 : workers * G;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
#define SPTK_LAUNCH_G(GG)                                                                     \
    if constexpr (COOP)                                                                       \
        launch_pdl(mttkrp_coop_kernel<T, N, GG, kU<N>, RB, kMinBlocks<N>, V>, blocks, 256, 0, s, a); \
    else                                                                                      \
        launch_pdl(mttkrp_fast_kernel<T, N, GG, kU<N>, RB, SORTED, kMinBlocks<N>, V, ROWREC>, blocks, 256, 0, s, a);
    switch (G) {
    case 1: SPTK_LAUNCH_G(1) break;
    case 2: SPTK_LAUNCH_G(2) break;
    case 4: SPTK_LAUNCH_G(4) break;
    case 8: SPTK_LAUNCH_G(8) break;
    case 16: SPTK_LAUNCH_G(16) break;
    case 32: SPTK_LAUNCH_G(32) break;
    default: return fail(SPTK_EINVAL, "fast MTTKRP: bad lane count");
    }
#undef SPTK_LAUNCH_G
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

// slice traversal: blocks of 8 rows x nslice slices (grid.y)
template <typename T, int N, int RC, int V>
inline sptk_status slice_launch_g(int G, const MttkrpArgs &a, cudaStream_t s) {
    const dim3 grid((unsigned)((a.row1 - a.row0 + 7) / 8), (unsigned)a.nslice);
#define SPTK_LAUNCH_S(GG) launch_pdl(mttkrp_slice_kernel<T, N, GG, kU<N>, RC, kMinBlocks<N>, V>, grid, dim3(256), 0, s, a);
    switch (G) {
    case 1: SPTK_LAUNCH_S(1) break;
    case 2: SPTK_LAUNCH_S(2) break;
    case 4: SPTK_LAUNCH_S(4) break;
    case 8: SPTK_LAUNCH_S(8) break;
    case 16: SPTK_LAUNCH_S(16) break;
    case 32: SPTK_LAUNCH_S(32) break;
    default: return fail(SPTK_EINVAL, "slice MTTKRP: bad lane count");
    }
#undef SPTK_LAUNCH_S
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

// Per-(T, N, V) launcher, explicitly instantiated in mttkrp_<t>_n<N>_v<V>.cu.
// `workers` counts groups (variant 0) or warps (variant 1); variant 2 is the
// slice traversal.  The perm-gather
// layout is compiled for the widest vector only (other R use the generic kernel).
template <typename T, int N, int V>
sptk_status launch_fast_tnv(int G, int variant, const MttkrpArgs &a, int64_t workers,
                            cudaStream_t s);

#define SPTK_INSTANTIATE_FAST(T, N, V)                                                       \
    template <>                                                                              \
    sptk_status launch_fast_tnv<T, N, V>(int G, int variant, const MttkrpArgs &a,            \
                                         int64_t workers, cudaStream_t s) {                  \
        constexpr int RB = (sizeof(T) + 4 * N <= 16) ? 16 : 32;        /* full record */      \
        constexpr int RC = (sizeof(T) + 4 * (N - 1) <= 16) ? 16 : 32;  /* compact copy */     \
        if (a.perm) {                                                                        \
            if constexpr (V * sizeof(T) == 32)                                               \
                return fast_launch_g<T, N, RB, false, false, V>(G, a, workers, s);           \
            return fail(SPTK_EINVAL, "perm-gather fast path needs 32-byte vectors");         \
        }                                                                                    \
        if (variant == 2) return slice_launch_g<T, N, RC, V>(G, a, s);                       \
        if (variant == 1) return fast_launch_g<T, N, RC, true, true, V>(G, a, workers, s);   \
        if constexpr (RC / 4 >= (int)sizeof(T) / 4 + N)       /* spare word: row in record */ \
            if (a.rowrec) return fast_launch_g<T, N, RC, true, false, V, true>(G, a, workers, s); \
        return fast_launch_g<T, N, RC, true, false, V>(G, a, workers, s);                    \
    }

template <typename T>
sptk_status launch_generic(int G, const MttkrpArgs &a, int64_t workers, cudaStream_t s);

}  // namespace sptk
