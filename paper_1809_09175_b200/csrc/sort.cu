// sort.cu -- build_perm: per-mode permutation arrays
// (§5: "a permutation array for each mode that sorts the tensor
// nonzeros in increasing index along that mode"), built on the GPU by a
// STABLE least-significant-digit radix sort of (key = l_in, value = i).
// Stability (P:584 names a *stable* sort) makes the permutation unique.
//
// Per digit pass (<= 8 bits, ceil(bits(I_n - 1) / passes) bits each):
//   upsweep    per-tile digit histograms          counts[digit][tile]
//   scan       exclusive scan of counts (digit-major) -> global offsets
//   downsweep  stable scatter: inside a 4096-key tile, warp w owns keys
//              [w*512, w*512+512) and ranks equal digits with per-bit ballots
//              in rounds of 32, so equal keys keep their storage order.
// Then rowptr_n[r] = first sorted position with key >= r (boundary kernel).
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace sptk {

constexpr int kSortThreads = 256;
#ifndef SPTK_SORT_ITEMS  // A/B builds only
#define SPTK_SORT_ITEMS 16
#endif
#ifndef SPTK_DS_MINB     // A/B builds only: min resident blocks of the leaner downsweep
#define SPTK_DS_MINB 3
#endif
constexpr int kSortItems = SPTK_SORT_ITEMS;                 // keys per thread
constexpr int kSortTile = kSortThreads * kSortItems;        // 4096
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kWarpChunk = kSortTile / kSortWarps;          // 512 keys per warp
constexpr int kScanChunk = 4096;

// radix-sort workspace in 32-bit words: keys x2, values, digit counts, scan sums
static size_t sort_ws_words(int64_t P) {
    const size_t nP = (size_t)P, ncnt = (size_t)((P + kSortTile - 1) / kSortTile) * 256;
    return 3 * nP + ncnt + (ncnt + kScanChunk - 1) / kScanChunk + 64;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Lanes of the warp holding the same digit (bits < 9), from `bits` ballots
// instead of __match_any_sync (MATCH is a slow MIO op); `valid` lanes only.
// (measured round 2: one __match_any_sync instead is 1.5x slower per pass,
// profiles/r02/ab_sort_match.log)
__device__ __forceinline__ uint32_t digit_peers(uint32_t digit, int bits, bool valid) {
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
    for (int b = 0; b < bits; ++b) {
        const bool on = (digit >> b) & 1u;
        const uint32_t m = __ballot_sync(0xffffffffu, on);
        peers &= on ? m : ~m;
    }
    return peers;
}

// keys[i] = l_i,mode from the packed records (one streaming pass)
__global__ void __launch_bounds__(256) extract_keys(const uint8_t *__restrict__ rec, int rb, int kw,
                                                    int64_t P, uint32_t *__restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = __ldg(reinterpret_cast<const uint32_t *>(rec + (size_t)i * rb) + kw);
}

__global__ void __launch_bounds__(kSortThreads)
    radix_upsweep(const uint32_t *__restrict__ keys, uint32_t P, int shift, int dbits,
                  uint32_t ntiles, uint32_t *__restrict__ counts) {
    __shared__ uint32_t hist[kSortWarps][256];  // per-warp: fewer colliding smem atomics
    const int nd = 1 << dbits;
    const int warp = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < kSortWarps * 256; d += blockDim.x) (&hist[0][0])[d] = 0;
    __syncthreads();
    const uint32_t base = blockIdx.x * (uint32_t)kSortTile;
    const uint32_t mask = (uint32_t)nd - 1;
    uint32_t k[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint32_t i = base + r * kSortThreads + threadIdx.x;
        k[r] = i < P ? __ldg(keys + i) : 0u;
    }
#pragma unroll
    for (int r = 0; r < kSortItems; ++r)
        if (base + r * kSortThreads + threadIdx.x < P) atomicAdd(&hist[warp][(k[r] >> shift) & mask], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < nd; d += blockDim.x) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) c += hist[w][d];
        counts[(size_t)d * ntiles + blockIdx.x] = c;
    }
}

// vals_in == NULL: the values are the positions i (first pass).
// Stable tile-local ranking (warp w owns keys [w*512, w*512+512) of the 4096-
// key tile; per-bit ballots rank equal digits within each round of 32, in
// storage order), then the tile is reordered by digit in shared memory and
// written out so that consecutive threads write consecutive positions of each
// digit's run (coalesced), global run start = scanned count of (digit, tile).
__global__ void __launch_bounds__(kSortThreads)
    radix_downsweep(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                    uint32_t P, int shift, int dbits, uint32_t ntiles,
                    const uint32_t *__restrict__ offsets, uint32_t *__restrict__ keys_out,
                    uint32_t *__restrict__ vals_out) {
    __shared__ uint32_t whist[kSortWarps][256];
    __shared__ uint32_t lstart[256];   // tile-local start of each digit
    __shared__ uint32_t gstart[256];   // global start of each digit's run of this tile
    __shared__ uint32_t skey[kSortTile];
    __shared__ uint32_t sval[kSortTile];
    const int nd = 1 << dbits;
    const uint32_t mask = (uint32_t)nd - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = lane; d < nd; d += 32) whist[warp][d] = 0;
    __syncwarp();
    const uint32_t tile0 = blockIdx.x * (uint32_t)kSortTile;
    const uint32_t tile_n = min((uint32_t)kSortTile, P - tile0);
    const uint32_t base = tile0 + warp * (uint32_t)kWarpChunk;
    const uint32_t lt = lanemask_lt();
    // all loads of the tile up front (the values too: loading them inside the
    // ranking loop left pass 2 latency-bound on long-scoreboard stalls)
    uint32_t key[kSortItems], val[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint32_t i = base + r * 32 + lane;
        key[r] = i < P ? __ldg(keys_in + i) : 0xffffffffu;
        val[r] = vals_in ? (i < P ? __ldg(vals_in + i) : 0u) : i;
    }
    // A: per-warp digit histogram of its 512-key sub-chunk (shared atomics:
    //    the ballot ranking is needed only for the stable positions in C)
#pragma unroll
    for (int r = 0; r < kSortItems; ++r)
        if (base + r * 32 + lane < P) atomicAdd(&whist[warp][(key[r] >> shift) & mask], 1u);
    __syncthreads();
    // B: tile-local digit starts (exclusive scan over digits of the tile counts)
    //    and per-warp starts within each digit
    {
        const int d = threadIdx.x;  // kSortThreads == 256 >= nd
        uint32_t tot = 0;
        if (d < nd) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t c = whist[w][d];
                whist[w][d] = run;  // offset of warp w within digit d
                run += c;
            }
            tot = run;
            gstart[d] = offsets[(size_t)d * ntiles + blockIdx.x];
        }
        // exclusive scan of tot over d (block-wide, 256 threads)
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        __shared__ uint32_t wsum[kSortWarps];
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += wsum[w];
        if (d < nd) lstart[d] = wpre + inc - tot;
    }
    __syncthreads();
    // C: stable local positions, scatter into shared memory (rounds in storage order)
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint32_t i = base + r * 32 + lane;
        const bool valid = i < P;
        const uint32_t digit = valid ? (key[r] >> shift) & mask : 0u;
        const uint32_t peers = digit_peers(digit, dbits, valid);
        uint32_t pos = 0;
        if (valid) pos = lstart[digit] + whist[warp][digit] + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers & lt) == 0) whist[warp][digit] += __popc(peers);
        __syncwarp();
        if (valid) {
            skey[pos] = key[r];
            sval[pos] = val[r];
        }
    }
    __syncthreads();
    // D: coalesced write-out of the digit runs
    for (uint32_t j = threadIdx.x; j < tile_n; j += kSortThreads) {
        const uint32_t k = skey[j];
        const uint32_t d = (k >> shift) & mask;
        const uint32_t g = gstart[d] + (j - lstart[d]);
        keys_out[g] = k;
        vals_out[g] = sval[j];
    }
}

// Leaner pass (round 2): the ranking produces the per-warp digit counts
// itself (no shared-memory atomics), the digit width is a template parameter
// (unrolled ballots), full tiles skip every bounds test, one shared load per
// key finds its tile position (warp base folded into the digit start) and one
// per key its global position (delta = global run start - tile start), and
// the last pass of a sort whose keys are not wanted writes values only.
// (round-1 kernel above: 4.6 warp instructions per key, issue-bound at
// 73 % issue-active, 0.43 of HBM; profiles/r02/prof_radix_raw.csv)
template <int DB>
struct DownsweepSmem {
    uint32_t wbase[kSortWarps][1 << DB];  // per-warp running count, then tile position base
    int32_t delta[1 << DB];               // global run start - tile start of each digit
    uint32_t wsum[kSortWarps];
    uint32_t skey[kSortTile];
    uint32_t sval[kSortTile];
};

template <int DB, bool FULL>
__device__ __forceinline__ void downsweep_body(DownsweepSmem<DB> &sm, uint32_t tile,
                                               const uint32_t *__restrict__ keys_in,
                                               const uint32_t *__restrict__ vals_in, uint32_t P,
                                               int shift, uint32_t ntiles,
                                               const uint32_t *__restrict__ offsets,
                                               uint32_t *__restrict__ keys_out,
                                               uint32_t *__restrict__ vals_out) {
    constexpr int ND = 1 << DB;
    constexpr uint32_t MASK = ND - 1;
    auto &wbase = sm.wbase;
    auto &delta = sm.delta;
    auto &wsum = sm.wsum;
    auto &skey = sm.skey;
    auto &sval = sm.sval;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = lane; d < ND; d += 32) wbase[warp][d] = 0;
    __syncwarp();
    const uint32_t tile0 = tile * (uint32_t)kSortTile;
    const uint32_t tile_n = FULL ? (uint32_t)kSortTile : P - tile0;
    const uint32_t base = tile0 + warp * (uint32_t)kWarpChunk;
    const uint32_t lt = lanemask_lt();
    uint32_t key[kSortItems], val[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const uint32_t i = base + r * 32 + lane;
        if (FULL || i < P) {
            key[r] = __ldg(keys_in + i);
            val[r] = vals_in ? __ldg(vals_in + i) : i;
        } else {
            key[r] = 0xffffffffu;
            val[r] = 0;
        }
    }
    // A: stable rank of every key among the equal digits of its warp chunk
    //    (rounds of 32 in storage order, per-bit ballots); the running count
    //    of each digit ends as the warp's digit histogram
    uint32_t rank[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const bool valid = FULL || base + r * 32 + lane < P;
        const uint32_t digit = (key[r] >> shift) & MASK;
        uint32_t peers = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int b = 0; b < DB; ++b)  // LOP3->P, VOTE, predicated NOT, AND per bit
            asm("{\n\t.reg .pred p;\n\t.reg .b32 m;\n\t"
                "and.b32 m, %1, %2;\n\t"
                "setp.ne.u32 p, m, 0;\n\t"
                "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
                "@!p not.b32 m, m;\n\t"
                "and.b32 %0, %0, m;\n\t}"
                : "+r"(peers) : "r"(digit), "r"(1u << b));
        const uint32_t below = __popc(peers & lt);
        uint32_t c = 0;
        if (valid) c = wbase[warp][digit];
        __syncwarp();
        if (valid && below == 0) wbase[warp][digit] = c + __popc(peers);
        __syncwarp();
        rank[r] = c + below;
    }
    __syncthreads();
    // B: per digit, the exclusive scan over warps and over digits: wbase :=
    //    tile position of the warp's first key of the digit; delta := global
    //    start of the digit's run of this tile - its tile start
    {
        const int d = threadIdx.x;  // kSortThreads == 256 >= ND
        uint32_t tot = 0;
        if (d < ND) {
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t c = wbase[w][d];
                wbase[w][d] = tot;
                tot += c;
            }
        }
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t wpre = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w)
            if (w < warp) wpre += wsum[w];
        if (d < ND) {
            const uint32_t lstart = wpre + inc - tot;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) wbase[w][d] += lstart;
            delta[d] = (int32_t)(offsets[(size_t)d * ntiles + tile] - lstart);
        }
    }
    __syncthreads();
    // C: tile-local scatter into shared memory
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        if (FULL || base + r * 32 + lane < P) {
            const uint32_t pos = wbase[warp][(key[r] >> shift) & MASK] + rank[r];
            skey[pos] = key[r];
            sval[pos] = val[r];
        }
    }
    __syncthreads();
    // D: coalesced write-out of the digit runs
#pragma unroll 4
    for (uint32_t j = threadIdx.x; j < tile_n; j += kSortThreads) {
        const uint32_t k = skey[j];
        const uint32_t g = (uint32_t)((int32_t)j + delta[(k >> shift) & MASK]);
        if (keys_out) keys_out[g] = k;
        vals_out[g] = sval[j];
    }
}

template <int DB>
__global__ void __launch_bounds__(kSortThreads, SPTK_DS_MINB)
    radix_downsweep2(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                     uint32_t P, int shift, uint32_t ntiles, const uint32_t *__restrict__ offsets,
                     uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out) {
    __shared__ DownsweepSmem<DB> sm;
    if ((blockIdx.x + 1) * (uint64_t)kSortTile <= P)
        downsweep_body<DB, true>(sm, blockIdx.x, keys_in, vals_in, P, shift, ntiles, offsets,
                                 keys_out, vals_out);
    else
        downsweep_body<DB, false>(sm, blockIdx.x, keys_in, vals_in, P, shift, ntiles, offsets,
                                  keys_out, vals_out);
}

static cudaError_t launch_downsweep2(int db, unsigned grid, cudaStream_t s, const uint32_t *kin,
                                     const uint32_t *vin, uint32_t P, int shift, uint32_t ntiles,
                                     const uint32_t *offsets, uint32_t *kout, uint32_t *vout) {
#define SPTK_DS(D) \
    case D: radix_downsweep2<D><<<grid, kSortThreads, 0, s>>>(kin, vin, P, shift, ntiles, offsets, kout, vout); break;
    switch (db) {
        SPTK_DS(1) SPTK_DS(2) SPTK_DS(3) SPTK_DS(4) SPTK_DS(5) SPTK_DS(6) SPTK_DS(7) SPTK_DS(8)
    default: return cudaErrorInvalidValue;
    }
#undef SPTK_DS
    return cudaGetLastError();
}

// ------------------------------------------------------------ exclusive scan
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// block-wide exclusive scan of one value per thread (256 threads); returns total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *excl) {
    __shared__ uint32_t wsum[kSortWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t inc = warp_incl_scan(v);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t s = wsum[w];
        if (w < warp) wpre += s;
        total += s;
    }
    __syncthreads();
    *excl = wpre + inc - v;
    return total;
}

__global__ void __launch_bounds__(256) scan_chunk_sums(const uint32_t *__restrict__ in, int64_t n,
                                                       uint32_t *__restrict__ bsum) {
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    uint32_t s = 0;
    for (int k = threadIdx.x; k < kScanChunk; k += blockDim.x) {
        const int64_t i = base + k;
        if (i < n) s += in[i];
    }
    __shared__ uint32_t sh[256];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) scan_block_sums(uint32_t *__restrict__ bsum, int64_t nb) {
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += 256) {
        const int64_t i = b0 + threadIdx.x;
        const uint32_t v = i < nb ? bsum[i] : 0;
        uint32_t ex;
        const uint32_t tot = block_excl_scan(v, &ex);
        if (i < nb) bsum[i] = carry + ex;
        carry += tot;
    }
}

// in-place allowed (in == out)
__global__ void __launch_bounds__(256) scan_chunk_apply(const uint32_t *in, int64_t n,
                                                        const uint32_t *__restrict__ bsum,
                                                        uint32_t *out) {
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    constexpr int per = kScanChunk / 256;  // 16 contiguous items per thread
    uint32_t v[per];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < per; ++k) {
        const int64_t i = base + threadIdx.x * per + k;
        v[k] = i < n ? in[i] : 0;
        s += v[k];
    }
    uint32_t ex;
    block_excl_scan(s, &ex);
    uint32_t run = bsum[blockIdx.x] + ex;
#pragma unroll
    for (int k = 0; k < per; ++k) {
        const int64_t i = base + threadIdx.x * per + k;
        if (i < n) out[i] = run;
        run += v[k];
    }
}

// tmp: at least ceil(n / kScanChunk) words
static sptk_status exclusive_scan(uint32_t *data, int64_t n, uint32_t *tmp, cudaStream_t s) {
    if (n == 0) return SPTK_OK;
    const int64_t nb = (n + kScanChunk - 1) / kScanChunk;
    scan_chunk_sums<<<(unsigned)nb, 256, 0, s>>>(data, n, tmp);
    scan_block_sums<<<1, 256, 0, s>>>(tmp, nb);
    scan_chunk_apply<<<(unsigned)nb, 256, 0, s>>>(data, n, tmp, data);
    count_launch(3);
    SPTK_CUDA(cudaGetLastError());
    return SPTK_OK;
}

// ------------------------------------------------------------ rowptr / iota
// rowptr[r] = first sorted position whose key >= r (binary search per row;
// balanced for any gap structure, including long runs of empty rows)
__global__ void rowptr_from_sorted(const uint32_t *__restrict__ keys, int64_t P, int64_t In,
                                   uint32_t *__restrict__ rowptr) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= In;
         r += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = P;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)__ldg(keys + mid) < r) lo = mid + 1;
            else hi = mid;
        }
        rowptr[r] = (uint32_t)lo;
    }
}

// out = max over rows of rowptr[r + 1] - rowptr[r] (the longest row)
__global__ void row_max_kernel(const uint32_t *__restrict__ rowptr, int64_t In,
                               uint32_t *__restrict__ out) {
    uint32_t m = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < In;
         r += (int64_t)gridDim.x * blockDim.x)
        m = max(m, __ldg(rowptr + r + 1) - __ldg(rowptr + r));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void iota_kernel(uint32_t *__restrict__ out, int64_t P) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)i;
}

__global__ void fill_u32(uint32_t *__restrict__ out, int64_t n, uint32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v;
}

// srec[i] = compact(rec[perm[i]]): the records in permuted order with the
// mode-n index dropped (it is implied by rowptr_n): {x, l_m for m != mode}.
template <int RB, int RC>
__global__ void __launch_bounds__(256)
    permute_records(const uint8_t *__restrict__ rec, const uint32_t *__restrict__ perm, int64_t P,
                    int vw, int N, int mode, uint8_t *__restrict__ srec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rec + (size_t)__ldg(perm + i) * RB);
        uint32_t w[8];
        const uint4 a = __ldg(src);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        if constexpr (RB == 32) {
            const uint4 b = __ldg(src + 1);
            w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
        } else {
            w[4] = w[5] = w[6] = w[7] = 0;
        }
        uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k < vw) o[k] = w[k];
        int d = vw;
#pragma unroll
        for (int m = 0; m < kMaxModes; ++m)
            if (m < N && m != mode && vw + m < 8 && d < 8) o[d++] = w[vw + m];
        if (d < RC / 4) o[d] = w[vw + mode];  // spare word: the row (mode-n index) itself
        uint4 *dst = reinterpret_cast<uint4 *>(srec + (size_t)i * RC);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        if constexpr (RC == 32) dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

static int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    const int64_t cap = (int64_t)dev_sms() * 16;
    if (b > cap) b = cap;
    return b < 1 ? 1 : (int)b;
}

static sptk_status stable_sort_ids(sptk_tensor t, int mode, const uint32_t *in, uint32_t *out,
                                   uint32_t **keys_out, cudaStream_t s, void *ext_ws = nullptr,
                                   size_t ext_bytes = 0, int kshift = 0);

// The longest row of `mode` (computed on the device at build_perm; one 4-byte
// read, cached).  -1 if unavailable.
int64_t row_max(sptk_tensor t, int mode, cudaStream_t s) {
    if (t->row_max[mode] >= 0) return t->row_max[mode];
    if (!t->has_perm[mode] || !t->rowmax_dev.p) return -1;
    uint32_t h = 0;
    if (cudaMemcpyAsync(&h, t->rowmax_dev.as<uint32_t>() + mode, sizeof h, cudaMemcpyDeviceToHost,
                        s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    t->row_max[mode] = h;
    return h;
}

// Secondary key of the copy order.  Balanced modes (longest row <= 2x the
// mean: the slice traversal applies) take the shortest other mode whose factor
// does not stay L1-resident (>= 2048 rows, 256 KB at R = 16 fp64) -- the factor
// the slice windows sweep.  Imbalanced (power-law) modes, which use the
// per-group / cooperative kernels, take the LARGEST other mode: a row's gathers
// of the biggest factor then go in increasing row order (Delicious mode 3
// -8 %, profiles/r02/ab_copy_secondary.log).  -1: no secondary order.
static int copy_secondary_mode(sptk_tensor t, int mode, cudaStream_t s) {
    if (!opt(OPT_COPY_ORDER)) return -1;
    // SPTK_COPY_SEC=a0,a1,...: per-mode override (tuning; -1 = none)
    if (const char *o = getenv("SPTK_COPY_SEC")) {
        int m = 0, v = 0, neg = 0, have = 0;
        for (const char *c = o;; ++c) {
            if (*c == '-') neg = 1;
            else if (*c >= '0' && *c <= '9') v = v * 10 + (*c - '0'), have = 1;
            else {
                if (m == mode && have) {
                    const int a = neg ? -v : v;
                    return (a >= 0 && a < t->N && a != mode) ? a : -1;
                }
                ++m;
                v = neg = have = 0;
                if (!*c) break;
            }
        }
    }
    const int64_t mx = row_max(t, mode, s);
    const bool imbalanced = opt(OPT_COPY_ORDER) == 1 && mx >= 0 && mx * t->dims[mode] > 2 * t->P;
    int a = -1;
    for (int m = 0; m < t->N; ++m) {
        if (m == mode || t->dims[m] < 2048) continue;
        if (a < 0 || (imbalanced ? t->dims[m] > t->dims[a] : t->dims[m] < t->dims[a])) a = m;
    }
    return a;
}

// Materialise the compact permuted copy of `mode` unless the tensor keeps the
// paper's perm-gather traversal or the copy would leave less than the reserve
// free (then that mode keeps gathering through perm_n).  Copies are caches:
// build_perm releases them if a sort needs their memory.
//
// Copy order: sorted by l_n like perm_n (same rows, same row segments, same
// rowptr_n), but inside a row by the secondary mode a's index, then storage
// order -- the stable sort by l_n of perm_a.  Nonzeros of one row that share
// l_a are then adjacent and their A_a row is gathered once into L1 instead of
// once per nonzero; the row's sum is the same up to summation order.
sptk_status ensure_sorted_copy(sptk_tensor t, int mode, cudaStream_t s) {
    if (t->has_srec[mode] || t->perm_gather_only || t->P == 0 || !t->has_perm[mode] ||
        t->copy_declined[mode])
        return SPTK_OK;
    // positions covered: all, or this shard's row range (sptk_sptensor_set_shard)
    int64_t p0 = 0, p1 = t->P;
    if (t->shard_n > 1) {
        SPTK_TRY(host_rowptr(t, mode, s));
        std::vector<int64_t> b((size_t)t->shard_n + 1);
        SPTK_TRY(sptk_partition_rows(t->host_rowptr[mode].data(), t->dims[mode], t->shard_n,
                                     b.data()));
        p0 = t->host_rowptr[mode][b[t->shard_r]];
        p1 = t->host_rowptr[mode][b[t->shard_r + 1]];
    }
    const bool whole = p0 == 0 && p1 == t->P;
    const int rc = compact_bytes(t->dtype, t->N);
    const size_t need = (size_t)rc * (size_t)std::max<int64_t>(p1 - p0, 1);
    size_t free_b = 0, total_b = 0;
    if (!device_free(t, &free_b, &total_b)) return SPTK_OK;
    const size_t reserve = std::max<size_t>(total_b / 32, (size_t)4 << 30);
    int a = copy_secondary_mode(t, mode, s);
    if (a >= 0 && !t->has_perm[a]) a = -1;
    // The secondary sort (over all P ids) runs inside the copy's own buffer
    // (>= 16 B = 4 words per nonzero, the sort needs ~3.1) before the copy
    // overwrites it; a shard's smaller copy uses the cached sort workspace
    // instead.  Only the order itself (4 B per nonzero) is extra.
    const size_t order_bytes = a >= 0 ? sizeof(uint32_t) * (size_t)t->P : 0;
    const bool ws_in_copy = whole && sizeof(uint32_t) * sort_ws_words(t->P) <= need;
    if (a >= 0 && !ws_in_copy && !t->sortws.p) a = -1;
    // the order lives in the idle sort workspace when the sort does not need it
    size_t extra = (ws_in_copy && t->sortws.p && t->sortws.bytes >= order_bytes) ? 0 : order_bytes;
    if (free_b < need + extra + reserve && t->sortws.p && (ws_in_copy || a < 0)) {
        free_b += t->sortws.bytes;  // the sort workspace is a cache too
        t->sortws.release();
        extra = order_bytes;
        if (!ws_in_copy) a = -1;
    }
    if (free_b < need + extra + reserve) {
        a = -1;
        if (free_b < need + reserve && t->sortws.p) {
            free_b += t->sortws.bytes;
            t->sortws.release();
        }
    }
    if (free_b < need + reserve && t->keys.p) {  // the resident ingest keys are a cache too
        free_b += t->keys.bytes;
        t->keys.release();
    }
    // declined: remembered, so later MTTKRPs of this mode do not query the
    // free memory again (a host stall while kernels are in flight) -- cleared
    // when memory is released (drop_copies) or the mode is re-sorted
    if (free_b < need + reserve) {
        t->copy_declined[mode] = true;
        return SPTK_OK;
    }
    if (t->srec[mode].reserve(need) != SPTK_OK) {
        set_error("");
        t->copy_declined[mode] = true;
        return SPTK_OK;
    }
    const uint32_t *order = t->perm[mode].as<uint32_t>();
    DevBuf ord;
    uint32_t *ordp = nullptr;
    if (a >= 0) {
        if (ws_in_copy && t->sortws.p && t->sortws.bytes >= order_bytes) ordp = t->sortws.as<uint32_t>();
        else if (ord.reserve(order_bytes) == SPTK_OK) ordp = ord.as<uint32_t>();
        else set_error("");
    }
    t->copy_sec[mode] = -1;
    t->copy_win[mode] = false;
    t->soff_key[mode][0] = -1;
    if (ordp) {
        SPTK_TRY(stable_sort_ids(t, mode, t->perm[a].as<uint32_t>(), ordp, nullptr, s,
                                 ws_in_copy ? t->srec[mode].p : nullptr, ws_in_copy ? need : 0));
        order = ordp;
        t->copy_sec[mode] = a;
    }
    // Window-major order (option win; SURVEY §8(a) a4-a5 on power-law tensors):
    // for a mode with few output rows whose secondary factor far exceeds L2,
    // the (l_n, l_a) order is re-sorted stably by the window of l_a (2^wshift
    // rows of A_a, an L2-sized slice at 128-byte rows), giving (window, l_n,
    // l_a).  The cooperative kernel then streams the copy in order with short
    // per-warp chunks, so the positions in flight gather A_a rows from about
    // one window, which stays in L2; every row is reached once per window and
    // flushed with red.add (I_n x windows flushes, few when I_n is small).
    const int vwd = dtype_bytes(t->dtype) / 4;
    if (ordp && opt(OPT_WIN) && !t->deterministic && whole && rc / 4 >= vwd + t->N) {
        int wshift = 0;
        const int64_t wrows = std::max<int64_t>(1, (int64_t)opt(OPT_SLICE_L2_KB) * 1024 / 128);
        while (((int64_t)2 << wshift) <= wrows) ++wshift;
        const int64_t nwin = (t->dims[a] + ((int64_t)1 << wshift) - 1) >> wshift;
        if (nwin >= 2 * (int64_t)opt(OPT_WIN) && t->dims[mode] * nwin * 64 <= t->P) {
            DevBuf ord2;
            if (ord2.reserve(order_bytes) == SPTK_OK) {
                SPTK_TRY(stable_sort_ids(t, a, ordp, ord2.as<uint32_t>(), nullptr, s,
                                         ws_in_copy ? t->srec[mode].p : nullptr,
                                         ws_in_copy ? need : 0, wshift));
                SPTK_CUDA(cudaMemcpyAsync(ordp, ord2.p, order_bytes, cudaMemcpyDeviceToDevice, s));
                SPTK_CUDA(cudaStreamSynchronize(s));  // ord2 is freed on return
                t->copy_win[mode] = true;
            } else {
                set_error("");
            }
        }
    }
    const int vw = dtype_bytes(t->dtype) / 4;
    const int64_t np = p1 - p0;
    const unsigned g = (unsigned)grid_for(std::max<int64_t>(np, 1));
    uint8_t *dst = t->srec[mode].as<uint8_t>();
    const uint8_t *src = t->rec.as<uint8_t>();
    if (np > 0) {
        if (t->rec_bytes == 32 && rc == 32)
            permute_records<32, 32><<<g, 256, 0, s>>>(src, order + p0, np, vw, t->N, mode, dst);
        else if (t->rec_bytes == 32)
            permute_records<32, 16><<<g, 256, 0, s>>>(src, order + p0, np, vw, t->N, mode, dst);
        else
            permute_records<16, 16><<<g, 256, 0, s>>>(src, order + p0, np, vw, t->N, mode, dst);
        count_launch();
        SPTK_CUDA(cudaGetLastError());
    }
    if (ord.p) SPTK_CUDA(cudaStreamSynchronize(s));  // `ord` is freed on return
    t->copy_p0[mode] = p0;
    t->copy_p1[mode] = p1;
    t->copy_rowrec[mode] = rc / 4 >= vw + t->N;
    t->has_srec[mode] = true;
    return SPTK_OK;
}

// Would build_perm of modes [m0, m1) allocate anything?  (perm / rowptr of
// the mode, the sort workspace, a missing copy)
bool build_needs_memory(sptk_tensor t, int m0, int m1) {
    const int64_t P = t->P;
    if (P > 0 && (!t->sortws.p || t->sortws.bytes < sizeof(uint32_t) * sort_ws_words(P)))
        return true;
    for (int m = m0; m < m1; ++m) {
        if (!t->perm[m].p || t->perm[m].bytes < sizeof(uint32_t) * (size_t)std::max<int64_t>(P, 1))
            return true;
        if (!t->rowptr[m].p || t->rowptr[m].bytes < sizeof(uint32_t) * (size_t)(t->dims[m] + 1))
            return true;
        if (!t->has_srec[m] && !t->copy_declined[m] && !t->perm_gather_only && P > 0) return true;
    }
    return false;
}

void drop_copies(sptk_tensor t) {
    for (int m = 0; m < t->N; ++m) {
        t->srec[m].release();
        t->has_srec[m] = false;
        t->wrow[m].release();
        t->wrow_key[m][0] = -1;
        t->copy_sec[m] = -1;
        t->copy_win[m] = false;
        t->soff[m].release();
        t->soff_key[m][0] = -1;
        t->copy_declined[m] = false;
    }
}

// keys[i] = l_{in[i], mode}: the key of the i-th id of an input order
__global__ void __launch_bounds__(256) extract_keys_through(const uint8_t *__restrict__ rec, int rb,
                                                            int kw, const uint32_t *__restrict__ in,
                                                            int64_t P, uint32_t *__restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = __ldg(reinterpret_cast<const uint32_t *>(rec + (size_t)__ldg(in + i) * rb) + kw);
}

// keys[i] = key_n[in[i]] from the ingest keys (4-byte gathers, not 16/32-byte records)
__global__ void __launch_bounds__(256) gather_keys(const uint32_t *__restrict__ key_n,
                                                   const uint32_t *__restrict__ in, int64_t P,
                                                   uint32_t *__restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = __ldg(key_n + __ldg(in + i));
}

// Stable LSD radix sort of nonzero ids by l_{., mode}.  `in` is the input
// order of ids (NULL = storage order 0..P-1); the sorted ids go to `out` (must
// not alias `in`) and, if keys_out != NULL, the sorted keys to keys_out.
// Uses the handle's cached workspace.
// ext_ws (optional, >= sort_ws_words(P) words): scratch to use instead of the
// handle's cached workspace (the copy buffer about to be overwritten).
// kshift > 0: sort by l >> kshift only (the window index of the window-major
// copy order)
static sptk_status stable_sort_ids(sptk_tensor t, int mode, const uint32_t *in, uint32_t *out,
                                   uint32_t **keys_out, cudaStream_t s, void *ext_ws,
                                   size_t ext_bytes, int kshift) {
    const int64_t P = t->P, In = t->dims[mode];
    int bits = 0;
    while (bits < 32 && ((uint64_t)(In - 1) >> (bits + kshift)) != 0) ++bits;
    const int npass = bits == 0 ? 1 : (bits + 7) / 8;
    const int dbits = bits == 0 ? 1 : (bits + npass - 1) / npass;
    const int64_t ntiles = (P + kSortTile - 1) / kSortTile;
    // workspace (kept in the handle across calls; a cache like the permuted
    // copies): keys x2, values, digit counts, scan block sums
    const size_t nP = (size_t)P, ncnt = (size_t)ntiles * 256;
    const size_t ws_words = sort_ws_words(P);
    uint32_t *ws;
    if (ext_ws && ext_bytes >= sizeof(uint32_t) * ws_words) {
        ws = static_cast<uint32_t *>(ext_ws);
    } else {
        if (t->sortws.reserve(sizeof(uint32_t) * ws_words) != SPTK_OK) {
            drop_copies(t);  // permuted copies and ingest keys are caches: free them, retry
            t->keys.release();
            SPTK_TRY(t->sortws.reserve(sizeof(uint32_t) * ws_words));
        }
        ws = t->sortws.as<uint32_t>();
    }
    uint32_t *kA = ws, *kB = ws + nP, *vA = ws + 2 * nP, *counts = ws + 3 * nP;
    uint32_t *tmp = counts + ncnt;
    // ping-pong: vals end in `out` after the last pass
    uint32_t *kbuf[2] = {kA, kB};
    uint32_t *vbuf[2] = {vA, out};
    const int kw = dtype_bytes(t->dtype) / 4 + mode;
    // pass-0 keys: one pass over the records (kbuf of the other parity is free until then)
    uint32_t *k0 = kbuf[(npass - 1) & 1] == kA ? kB : kA;
    if (!in && t->keys.p) {
        k0 = t->keys.as<uint32_t>() + (size_t)mode * P;  // emitted at ingest (pack.cu)
    } else if (in && t->keys.p)
        gather_keys<<<grid_for(P), 256, 0, s>>>(t->keys.as<uint32_t>() + (size_t)mode * P, in, P, k0);
    else if (in)
        extract_keys_through<<<grid_for(P), 256, 0, s>>>(t->rec.as<uint8_t>(), t->rec_bytes, kw, in,
                                                         P, k0);
    else
        extract_keys<<<grid_for(P), 256, 0, s>>>(t->rec.as<uint8_t>(), t->rec_bytes, kw, P, k0);
    if (in || !t->keys.p) {  // a key kernel ran
        count_launch();
        SPTK_CUDA(cudaGetLastError());
    }
    const uint32_t *kin = k0, *vin = in;
    for (int p = 0; p < npass; ++p) {
        const int db = bits == 0 ? 1 : ((p * dbits + dbits > bits) ? bits - p * dbits : dbits);
        const int shift = kshift + p * dbits;
        uint32_t *kout = kbuf[(npass - 1 - p) & 1];
        uint32_t *vout = vbuf[((npass - 1 - p) & 1) ^ 1];
        radix_upsweep<<<(unsigned)ntiles, kSortThreads, 0, s>>>(kin, (uint32_t)P, shift, db,
                                                                (uint32_t)ntiles, counts);
        count_launch();
        SPTK_CUDA(cudaGetLastError());
        SPTK_TRY(exclusive_scan(counts, ntiles * ((int64_t)1 << db), tmp, s));
        if (opt(OPT_SORT_V1)) {
            radix_downsweep<<<(unsigned)ntiles, kSortThreads, 0, s>>>(
                kin, vin, (uint32_t)P, shift, db, (uint32_t)ntiles, counts, kout, vout);
        } else {
            // the last pass writes the keys only if the caller wants them
            const bool keys_needed = keys_out || p + 1 < npass;
            SPTK_CUDA(launch_downsweep2(db, (unsigned)ntiles, s, kin, vin, (uint32_t)P, shift,
                                        (uint32_t)ntiles, counts, keys_needed ? kout : nullptr,
                                        vout));
        }
        count_launch();
        SPTK_CUDA(cudaGetLastError());
        kin = kout;
        vin = vout;
    }
    if (keys_out) *keys_out = const_cast<uint32_t *>(kin);
    return SPTK_OK;
}

sptk_status build_perm_mode(sptk_tensor t, int mode, cudaStream_t s) {
    const int64_t P = t->P, In = t->dims[mode];
    SPTK_TRY(t->perm[mode].reserve(sizeof(uint32_t) * (P > 0 ? P : 1)));
    SPTK_TRY(t->rowptr[mode].reserve(sizeof(uint32_t) * (In + 1)));
    uint32_t *perm = t->perm[mode].as<uint32_t>();
    uint32_t *rowptr = t->rowptr[mode].as<uint32_t>();
    t->host_rowptr[mode].clear();
    t->row_max[mode] = -1;
    t->wrow_key[mode][0] = -1;
    t->copy_declined[mode] = false;
    if (P == 0) {
        SPTK_CUDA(cudaMemsetAsync(rowptr, 0, sizeof(uint32_t) * (In + 1), s));
        t->has_perm[mode] = true;
        return SPTK_OK;
    }
    if (In == 1) {  // every key is 0, the stable order is the identity
        iota_kernel<<<grid_for(P), 256, 0, s>>>(perm, P);
        fill_u32<<<1, 32, 0, s>>>(rowptr, 1, 0u);
        fill_u32<<<1, 32, 0, s>>>(rowptr + 1, 1, (uint32_t)P);
        count_launch(3);
        SPTK_CUDA(cudaGetLastError());
        t->has_perm[mode] = true;
        t->row_max[mode] = P;  // the single row holds every nonzero
        return SPTK_OK;
    }
    uint32_t *keys = nullptr;
    SPTK_TRY(stable_sort_ids(t, mode, nullptr, perm, &keys, s));
    rowptr_from_sorted<<<grid_for(In + 1), 256, 0, s>>>(keys, P, In, rowptr);
    SPTK_TRY(t->rowmax_dev.reserve(sizeof(uint32_t) * kMaxModes));
    SPTK_CUDA(cudaMemsetAsync(t->rowmax_dev.as<uint32_t>() + mode, 0, sizeof(uint32_t), s));
    row_max_kernel<<<grid_for(In), 256, 0, s>>>(rowptr, In, t->rowmax_dev.as<uint32_t>() + mode);
    count_launch(2);
    SPTK_CUDA(cudaGetLastError());
    t->has_perm[mode] = true;
    return SPTK_OK;
}

// ------------------------------------------------------------ duplicates
// Coordinates of ids L[i] and L[i-1] equal? (L in lexicographic order)
__device__ __forceinline__ bool same_coords(const uint8_t *rec, int rb, int kw0, int N, uint32_t a,
                                            uint32_t b) {
    const uint32_t *ra = reinterpret_cast<const uint32_t *>(rec + (size_t)a * rb) + kw0;
    const uint32_t *rbp = reinterpret_cast<const uint32_t *>(rec + (size_t)b * rb) + kw0;
    for (int m = 0; m < N; ++m)
        if (ra[m] != rbp[m]) return false;
    return true;
}

// keep[p] = 1 iff storage position p is the first occurrence of its coordinate
// (the head of its run in lexicographic order L; ties are in storage order, so
// the head is the earliest); sumv[p] = sum of the run's values in storage order
template <typename T>
__global__ void dup_heads_kernel(const uint8_t *__restrict__ rec, int rb, int N,
                                 const uint32_t *__restrict__ L, int64_t P,
                                 uint32_t *__restrict__ keep, T *__restrict__ sumv,
                                 int *__restrict__ any_dup) {
    const int kw0 = sizeof(T) / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t p = L[i];
        const bool head = i == 0 || !same_coords(rec, rb, kw0, N, p, L[i - 1]);
        keep[p] = head ? 1u : 0u;
        if (!head) {
            *any_dup = 1;
            continue;
        }
        T s = *reinterpret_cast<const T *>(rec + (size_t)p * rb);
        for (int64_t j = i + 1; j < P && same_coords(rec, rb, kw0, N, p, L[j]); ++j)
            s += *reinterpret_cast<const T *>(rec + (size_t)L[j] * rb);
        sumv[p] = s;
    }
}

// compact the kept records (storage order) with their merged values
template <typename T>
__global__ void dup_compact_kernel(const uint8_t *__restrict__ rec, int rb, int64_t P,
                                   const uint32_t *__restrict__ keep,
                                   const uint32_t *__restrict__ newidx,
                                   const T *__restrict__ sumv, uint8_t *__restrict__ out,
                                   double *__restrict__ partial) {
    __shared__ double sh[256];
    double sq = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        if (!keep[p]) continue;
        uint8_t *d = out + (size_t)newidx[p] * rb;
        const uint4 *srcv = reinterpret_cast<const uint4 *>(rec + (size_t)p * rb);
        uint4 *dv = reinterpret_cast<uint4 *>(d);
        dv[0] = srcv[0];
        if (rb == 32) dv[1] = srcv[1];
        *reinterpret_cast<T *>(d) = sumv[p];
        sq += (double)sumv[p] * (double)sumv[p];
    }
    sh[threadIdx.x] = sq;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

sptk_status launch_sum_f64(const double *in, int64_t n, double *out, cudaStream_t s);

// SPTK_CREATE_DUP_SUM / DUP_ERROR: lexicographic stable order by chaining
// stable sorts from the last mode to the first, heads of equal-coordinate
// runs keep their storage position and the run's value sum.
sptk_status merge_duplicates(sptk_tensor t, bool error_only, cudaStream_t s) {
    const int64_t P = t->P;
    if (P <= 1) return SPTK_OK;
    DevBuf o1, o2, keep, sumv, flag;
    SPTK_TRY(o1.reserve(sizeof(uint32_t) * P));
    SPTK_TRY(o2.reserve(sizeof(uint32_t) * P));
    uint32_t *cur = nullptr, *nxt = o1.as<uint32_t>(), *spare = o2.as<uint32_t>();
    for (int m = t->N - 1; m >= 0; --m) {
        SPTK_TRY(stable_sort_ids(t, m, cur, nxt, nullptr, s));
        cur = nxt;
        nxt = spare;
        spare = cur;
    }
    const uint32_t *L = cur;
    SPTK_TRY(keep.reserve(sizeof(uint32_t) * (P + 1)));
    SPTK_TRY(sumv.reserve((size_t)dtype_bytes(t->dtype) * P));
    SPTK_TRY(flag.reserve(64));
    SPTK_CUDA(cudaMemsetAsync(flag.p, 0, 64, s));
    int *any = flag.as<int>();
    if (t->dtype == SPTK_F64)
        dup_heads_kernel<double><<<grid_for(P), 256, 0, s>>>(t->rec.as<uint8_t>(), t->rec_bytes,
                                                             t->N, L, P, keep.as<uint32_t>(),
                                                             sumv.as<double>(), any);
    else
        dup_heads_kernel<float><<<grid_for(P), 256, 0, s>>>(t->rec.as<uint8_t>(), t->rec_bytes,
                                                            t->N, L, P, keep.as<uint32_t>(),
                                                            sumv.as<float>(), any);
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    int h_any = 0;
    SPTK_CUDA(cudaMemcpyAsync(&h_any, any, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPTK_CUDA(cudaStreamSynchronize(s));
    if (!h_any) return SPTK_OK;
    if (error_only) return fail(SPTK_EDUP, "duplicate coordinates (SPTK_CREATE_DUP_ERROR)");
    // new index of each kept record: exclusive scan of keep (storage order)
    DevBuf newidx, tmp, out, part;
    SPTK_TRY(newidx.reserve(sizeof(uint32_t) * (P + 1)));
    SPTK_CUDA(cudaMemcpyAsync(newidx.p, keep.p, sizeof(uint32_t) * P, cudaMemcpyDeviceToDevice, s));
    SPTK_CUDA(cudaMemsetAsync(newidx.as<uint32_t>() + P, 0, sizeof(uint32_t), s));
    SPTK_TRY(tmp.reserve(sizeof(uint32_t) * ((P + 1 + kScanChunk - 1) / kScanChunk + 1)));
    SPTK_TRY(exclusive_scan(newidx.as<uint32_t>(), P + 1, tmp.as<uint32_t>(), s));
    uint32_t newP = 0;
    SPTK_CUDA(cudaMemcpyAsync(&newP, newidx.as<uint32_t>() + P, sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, s));
    SPTK_CUDA(cudaStreamSynchronize(s));
    SPTK_TRY(out.reserve((size_t)t->rec_bytes * (newP > 0 ? newP : 1)));
    const int blocks = grid_for(P);
    SPTK_TRY(part.reserve(sizeof(double) * (blocks + 1)));
    if (t->dtype == SPTK_F64)
        dup_compact_kernel<double><<<blocks, 256, 0, s>>>(
            t->rec.as<uint8_t>(), t->rec_bytes, P, keep.as<uint32_t>(), newidx.as<uint32_t>(),
            sumv.as<double>(), out.as<uint8_t>(), part.as<double>());
    else
        dup_compact_kernel<float><<<blocks, 256, 0, s>>>(
            t->rec.as<uint8_t>(), t->rec_bytes, P, keep.as<uint32_t>(), newidx.as<uint32_t>(),
            sumv.as<float>(), out.as<uint8_t>(), part.as<double>());
    count_launch();
    SPTK_CUDA(cudaGetLastError());
    SPTK_TRY(launch_sum_f64(part.as<double>(), blocks, part.as<double>() + blocks, s));
    double normX2 = 0.0;
    SPTK_CUDA(cudaMemcpyAsync(&normX2, part.as<double>() + blocks, sizeof(double),
                              cudaMemcpyDeviceToHost, s));
    SPTK_CUDA(cudaStreamSynchronize(s));
    std::swap(t->rec.p, out.p);
    std::swap(t->rec.bytes, out.bytes);
    t->P = newP;
    t->normX2 = normX2;
    t->sortws.release();  // sized for the old P
    return SPTK_OK;
}

}  // namespace sptk
