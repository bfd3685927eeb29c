// gs_bin_sort.cu -- O11: duplicate each projected record
// into one pair per 16x16 tile of its rectangle, order every tile's pairs by
// (depth_bits, gid) and emit lower-bound tile ranges.  P:132 "tile-based
// rasterization"; "Tile size 16x16; front-to-back sort by primitive
// depth per tile with stable index tiebreak"; readings Q10, Q12, Q13, Q22.
//
// Design (B200, no global radix sort): the range table IS the exclusive scan
// of a per-tile histogram, so the sort is only needed inside each tile:
//   1. count    : per record, histogram over the tiles of its rectangle (on-chip
//                 per CTA chunk, merged with one global atomic per non-zero bin)
//   2. scan     : exclusive scan -> ranges [start, end) and scatter cursors
//   3. scatter  : per record, {depth_bits, record slot, gid} into its tiles'
//                 buckets (order inside a bucket is arbitrary)
//   4. tile sort: one WARP per tile sorts up to 512 pairs in registers
//                 (bitonic network, keys held transposed so most steps are
//                 in-register; (depth - min depth | gid | bucket index) packed
//                 in one 64-bit key when it fits, so the payload rides in the
//                 key; else a 64-bit key + 32-bit payload).  Longer tiles go to a
//                 persistent CTA pass: shared-memory bitonic up to 8192, then
//                 merge-path merges in global memory for the rare longer lists
//                 (coarse pyramid levels).
// (depth_bits, gid) keys are unique inside a tile, so the result is canonical
// and bit-identical run to run whatever order the atomics produced.
#include <algorithm>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER_THREAD = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_PER_THREAD;
constexpr int WARP_SORT_MAX = 512;      // 16 keys per lane
constexpr int SMEM_SORT_MAX = 2048;     // run length sorted on chip (2 padded buffers: 52 KB)
constexpr int BIG_THREADS = 128;        // 4 warps per long list (throughput mode)
constexpr int LAT_THREADS = 512;        // 16 warps per list > 256 (latency mode, small batches)
constexpr int64_t LAT_TILES = 16384;    // batches with at most this many tiles use latency mode
constexpr uint64_t PAD_KEY = ~0ull;

struct BinWs {
    uint32_t* counts;
    uint32_t* cursor;
    unsigned long long* block_sums;
    uint32_t* big_count;   // [0] mid list size, [1] big list size
    uint32_t* mid_list;
    uint32_t* big_list;
    uint32_t* cls_list;    // [5][T]: tiles of 2-32, 33-64, 65-128, 129-256, 513-1024 pairs (throughput mode)
    uint4* bucket;
    uint64_t* ka;
    uint32_t* va;
    uint64_t* kb;
    uint32_t* vb;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

BinWs carve(void* ws, int64_t cap, int64_t T) {
    char* p = static_cast<char*>(ws);
    BinWs w;
    const int64_t nb = (T + SCAN_TILE - 1) / SCAN_TILE + 1;
    w.counts = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * T);
    w.cursor = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * T);
    w.block_sums = reinterpret_cast<unsigned long long*>(p); p += align256(sizeof(unsigned long long) * nb);
    w.big_count = reinterpret_cast<uint32_t*>(p); p += 256;
    w.mid_list = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * T);
    w.big_list = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * T);
    w.cls_list = reinterpret_cast<uint32_t*>(p); p += 5 * align256(sizeof(uint32_t) * T);
    w.bucket = reinterpret_cast<uint4*>(p); p += align256(sizeof(uint4) * cap);
    w.ka = reinterpret_cast<uint64_t*>(p); p += align256(sizeof(uint64_t) * cap);
    w.va = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * cap);
    w.kb = reinterpret_cast<uint64_t*>(p); p += align256(sizeof(uint64_t) * cap);
    w.vb = reinterpret_cast<uint32_t*>(p); p += align256(sizeof(uint32_t) * cap);
    return w;
}

size_t ws_bytes(int64_t cap, int64_t T) {
    const int64_t nb = (T + SCAN_TILE - 1) / SCAN_TILE + 1;
    return align256(sizeof(uint32_t) * T) * 2 + align256(sizeof(unsigned long long) * nb) + 256 +
           7 * align256(sizeof(uint32_t) * T) + align256(sizeof(uint4) * cap) +
           2 * (align256(sizeof(uint64_t) * cap) + align256(sizeof(uint32_t) * cap));
}

// ---------------------------------------------------------------- 1. count
// One CTA per (view, contiguous chunk of its records).  When the view's tile
// grid fits in shared memory the CTA histograms its chunk on chip and merges
// the non-zero bins with one global atomic each (few global atomics even for a
// single view where every counter is hot); otherwise it falls back to one
// global reduction per pair.
constexpr int BIN_THREADS = 512;
#ifndef GS_BIN_MINB
#define GS_BIN_MINB 2                  // count / scatter CTAs per SM the register budget is sized for (r2: 3 -> 2, C5 -0.16 ms)
#endif
#ifndef GS_CLS_GRID
#define GS_CLS_GRID 16                 // class-sort CTAs per SM (persistent, 8 warps each; r2: 8 -> 16)
#endif
#ifndef GS_MID_GRID
#define GS_MID_GRID 8                  // mid-sort CTAs per SM (r2: 4 -> 8)
#endif
#ifndef GS_BIN_CTAS_PER_SM
#define GS_BIN_CTAS_PER_SM 32                // r2: 8 -> 32 (C4 bin_sort 4.48 -> 4.18 ms, C5 11.51 -> 11.02)
#endif
constexpr int HIST_MAX = 16384;   // tiles per view handled on chip (64 KB)

__device__ __forceinline__ void chunk_of(uint32_t nv, uint32_t& k0, uint32_t& k1) {
    const uint32_t per = (nv + gridDim.x - 1) / gridDim.x;
    k0 = min(nv, blockIdx.x * per);
    k1 = min(nv, k0 + per);
}

// p / nx and p % nx for the flattened (tile) index p of a rectangle nx tiles wide without a
// per-tile integer division: m = ceil(2^32 / nx) = floor((2^32 - 1) / nx) + 1 (one 32-bit
// division per record), q = (p m) >> 32 is exact for p nx < 2^32 (rectangles < 2^16 wide and long)
__device__ __forceinline__ uint64_t div_magic(uint32_t nx) { return (uint64_t)(0xffffffffu / nx) + 1u; }
__device__ __forceinline__ uint32_t div_by(uint32_t p, uint64_t m) { return (uint32_t)(((uint64_t)p * m) >> 32); }

__device__ __forceinline__ void rect_of(const uint4& q3, uint32_t& x0, uint32_t& y0, uint32_t& nx, uint32_t& npair) {
    x0 = q3.z & 0xffffu;
    y0 = q3.w & 0xffffu;
    nx = (q3.z >> 16) - x0 + 1;
    npair = nx * ((q3.w >> 16) - y0 + 1);
}

__global__ void __launch_bounds__(BIN_THREADS, GS_BIN_MINB)
count_kernel(gs_record* __restrict__ rec, int64_t cap, const uint32_t* __restrict__ n_rec,
             const gs_view* __restrict__ views, uint32_t* __restrict__ counts, const uint32_t* __restrict__ status,
             int tight, uint32_t* __restrict__ chunk_base, int cb_stride) {
    if (*status & GS_STATUS_RECORD_OVERFLOW) return;
    extern __shared__ uint32_t hist[];
    const int v = blockIdx.y;
    const uint32_t nv = min((uint64_t)n_rec[v], (uint64_t)cap);
    const uint32_t toff = views[v].tile_offset;
    const int TX = view_tiles_x(views[v]);
    const int Tv = TX * ((views[v].height + GS_TILE - 1) / GS_TILE);
    const bool onchip = Tv <= HIST_MAX;
    uint32_t k0, k1;
    chunk_of(nv, k0, k1);
    if (k0 >= k1) return;
    if (onchip) {
        for (int t = threadIdx.x; t < Tv; t += blockDim.x) hist[t] = 0u;
        __syncthreads();
    }
    auto bump = [&](uint32_t t) {
        GS_DCHECK(t < (uint32_t)Tv);
        if (onchip) atomicAdd(&hist[t], 1u);
        else atomicAdd(&counts[toff + t], 1u);
    };
    if (!tight) {
        for (uint32_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
            const uint4 q3 = __ldg(reinterpret_cast<const uint4*>(rec + (int64_t)v * cap + k) + 3);
            uint32_t x0, y0, nx, np;
            rect_of(q3, x0, y0, nx, np);
            const uint32_t ny = nx ? np / nx : 0u;
            for (uint32_t ty = y0; ty < y0 + ny; ++ty)
                for (uint32_t tx = x0; tx < x0 + nx; ++tx) bump(ty * TX + tx);
        }
    } else {
        // N3 (reading Q30): decide every (record, tile) of rectangles of <= 31 tiles with
        // the whole warp -- the warp's 32 records' tiles are flattened over the lanes --
        // and store the decision as the record's tile_mask for the scatter pass
        __shared__ TightRec tr[BIN_THREADS];
        __shared__ uint32_t trect[BIN_THREADS], tnx[BIN_THREADS], tpre[BIN_THREADS], tmask[BIN_THREADS];
        __shared__ uint64_t tdiv[BIN_THREADS];
        const uint32_t lane = threadIdx.x & 31u, wb = threadIdx.x & ~31u;
        for (uint32_t kb = k0 + wb; kb < k1; kb += blockDim.x) {
            const uint32_t k = kb + lane;
            gs_record* r = rec + (int64_t)v * cap + k;
            uint32_t x0 = 0, y0 = 0, nx = 1, np = 0, small = 0;
            if (k < k1) {
                const uint4 q3 = __ldg(reinterpret_cast<const uint4*>(r) + 3);
                rect_of(q3, x0, y0, nx, np);
                if (np <= 31u) {
                    tr[threadIdx.x] = tight_of(r);
                    small = np;
                }
            }
            trect[threadIdx.x] = x0 | (y0 << 16);
            tnx[threadIdx.x] = nx;
            tdiv[threadIdx.x] = div_magic(nx);
            tmask[threadIdx.x] = 0u;
            uint32_t inc = small;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if ((int)lane >= o) inc += y;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
            tpre[threadIdx.x] = inc - small;
            __syncwarp();
            for (uint32_t idx = lane; idx < total; idx += 32u) {
                // owner: the last record of the warp whose exclusive prefix is <= idx
                uint32_t lo = 0;
#pragma unroll
                for (uint32_t step = 16; step; step >>= 1)
                    if (tpre[wb + lo + step] <= idx) lo += step;
                const uint32_t o = wb + lo, p = idx - tpre[o], nxo = tnx[o], rx = trect[o];
                const uint32_t pq = div_by(p, tdiv[o]);
                const uint32_t tx = (rx & 0xffffu) + (p - pq * nxo), ty = (rx >> 16) + pq;
                if (tile_hit(tr[o], tx, ty)) {
                    atomicOr(&tmask[o], 1u << p);
                    bump(ty * TX + tx);
                }
            }
            __syncwarp();
            if (k < k1) {
                uint32_t m = tmask[threadIdx.x];
                if (np > 31u) {   // large rectangle: decided per tile here and again in the scatter
                    m = GS_TILE_MASK_FULL;
                    const TightRec g = tight_of(r);
                    const uint32_t ny = np / nx;
                    for (uint32_t ty = y0; ty < y0 + ny; ++ty)
                        for (uint32_t tx = x0; tx < x0 + nx; ++tx)
                            if (tile_hit(g, tx, ty)) bump(ty * TX + tx);
                }
                r->tile_mask = m;
            }
            __syncwarp();
        }
    }
    if (onchip) {
        __syncthreads();
        // with chunk_base: keep this chunk's offset inside every tile's range (the scatter
        // then needs no second histogram pass)
        uint32_t* cb = chunk_base ? chunk_base + ((int64_t)v * gridDim.x + blockIdx.x) * cb_stride : nullptr;
        for (int t = threadIdx.x; t < Tv; t += blockDim.x) {
            const uint32_t c = hist[t];
            const uint32_t b = c ? atomicAdd(&counts[toff + t], c) : 0u;
            if (cb) cb[t] = b;
        }
    }
}

// ---------------------------------------------------------------- 2. scan
__device__ __forceinline__ unsigned long long block_exclusive_scan(unsigned long long x,
                                                                   unsigned long long* total) {
    __shared__ unsigned long long wsum[SCAN_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0ull;
        unsigned long long si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += y;
        }
        if (lane < (int)(blockDim.x >> 5)) wsum[lane] = si - s;
        if (lane == 31) *total = si;
    }
    __syncthreads();
    const unsigned long long r = wsum[warp] + inc - x;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_THREADS)
scan_reduce_kernel(const uint32_t* __restrict__ counts, int64_t T, unsigned long long* __restrict__ block_sums) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_PER_THREAD;
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k)
        if (base + k < T) s += counts[base + k];
    __shared__ unsigned long long tot;
    unsigned long long dummy = block_exclusive_scan(s, &tot);
    (void)dummy;
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

// single CTA: exclusive scan of block sums; writes n_pairs and the overflow bit
__global__ void __launch_bounds__(SCAN_THREADS)
scan_blocks_kernel(unsigned long long* __restrict__ block_sums, int64_t nb, uint64_t* __restrict__ n_pairs,
                   int64_t pair_cap, uint32_t* __restrict__ status) {
    __shared__ unsigned long long tot;
    unsigned long long carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += SCAN_THREADS) {
        const int64_t b = b0 + threadIdx.x;
        const unsigned long long x = b < nb ? block_sums[b] : 0ull;
        const unsigned long long ex = block_exclusive_scan(x, &tot);
        if (b < nb) block_sums[b] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *n_pairs = carry;
        if ((int64_t)carry > pair_cap) atomicOr(status, GS_STATUS_PAIR_OVERFLOW);
    }
}

__global__ void __launch_bounds__(SCAN_THREADS)
scan_down_kernel(const uint32_t* __restrict__ counts, int64_t T, const unsigned long long* __restrict__ block_sums,
                 uint32_t* __restrict__ ranges, uint32_t* __restrict__ cursor) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_PER_THREAD;
    uint32_t c[SCAN_PER_THREAD];
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        c[k] = base + k < T ? counts[base + k] : 0u;
        s += c[k];
    }
    __shared__ unsigned long long tot;
    unsigned long long run = block_sums[blockIdx.x] + block_exclusive_scan(s, &tot);
#pragma unroll
    for (int k = 0; k < SCAN_PER_THREAD; ++k) {
        if (base + k < T) {
            const uint32_t st = (uint32_t)run;
            ranges[2 * (base + k)] = st;
            ranges[2 * (base + k) + 1] = st + c[k];
            cursor[base + k] = st;
        }
        run += c[k];
    }
}

// ---------------------------------------------------------------- 3. scatter
// bucket entry: {depth_bits, record slot, gid, 0}; order inside a bucket is
// arbitrary.  On-chip path: histogram the chunk, reserve each non-zero bin's
// range with one global atomic, then place pairs with shared-memory atomics.
__global__ void __launch_bounds__(BIN_THREADS, GS_BIN_MINB)
scatter_kernel(const gs_record* __restrict__ rec, int64_t cap, const uint32_t* __restrict__ n_rec,
               const gs_view* __restrict__ views, uint32_t* __restrict__ cursor, uint4* __restrict__ bucket,
               const uint32_t* __restrict__ status, int tight, const uint32_t* __restrict__ chunk_base,
               int cb_stride, uint64_t pair_cap) {
    if (*status) return;
    extern __shared__ uint32_t hist[];
    const int v = blockIdx.y;
    const uint32_t nv = min((uint64_t)n_rec[v], (uint64_t)cap);
    const uint32_t toff = views[v].tile_offset;
    const int TX = view_tiles_x(views[v]);
    const int Tv = TX * ((views[v].height + GS_TILE - 1) / GS_TILE);
    const bool onchip = Tv <= HIST_MAX;
    uint32_t k0, k1;
    chunk_of(nv, k0, k1);
    if (k0 >= k1) return;
    if (onchip && chunk_base) {
        // this chunk's base in bucket t = tile start + the chunk's offset from count_kernel
        const uint32_t* cb = chunk_base + ((int64_t)v * gridDim.x + blockIdx.x) * cb_stride;
        for (int t = threadIdx.x; t < Tv; t += blockDim.x) hist[t] = cursor[toff + t] + cb[t];
        __syncthreads();
    } else if (onchip) {
        for (int t = threadIdx.x; t < Tv; t += blockDim.x) hist[t] = 0u;
        __syncthreads();
        for (uint32_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
            const gs_record* r = rec + (int64_t)v * cap + k;
            const uint4 q3 = __ldg(reinterpret_cast<const uint4*>(r) + 3);
            uint32_t x0, y0, nx, np;
            rect_of(q3, x0, y0, nx, np);
            if (tight) {
                const uint32_t tm = __ldg(&r->tile_mask);
                if (!(tm & GS_TILE_MASK_FULL)) {
                    const uint64_t dm = div_magic(nx);
                    for (uint32_t m = tm; m; m &= m - 1u) {
                        const uint32_t p = __ffs(m) - 1u, pq = div_by(p, dm);
                        atomicAdd(&hist[(y0 + pq) * TX + x0 + (p - pq * nx)], 1u);
                    }
                    continue;
                }
            }
            const TightRec g = tight ? tight_of(r) : TightRec{};
            const uint32_t ny = np / nx;
            for (uint32_t ty = y0; ty < y0 + ny; ++ty)
                for (uint32_t tx = x0; tx < x0 + nx; ++tx) {
                    if (tight && !tile_hit(g, tx, ty)) continue;
                    atomicAdd(&hist[ty * TX + tx], 1u);
                }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < Tv; t += blockDim.x) {
            const uint32_t c = hist[t];
            hist[t] = c ? atomicAdd(&cursor[toff + t], c) : 0u;   // this chunk's base in bucket t
        }
        __syncthreads();
    }
    // one record per thread and iteration; the next record's fields are loaded before
    // the current one's atomics and stores (the loop was bound by this load latency)
    uint32_t k = k0 + threadIdx.x;
    uint4 n1 = make_uint4(0u, 0u, 0u, 0u), n2 = n1, n3 = n1;
    auto fetch = [&](uint32_t kk) {
        const uint4* q4 = reinterpret_cast<const uint4*>(rec + (int64_t)v * cap + kk);
        n1 = __ldg(q4 + 1);
        n2 = __ldg(q4 + 2);
        n3 = __ldg(q4 + 3);
    };
    if (k < k1) fetch(k);
    for (; k < k1; k += blockDim.x) {
        const uint32_t slot = (uint32_t)((int64_t)v * cap + k);
        const uint4 q1 = n1, q2 = n2, q3 = n3;
        if (k + blockDim.x < k1) fetch(k + blockDim.x);
        const uint4 ent = make_uint4(q2.w, slot, q3.x, 0u);   // bits(z), slot, gid
        uint32_t x0, y0, nx, np;
        rect_of(q3, x0, y0, nx, np);
        if (tight) {
            const uint32_t tm = q1.w;                            // tile_mask
            if (!(tm & GS_TILE_MASK_FULL)) {
                const uint64_t dm = div_magic(nx);
                for (uint32_t m = tm; m;) {
                    uint32_t pos[4], pp[4];
                    int c = 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (m) {
                            pp[q] = __ffs(m) - 1u;
                            m &= m - 1u;
                            const uint32_t pq = div_by(pp[q], dm);
                            const uint32_t t = (y0 + pq) * TX + x0 + (pp[q] - pq * nx);
                            pos[q] = onchip ? atomicAdd(&hist[t], 1u) : atomicAdd(&cursor[toff + t], 1u);
                            c = q + 1;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (q < c) {
                            GS_DCHECK(pos[q] < pair_cap);
                            bucket[pos[q]] = ent;
                        }
                }
                continue;
            }
        }
        const TightRec g = tight ? tight_of(rec + slot) : TightRec{};
        const uint64_t dm = div_magic(nx);
        for (uint32_t p0 = 0; p0 < np; p0 += 4) {
            uint32_t pos[4];
            bool keep[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t p = p0 + q, pq = div_by(p, dm);
                const uint32_t tx = x0 + (p - pq * nx), ty = y0 + pq;
                keep[q] = p < np && (!tight || tile_hit(g, tx, ty));
                if (keep[q]) {
                    const uint32_t t = ty * TX + tx;
                    pos[q] = onchip ? atomicAdd(&hist[t], 1u) : atomicAdd(&cursor[toff + t], 1u);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (keep[q]) {
                    GS_DCHECK(pos[q] < pair_cap);
                    bucket[pos[q]] = ent;
                }
        }
    }
}

// ---------------------------------------------------------------- 4. tile sort
// The order is (depth_bits, gid) ascending (Q12).  Depth ties are frequent (an
// fp32 depth at 150 m has a 1.5e-5 m ulp), so gid is always part of the key.
// Fast path (per warp): pack (depth_bits - min_depth) | gid | bucket index into
// one 64-bit key when the tile's depth spread fits -- the payload rides in the
// key and a compare-exchange moves 64 bits.  Otherwise sort the 64-bit key
// (depth_bits << 32 | gid) with the bucket index as a 32-bit payload.

// warp bitonic of 32*PER keys held transposed: element e = lane*PER + j
template <int PER, bool PAY>
__device__ __forceinline__ void warp_bitonic_t(uint64_t (&k)[PER], uint32_t (&v)[PER], uint32_t lane) {
    constexpr int LP = PER == 1 ? 0 : PER == 2 ? 1 : PER == 4 ? 2 : PER == 8 ? 3 : PER == 16 ? 4 : 5;
    constexpr int LOGN = 5 + LP;
#pragma unroll
    for (int s = 1; s <= LOGN; ++s) {
#pragma unroll
        for (int d = s - 1; d >= 0; --d) {
            if (d < LP) {                         // partner in the same lane
                const int jd = 1 << d;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    if ((j & jd) == 0) {
                        // branch-free compare-exchange (selects, no divergent swap)
                        const uint32_t e = lane * PER + (uint32_t)j;
                        const bool up = ((e >> s) & 1u) == 0u;
                        const uint64_t a = k[j], b = k[j + jd];
                        const bool sw = (a > b) == up;
                        k[j] = sw ? b : a;
                        k[j + jd] = sw ? a : b;
                        if (PAY) {
                            const uint32_t va = v[j], vb = v[j + jd];
                            v[j] = sw ? vb : va;
                            v[j + jd] = sw ? va : vb;
                        }
                    }
                }
            } else {                              // partner lane = lane ^ 2^(d - LP)
                const uint32_t ld = 1u << (d - LP);
                const bool lower = (lane & ld) == 0u;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    // keep min(k, ok) when (lower == up), else max: one 64-bit compare + selects
                    const uint32_t e = lane * PER + (uint32_t)j;
                    const bool up = ((e >> s) & 1u) == 0u;
                    const uint64_t ok = __shfl_xor_sync(0xffffffffu, k[j], ld);
                    uint32_t ov = 0;
                    if (PAY) ov = __shfl_xor_sync(0xffffffffu, v[j], ld);
                    const bool lt = ok < k[j];                 // keys are unique (index / gid in the key)
                    const bool take = lt == (lower == up);
                    k[j] = take ? ok : k[j];
                    if (PAY) v[j] = take ? ov : v[j];
                }
            }
        }
    }
}

__device__ __forceinline__ uint32_t warp_min(uint32_t x) { return __reduce_min_sync(0xffffffffu, x); }
__device__ __forceinline__ uint32_t warp_max(uint32_t x) { return __reduce_max_sync(0xffffffffu, x); }

template <int PER>
__device__ __forceinline__ void warp_sort_tile(const uint4* __restrict__ bucket, uint32_t s, uint32_t len,
                                               uint32_t tile, uint32_t lane, uint2* __restrict__ stage,
                                               uint32_t* __restrict__ out, uint32_t* __restrict__ ogid,
                                               uint64_t* __restrict__ dbg) {
    constexpr int IB = 5 + (PER == 1 ? 0 : PER == 2 ? 1 : PER == 4 ? 2 : PER == 8 ? 3 : 4);   // index bits
    // coalesced load of (depth_bits, gid) through this warp's shared staging buffer, then read transposed
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t e = (uint32_t)j * 32u + lane;
        if (e < len) {
            const uint4 b = __ldg(&bucket[s + e]);
            stage[e] = make_uint2(b.x, b.z);
        }
    }
    __syncwarp();
    uint32_t dep[PER], gid[PER];
    uint32_t dmin = 0xffffffffu, dmax = 0u, gmax = 0u;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t e = lane * PER + (uint32_t)j;
        if (e < len) {
            const uint2 b = stage[e];
            dep[j] = b.x;
            gid[j] = b.y;
            dmin = min(dmin, b.x);
            dmax = max(dmax, b.x);
            gmax = max(gmax, b.y);
        } else {
            dep[j] = gid[j] = 0u;
        }
    }
    __syncwarp();
    dmin = warp_min(dmin);
    dmax = warp_max(dmax);
    gmax = warp_max(gmax);
    const int GB = 32 - __clz(gmax | 1u);          // bits to hold every gid of the tile
    const int DB = 64 - GB - IB;                   // bits left for the depth offset
    uint64_t k[PER];
    uint32_t v[PER];
    if (DB >= 32 || (uint64_t)(dmax - dmin) < (1ull << DB)) {
        const int sg = IB, sd = GB + IB;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t e = lane * PER + (uint32_t)j;
            k[j] = e < len ? (((uint64_t)(dep[j] - dmin) << sd) | ((uint64_t)gid[j] << sg) | e) : PAD_KEY;
        }
        warp_bitonic_t<PER, false>(k, v, lane);
#pragma unroll
        for (int j = 0; j < PER; ++j) v[j] = (uint32_t)k[j] & ((1u << IB) - 1u);
    } else {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t e = lane * PER + (uint32_t)j;
            k[j] = e < len ? (((uint64_t)dep[j] << 32) | gid[j]) : PAD_KEY;
            v[j] = e;
        }
        warp_bitonic_t<PER, true>(k, v, lane);
    }
    // write out in the transposed order via the staging buffer so global stores coalesce
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t e = lane * PER + (uint32_t)j;
        if (e < len) stage[e] = make_uint2(v[j], 0u);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const uint32_t e = (uint32_t)j * 32u + lane;
        if (e < len) {
            const uint4 b = __ldg(&bucket[s + stage[e].x]);   // L1-resident: this warp just read the bucket
            out[s + e] = b.y;
            if (ogid) ogid[s + e] = b.z;
            if (dbg) dbg[s + e] = ((uint64_t)tile << 32) | b.x;
        }
    }
    __syncwarp();
}

constexpr int SMALL_MAX = 256;   // warp_sort_kernel: PER <= 8

__global__ void __launch_bounds__(256)
warp_sort_kernel(const uint32_t* __restrict__ ranges, int64_t T, const uint4* __restrict__ bucket,
                 uint32_t* __restrict__ out, uint32_t* __restrict__ ogid, uint64_t* __restrict__ dbg,
                 uint32_t* __restrict__ lists_count, uint32_t* __restrict__ mid_list,
                 uint32_t* __restrict__ big_list, uint32_t mid_max, const uint32_t* __restrict__ status) {
    if (*status) return;
    __shared__ uint2 stage[8][SMALL_MAX];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const int64_t tile = (int64_t)blockIdx.x * 8 + warp;
    if (tile >= T) return;
    const uint32_t s = ranges[2 * tile], e = ranges[2 * tile + 1], len = e - s;
    if (len == 0) return;
    uint2* st = stage[warp];
    if (len == 1) {
        if (lane == 0) {
            const uint4 b = bucket[s];
            out[s] = b.y;
            if (ogid) ogid[s] = b.z;
            if (dbg) dbg[s] = ((uint64_t)tile << 32) | b.x;
        }
    } else if (len <= 32) warp_sort_tile<1>(bucket, s, len, (uint32_t)tile, lane, st, out, ogid, dbg);
    else if (len <= 64) warp_sort_tile<2>(bucket, s, len, (uint32_t)tile, lane, st, out, ogid, dbg);
    else if (len <= 128) warp_sort_tile<4>(bucket, s, len, (uint32_t)tile, lane, st, out, ogid, dbg);
    else if (len <= SMALL_MAX) warp_sort_tile<8>(bucket, s, len, (uint32_t)tile, lane, st, out, ogid, dbg);
    else if (lane == 0) {
        if (len <= mid_max) mid_list[atomicAdd(&lists_count[0], 1u)] = (uint32_t)tile;
        else big_list[atomicAdd(&lists_count[1], 1u)] = (uint32_t)tile;
    }
}

// Throughput mode: one thread per tile sorts it into a size-class list (warp-aggregated
// appends; single-pair tiles are written here directly), then one kernel per class
// runs the same warp sort for every tile of the class -- uniform work per warp and one
// code path per kernel (the mixed-size kernel above spent a fifth of its stalls on
// instruction fetch).  counts: [0] mid, [1] big, [2 + c] class c.
__global__ void __launch_bounds__(256)
classify_kernel(const uint32_t* __restrict__ ranges, int64_t T, const uint4* __restrict__ bucket,
                uint32_t* __restrict__ out, uint32_t* __restrict__ ogid, uint64_t* __restrict__ dbg,
                uint32_t* __restrict__ counts, uint32_t* __restrict__ mid_list, uint32_t* __restrict__ big_list,
                uint32_t* __restrict__ cls_list, uint32_t mid_max, const uint32_t* __restrict__ status) {
    if (*status) return;
    const int64_t tile = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31u;
    int cls = -1;
    if (tile < T) {
        const uint32_t st = ranges[2 * tile], len = ranges[2 * tile + 1] - st;
        if (len == 1) {
            const uint4 b = bucket[st];
            out[st] = b.y;
            if (ogid) ogid[st] = b.z;
            if (dbg) dbg[st] = ((uint64_t)tile << 32) | b.x;
        } else if (len >= 2) {
            cls = len <= 32 ? 2 : len <= 64 ? 3 : len <= 128 ? 4 : len <= SMALL_MAX ? 5 : len <= mid_max ? 0
                : len <= 1024u ? 6 : 1;
        }
    }
#pragma unroll
    for (int c = 0; c < 7; ++c) {
        const uint32_t m = __ballot_sync(0xffffffffu, cls == c);
        if (!m) continue;
        const uint32_t leader = __ffs(m) - 1u;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&counts[c], (uint32_t)__popc(m));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (cls == c) {
            uint32_t* list = c == 0 ? mid_list : c == 1 ? big_list : cls_list + (int64_t)(c - 2) * T;   // c = 6: 513..1024
            list[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)tile;
        }
    }
}

template <int PER>
__global__ void __launch_bounds__(256)
class_sort_kernel(const uint32_t* __restrict__ ranges, const uint4* __restrict__ bucket, uint32_t* __restrict__ out,
                  uint32_t* __restrict__ ogid, uint64_t* __restrict__ dbg, const uint32_t* __restrict__ count,
                  const uint32_t* __restrict__ list, const uint32_t* __restrict__ status) {
    if (*status) return;
    __shared__ uint2 stage[8][32 * PER];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t n = *count;
    for (uint32_t i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
        const uint32_t tile = list[i];
        const uint32_t s = ranges[2 * tile], len = ranges[2 * tile + 1] - s;
        warp_sort_tile<PER>(bucket, s, len, tile, lane, stage[warp], out, ogid, dbg);
    }
}

// 257..512 pairs: one warp per tile (PER = 16), persistent over the mid list
__global__ void __launch_bounds__(256)
mid_sort_kernel(const uint32_t* __restrict__ ranges, const uint4* __restrict__ bucket, uint32_t* __restrict__ out,
                uint32_t* __restrict__ ogid, uint64_t* __restrict__ dbg, const uint32_t* __restrict__ lists_count,
                const uint32_t* __restrict__ mid_list, const uint32_t* __restrict__ status) {
    if (*status) return;
    __shared__ uint2 stage[8][WARP_SORT_MAX];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t n = lists_count[0];
    for (uint32_t i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
        const uint32_t tile = mid_list[i];
        const uint32_t s = ranges[2 * tile], len = ranges[2 * tile + 1] - s;
        warp_sort_tile<16>(bucket, s, len, tile, lane, stage[warp], out, ogid, dbg);
    }
}

// merge sorted runs A = [a0, a0+na), B = [a0+na, a0+na+nb) of (key, val) into dst (unique keys)
__device__ void cta_merge(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv, uint64_t* __restrict__ dk,
                          uint32_t* __restrict__ dv, uint32_t a0, uint32_t na, uint32_t nb) {
    const uint32_t total = na + nb;
    const uint32_t per = (total + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(total, threadIdx.x * per), hi = min(total, lo + per);
    if (lo >= hi) return;
    const uint64_t* A = sk + a0;
    const uint64_t* B = sk + a0 + na;
    uint32_t ilo = lo > nb ? lo - nb : 0u, ihi = min(lo, na);
    while (ilo < ihi) {   // merge path: i elements of A among the first lo outputs
        const uint32_t i = (ilo + ihi) >> 1;
        if (A[i] < B[lo - i - 1]) ilo = i + 1; else ihi = i;
    }
    uint32_t i = ilo, j = lo - ilo;
    for (uint32_t o = lo; o < hi; ++o) {
        const bool takeA = j >= nb || (i < na && A[i] < B[j]);
        if (takeA) { dk[a0 + o] = A[i]; dv[a0 + o] = sv[a0 + i]; ++i; }
        else { dk[a0 + o] = B[j]; dv[a0 + o] = sv[a0 + na + j]; ++j; }
    }
}

// Long lists (> 512 pairs; dense areas and coarse pyramid levels): one CTA of
// 4 warps per tile.  Runs of up to 2048 (depth_bits << 32 | gid, bucket index)
// pairs are sorted in shared memory as 512-element warp register sorts
// (transposed bitonic, as in the warp path) followed by merge-path merges in
// shared memory; lists longer than 2048 merge those runs in global memory.
// Shared arrays are padded one slot every 16 elements so the transposed
// (lane*16 + j) register loads are (at most) 2-way bank conflicted.
__device__ __forceinline__ uint32_t pidx(uint32_t e) { return e + (e >> 4); }
constexpr int RUN_PAD = SMEM_SORT_MAX + SMEM_SORT_MAX / 16;

// one merge round over all adjacent run pairs of width w (padded shared arrays):
// every output element is placed independently (merge-path split of its pair +
// one comparison), so all threads stay busy however many pairs there are
__device__ void smem_merge_round(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv,
                                 uint64_t* __restrict__ dk, uint32_t* __restrict__ dv, uint32_t rl, uint32_t w) {
    for (uint32_t o = threadIdx.x; o < rl; o += blockDim.x) {
        const uint32_t a0 = o / (2 * w) * (2 * w);
        const uint32_t na = min(w, rl - a0);
        const uint32_t nb = a0 + na < rl ? min(w, rl - a0 - na) : 0u;
        const uint32_t j = o - a0, A = a0, B = a0 + na;
        // i = number of A elements among the first j outputs
        uint32_t ilo = j > nb ? j - nb : 0u, ihi = min(j, na);
        while (ilo < ihi) {
            const uint32_t i = (ilo + ihi) >> 1;
            if (sk[pidx(A + i)] < sk[pidx(B + j - i - 1)]) ilo = i + 1; else ihi = i;
        }
        const uint32_t i = ilo, jb = j - ilo;
        const bool takeA = jb >= nb || (i < na && sk[pidx(A + i)] < sk[pidx(B + jb)]);
        const uint32_t src = takeA ? A + i : B + jb;
        dk[pidx(o)] = sk[pidx(src)];
        dv[pidx(o)] = sv[pidx(src)];
    }
}

template <int PER>
__device__ void warp_runs(uint64_t* ak, uint32_t* av, uint32_t rl) {
    constexpr uint32_t RUN = 32u * PER;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const uint32_t nrun = (rl + RUN - 1) / RUN;
    for (uint32_t r = warp; r < nrun; r += nwarp) {
        uint64_t k[PER];
        uint32_t v[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t e = r * RUN + lane * PER + (uint32_t)j;
            k[j] = e < rl ? ak[pidx(e)] : PAD_KEY;
            v[j] = e < rl ? av[pidx(e)] : 0u;
        }
        warp_bitonic_t<PER, true>(k, v, lane);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const uint32_t e = r * RUN + lane * PER + (uint32_t)j;
            if (e < rl) { ak[pidx(e)] = k[j]; av[pidx(e)] = v[j]; }
        }
    }
}

// sort rl <= SMEM_SORT_MAX pairs already placed in (ak, av): warp register sorts of
// runs of `run` (32..512) elements, then merge rounds; returns 0 if the result is
// in (ak, av), 1 if in (bk, bv).  Short runs + more merge rounds = lower latency
// for a CTA working on one list; long runs = fewer instructions.
__device__ int smem_sort_run(uint64_t* ak, uint32_t* av, uint64_t* bk, uint32_t* bv, uint32_t rl, uint32_t run) {
    switch (run) {
        case 32: warp_runs<1>(ak, av, rl); break;
        case 64: warp_runs<2>(ak, av, rl); break;
        case 128: warp_runs<4>(ak, av, rl); break;
        case 256: warp_runs<8>(ak, av, rl); break;
        default: warp_runs<16>(ak, av, rl); run = 512; break;
    }
    __syncthreads();
    int in_b = 0;
    for (uint32_t width = run; width < rl; width <<= 1) {
        smem_merge_round(in_b ? bk : ak, in_b ? bv : av, in_b ? ak : bk, in_b ? av : bv, rl, width);
        __syncthreads();
        in_b ^= 1;
    }
    return in_b;
}

#ifndef GS_BIG_TP_THREADS
#define GS_BIG_TP_THREADS 256          // threads of the throughput-mode 2048-entry sort CTA
#endif
template <int SMAX, int NT = (SMAX <= 1024 ? BIG_THREADS : LAT_THREADS)>
__global__ void __launch_bounds__(NT, SMAX <= 1024 ? 6 : (NT <= 256 ? 4 : 1))
big_sort_kernel(const uint32_t* __restrict__ ranges, const uint4* __restrict__ bucket, uint64_t* __restrict__ ka,
                uint32_t* __restrict__ va, uint64_t* __restrict__ kb, uint32_t* __restrict__ vb,
                uint32_t* __restrict__ out, uint32_t* __restrict__ ogid, uint64_t* __restrict__ dbg,
                const uint32_t* __restrict__ big_count, const uint32_t* __restrict__ big_list,
                const uint32_t* __restrict__ status) {
    if (*status) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t nwarp = blockDim.x >> 5;
    uint64_t* sk0 = reinterpret_cast<uint64_t*>(smem_raw);
    constexpr int PAD = SMAX + SMAX / 16;
    uint64_t* sk1 = sk0 + PAD;
    uint32_t* sv0 = reinterpret_cast<uint32_t*>(sk1 + PAD);
    uint32_t* sv1 = sv0 + PAD;
    const uint32_t nbig = *big_count;
    for (uint32_t bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
        const uint32_t tile = big_list[bi];
        const uint32_t s = ranges[2 * tile], len = ranges[2 * tile + 1] - s;
        const bool one_run = len <= SMAX;
        for (uint32_t r0 = 0; r0 < len; r0 += SMAX) {
            const uint32_t rl = min((uint32_t)SMAX, len - r0);
            for (uint32_t e = threadIdx.x; e < rl; e += blockDim.x) {
                const uint4 b = bucket[s + r0 + e];
                sk0[pidx(e)] = ((uint64_t)b.x << 32) | b.z;
                sv0[pidx(e)] = r0 + e;
            }
            __syncthreads();
            // runs sized so every warp of the CTA gets one (latency), at least 32
            uint32_t run = 32;
            while (run < 512 && run * nwarp < rl) run <<= 1;
            const int in_b = smem_sort_run(sk0, sv0, sk1, sv1, rl, run);
            const uint64_t* rk = in_b ? sk1 : sk0;
            const uint32_t* rv = in_b ? sv1 : sv0;
            if (one_run) {
                for (uint32_t e = threadIdx.x; e < rl; e += blockDim.x) {
                    const uint4 b = bucket[s + rv[pidx(e)]];
                    out[s + e] = b.y;
                    if (ogid) ogid[s + e] = b.z;
                    if (dbg) dbg[s + e] = ((uint64_t)tile << 32) | b.x;
                }
            } else {
                for (uint32_t e = threadIdx.x; e < rl; e += blockDim.x) {
                    ka[s + r0 + e] = rk[pidx(e)];
                    va[s + r0 + e] = rv[pidx(e)];
                }
            }
            __syncthreads();
        }
        if (one_run) continue;
        uint64_t* ck = ka + s; uint32_t* cv = va + s;
        uint64_t* nk = kb + s; uint32_t* nv = vb + s;
        for (uint32_t width = SMAX; width < len; width <<= 1) {
            for (uint32_t a0 = 0; a0 < len; a0 += 2 * width) {
                const uint32_t na = min(width, len - a0);
                const uint32_t nb = a0 + na < len ? min(width, len - a0 - na) : 0u;
                cta_merge(ck, cv, nk, nv, a0, na, nb);
            }
            __syncthreads();
            uint64_t* t = ck; ck = nk; nk = t;
            uint32_t* tv = cv; cv = nv; nv = tv;
        }
        for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) {
            const uint4 b = bucket[s + cv[e]];
            out[s + e] = b.y;
            if (ogid) ogid[s + e] = b.z;
            if (dbg) dbg[s + e] = ((uint64_t)tile << 32) | b.x;
        }
        __syncthreads();
    }
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" {

size_t gs_bin_sort_workspace_bytes(int64_t pair_capacity, int64_t total_tiles) {
    if (pair_capacity < 1) pair_capacity = 1;
    if (total_tiles < 1) total_tiles = 1;
    return ws_bytes(pair_capacity, total_tiles);
}

gs_status gs_bin_sort(const gs_projected* proj, const gs_view* views_host, const gs_view* views_dev,
                      int32_t n_views, gs_bins* out, void* ws, size_t ws_size, void* stream) {
    int64_t total_pixels = 0, T = 0;
    gs_status st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(proj && proj->rec && proj->n_rec && proj->status, GS_INVALID_ARG, "proj has a NULL pointer");
    GS_REQUIRE(out && out->ranges && out->sorted_rec && out->n_pairs, GS_INVALID_ARG, "bins has a NULL pointer");
    GS_REQUIRE(out->mode == GS_BIN_SQUARE || out->mode == GS_BIN_TIGHT, GS_INVALID_ARG, "bins mode = %d invalid",
               out->mode);
    GS_REQUIRE(out->pair_capacity >= 1 && out->pair_capacity < (int64_t(1) << 32), GS_INVALID_ARG,
               "pair_capacity = %lld not in [1, 2^32)", (long long)out->pair_capacity);
    const size_t need = ws_bytes(out->pair_capacity, T);
    GS_REQUIRE(ws != nullptr && ws_size >= need, GS_WORKSPACE_TOO_SMALL, "gs_bin_sort workspace %zu < %zu", ws_size,
               need);
    cudaStream_t s = (cudaStream_t)stream;
    BinWs w = carve(ws, out->pair_capacity, T);
    const int64_t cap = proj->rec_capacity;
    cudaMemsetAsync(w.counts, 0, sizeof(uint32_t) * T, s);
    cudaMemsetAsync(w.big_count, 0, 7 * sizeof(uint32_t), s);

    // chunks of >= 1024 records, ~GS_BIN_CTAS_PER_SM CTAs per SM over the whole batch (many
    // short chunks balance the per-record tile loops across SMs; each CTA flushes its
    // on-chip histogram once)
    const int64_t blocks_per_view =
        std::max<int64_t>(1, std::min<int64_t>((cap + 1023) / 1024, (GS_BIN_CTAS_PER_SM * num_sms() + n_views - 1) / n_views));
    dim3 rgrid((unsigned)blocks_per_view, (unsigned)n_views);
    int max_tiles = 0;
    for (int i = 0; i < n_views; ++i)
        max_tiles = std::max(max_tiles, tiles_x(views_host[i]) * tiles_y(views_host[i]));
    const int hist_smem = (int)sizeof(uint32_t) * std::min(max_tiles, HIST_MAX);
    // kernel attributes are per device: set on every call (cheap)
    cudaFuncSetAttribute(count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, HIST_MAX * 4);
    cudaFuncSetAttribute(scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, HIST_MAX * 4);
    const int tight = out->mode == GS_BIN_TIGHT;
    // per-(view, chunk, tile) offsets of count_kernel for the scatter, kept in the big-sort
    // scratch (unused until after the scatter) when it is large enough
    const int cb_stride = std::min(max_tiles, HIST_MAX);
    uint32_t* chunk_base = (max_tiles <= HIST_MAX &&
                            (size_t)blocks_per_view * n_views * cb_stride * sizeof(uint32_t) <=
                                sizeof(uint64_t) * (size_t)out->pair_capacity)
                               ? reinterpret_cast<uint32_t*>(w.ka)
                               : nullptr;
    count_kernel<<<rgrid, BIN_THREADS, hist_smem, s>>>(proj->rec, cap, proj->n_rec, views_dev, w.counts, proj->status,
                                                       tight, chunk_base, cb_stride);
    if ((st = check_launch("count_kernel")) != GS_OK) return st;
    const int64_t nb = (T + SCAN_TILE - 1) / SCAN_TILE;
    scan_reduce_kernel<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(w.counts, T, w.block_sums);
    scan_blocks_kernel<<<1, SCAN_THREADS, 0, s>>>(w.block_sums, nb, out->n_pairs, out->pair_capacity, proj->status);
    scan_down_kernel<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(w.counts, T, w.block_sums, out->ranges, w.cursor);
    if ((st = check_launch("scan kernels")) != GS_OK) return st;
    scatter_kernel<<<rgrid, BIN_THREADS, hist_smem, s>>>(proj->rec, cap, proj->n_rec, views_dev, w.cursor, w.bucket,
                                                          proj->status, tight, chunk_base, cb_stride,
                                                          (uint64_t)out->pair_capacity);
    if ((st = check_launch("scatter_kernel")) != GS_OK) return st;
    // small batches (single views, pyramids): every list > 256 gets a 16-warp CTA
    // (latency); large batches: one warp per list <= 512, 4-warp CTAs above (throughput)
    const bool latency = T <= LAT_TILES;
    if (latency) {
        warp_sort_kernel<<<(unsigned)((T + 7) / 8), 256, 0, s>>>(out->ranges, T, w.bucket, out->sorted_rec,
                                                                 out->sorted_gid, out->sorted_key, w.big_count,
                                                                 w.mid_list, w.big_list, 0u, proj->status);
        if ((st = check_launch("warp_sort_kernel")) != GS_OK) return st;
    } else {
        classify_kernel<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(out->ranges, T, w.bucket, out->sorted_rec,
                                                                    out->sorted_gid, out->sorted_key, w.big_count,
                                                                    w.mid_list, w.big_list, w.cls_list,
                                                                    WARP_SORT_MAX, proj->status);
        if ((st = check_launch("classify_kernel")) != GS_OK) return st;
        const unsigned cg = GS_CLS_GRID * num_sms();
        class_sort_kernel<1><<<cg, 256, 0, s>>>(out->ranges, w.bucket, out->sorted_rec, out->sorted_gid,
                                                out->sorted_key, w.big_count + 2, w.cls_list, proj->status);
        class_sort_kernel<2><<<cg, 256, 0, s>>>(out->ranges, w.bucket, out->sorted_rec, out->sorted_gid,
                                                out->sorted_key, w.big_count + 3, w.cls_list + T, proj->status);
        class_sort_kernel<4><<<cg, 256, 0, s>>>(out->ranges, w.bucket, out->sorted_rec, out->sorted_gid,
                                                out->sorted_key, w.big_count + 4, w.cls_list + 2 * T, proj->status);
        class_sort_kernel<8><<<cg, 256, 0, s>>>(out->ranges, w.bucket, out->sorted_rec, out->sorted_gid,
                                                out->sorted_key, w.big_count + 5, w.cls_list + 3 * T, proj->status);
        if ((st = check_launch("class_sort_kernel")) != GS_OK) return st;
    }
    if (!latency) {
        mid_sort_kernel<<<GS_MID_GRID * num_sms(), 256, 0, s>>>(out->ranges, w.bucket, out->sorted_rec, out->sorted_gid,
                                                      out->sorted_key, w.big_count, w.mid_list, proj->status);
        if ((st = check_launch("mid_sort_kernel")) != GS_OK) return st;
    }
    const int smem = 2 * RUN_PAD * (int)(sizeof(uint64_t) + sizeof(uint32_t));
    cudaFuncSetAttribute(big_sort_kernel<SMEM_SORT_MAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int big_threads = latency ? LAT_THREADS : BIG_THREADS;
    const int big_grid = latency ? 2 * num_sms() : 4 * num_sms();
    if (!latency) {
        // 513..1024 pairs: half the shared memory per CTA, twice the CTAs per SM
        constexpr int S1K = 1024;
        const int smem1k = 2 * (S1K + S1K / 16) * (int)(sizeof(uint64_t) + sizeof(uint32_t));
        cudaFuncSetAttribute(big_sort_kernel<S1K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1k);
        big_sort_kernel<S1K><<<6 * num_sms(), BIG_THREADS, smem1k, s>>>(
            out->ranges, w.bucket, w.ka, w.va, w.kb, w.vb, out->sorted_rec, out->sorted_gid, out->sorted_key,
            w.big_count + 6, w.cls_list + 4 * T, proj->status);
        if ((st = check_launch("big_sort_kernel<1024>")) != GS_OK) return st;
    }
    if (latency) {
        big_sort_kernel<SMEM_SORT_MAX><<<big_grid, big_threads, smem, s>>>(out->ranges, w.bucket, w.ka, w.va, w.kb, w.vb,
                                                                out->sorted_rec, out->sorted_gid, out->sorted_key,
                                                                w.big_count + 1, w.big_list, proj->status);
    } else {
        // throughput mode: more warps per list (shorter warp runs, one more merge round) at
        // 4 CTAs/SM (the shared-memory limit)
        constexpr int NT = GS_BIG_TP_THREADS;
        cudaFuncSetAttribute(big_sort_kernel<SMEM_SORT_MAX, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        big_sort_kernel<SMEM_SORT_MAX, NT><<<4 * num_sms(), NT, smem, s>>>(
            out->ranges, w.bucket, w.ka, w.va, w.kb, w.vb, out->sorted_rec, out->sorted_gid, out->sorted_key,
            w.big_count + 1, w.big_list, proj->status);
    }
    return check_launch("big_sort_kernel");
}

}  // extern "C"
