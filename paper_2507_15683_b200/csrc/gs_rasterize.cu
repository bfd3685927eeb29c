// gs_rasterize.cu -- O12: per pixel front-to-back alpha
// compositing of colour, depth (sum w z), opacity (1 - T) and an optional
// D-channel feature.  P:136 "Color attributes c are rasterized ... using alpha
// blending, while feature attributes f are rendered ... through identical
// rasterization"; "render dense feature and depth maps"; S:157;
// readings Q4, Q11, Q14-Q18.
//
// Design (B200):
//   * a 16x16 tile is rendered by 8 consumer warps (one 8x4 sub-tile each)
//     fed by 1 producer warp;
//   * persistent CTAs (grid = SMs x resident CTAs, tiles handed out in order by
//     a dynamic scheduler); the producer streams the sorted lists of the CTA's
//     tiles through a shared-memory ring (cp.async 16-B gathers of the 64-B
//     records -- and, on the mma.sync feature path only, the feature rows --
//     completion signalled on "full" mbarriers via cp.async.mbarrier.arrive),
//     running ahead across tile boundaries; consumers take stages in same-tile
//     pairs and release them through "empty" mbarriers -- no CTA-wide barrier
//     anywhere in the loop;
//   * exact warp-level culling: each lane tests staged entries: does the
//     entry's alpha >= alpha_min ellipse (p >= e_cut, inflated) touch the warp's
//     8x4 pixel rectangle?  Ballots give the entries the warp walks
//     (conservative, so it never drops a Gaussian the oracle blends -- Q11);
//   * per pixel the skip / stop decisions (exponent, alpha, Tn) are evaluated
//     with explicit _rn / fma intrinsics in the oracle's operation order (Q29);
//   * the feature blend F[px][:] += w[px][k] f[k][:] -- the one dense
//     contraction of the path -- runs on the tensor cores; 16 walked entries
//     are one K = 16 step.  tcgen05 path (D in {16,32,48,64}, fp16 feature
//     rows from gs_scene_features_f16): the warp writes its 32 pixel rows of A
//     (weights as fp16 hi + lo) to TMEM with tcgen05.st, its lanes cp.async the
//     16 feature rows from global/L2 straight into a canonical (no-swizzle,
//     MN-major) smem B tile as the entries are walked, and
//     one lane issues two M=128 N=D K=16 kind::f16 MMAs whose
//     disable-output-lane mask leaves only the warp's own 32 TMEM lanes
//     writable -- the 8 warps share two D-column accumulators (one per lane
//     group of 4 warps) without synchronising with each other; completion is
//     tracked per warp and buffer by tcgen05.commit -> mbarrier, and the tile's
//     epilogue reads the accumulator row with tcgen05.ld.  mma.sync path
//     (other D, or no fp16 copy): m16n8k16 FP16 MMAs with register
//     accumulators.  Both: weights split hi + lo (~2^-22 relative), features
//     rounded once to fp16: error <= 2^-11 sum w|f|, inside the 1e-3
//     max(1,|f|) tolerance;
//   * warp-ballot early termination once all 32 pixels have T < t_min.
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "gs_common.cuh"
#include "gs_tc.cuh"

namespace gs {
namespace {

constexpr int NCW = 8;                 // consumer warps
constexpr int RT_THREADS = (NCW + 1) * 32;
#ifndef GS_SE
#define GS_SE 64                       // r2: 64-entry stages, 5 of them (C4 27.66 -> 27.34 ms)
#endif
#ifndef GS_NST
#define GS_NST 5
#endif
#ifndef GS_NST_D0
#define GS_NST_D0 10                   // r2: without feature rows a stage is 4 KB: a deeper ring
#endif                                 // absorbs the 8 warps' per-tile imbalance (C5 20.86 -> ~20.2 ms)
#ifndef GS_TC_DIRECT_B
#define GS_TC_DIRECT_B 1               // r2: tcgen05 path fetches a k-step's feature rows straight into its B tile
#endif
#ifndef GS_NST_TCB
#define GS_NST_TCB 5                   // ring stages when the ring carries records only (tcgen05, direct B)
#endif
#ifndef GS_SE_TCB
#define GS_SE_TCB 128                  // entries per stage there (C4: 128 x 5 24.51 ms, 64 x 10 24.85 ms)
#endif
// ring stages: a ring carrying feature rows is bounded by shared memory (3 CTAs/SM)
constexpr int nst_for(int D, bool TC) {
    return D == 0 ? GS_NST_D0 : (TC && GS_TC_DIRECT_B) ? GS_NST_TCB : GS_NST;
}
// entries per stage (SE / 32 ballots per lane)
constexpr int se_for(int D, bool TC) { return (D > 0 && TC && GS_TC_DIRECT_B) ? GS_SE_TCB : GS_SE; }
// 16-B global->shared copy that zero-fills instead when !valid (src-size 0)
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
constexpr int WB_STRIDE = 36;          // weight-buffer row stride (conflict-free m16n8k16 A fragments)
constexpr int WB_ROWS = 16;            // one tensor-core k-step of weights (m16n8k16)
constexpr uint32_t ST_FIRST = 1u, ST_LAST = 2u, ST_END = 4u;
#ifndef GS_SCHED_CHUNK
#define GS_SCHED_CHUNK 2
#endif
constexpr uint32_t SCHED_CHUNK = GS_SCHED_CHUNK;   // tiles per scheduler claim
#ifndef GS_WALK4
#define GS_WALK4 1                     // r2: four entries per walk iteration (4 independent alphas)
#endif

// 16-B global->shared copy that asks L2 to keep the line (records and feature rows
// are re-read by the ~4 neighbouring tiles a Gaussian overlaps)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint64_t policy) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "l"(policy)
                 : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
// the mbarrier receives one arrival when all prior cp.async of this thread have landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int D>
struct TcCfg {
    static constexpr bool eligible = D == 16 || D == 32 || D == 48 || D == 64;
    static constexpr uint32_t need = 2 * D + 64;
    static constexpr uint32_t cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
};

#ifdef GS_RASTER_STATS
__device__ unsigned long long g_raster_stats[4];   // debug: entry-walks, live lane-walks
#endif

struct StageMeta {
    uint32_t tile, c0;
    int32_t cnt, view;
    uint32_t flags, pad0, pad1, pad2;
};

template <int D, bool CONTRIB, bool TC>
struct RasterSmem {
    static constexpr int NST = nst_for(D, TC);
    static constexpr int SE = se_for(D, TC);       // entries per stage
    static constexpr int SPL = SE / 32;            // entries per lane per stage
    // tcgen05 direct-B: feature rows skip the ring (the consumer warps cp.async them into
    // their B tiles), so weight rows pin no ring stage
    static constexpr bool DIRECT_B = TC && GS_TC_DIRECT_B;
    static constexpr int FS = D > 0 ? D + 8 : 1;   // fp32 feature row stride (floats)
    static constexpr int FSH = D + 8;              // fp16 feature row stride (halves; 16-B aligned rows)
    static constexpr bool WB = D > 0;              // weight rows are collected (features)
    // tcgen05: each walked entry pair's fp16 hi / lo weights go straight from registers
    // into the TMEM A buffer (no shared-memory weight rows)
    static constexpr bool DIRECT = TC;
    static constexpr bool WSTAGE = WB && !DIRECT;
    float4 rec[NST][SE + 1][4];                    // 64-byte records; row SE = null record (opacity 0)
    float feat[(D > 0 && !TC) ? NST : 1][(D > 0 && !TC) ? SE + 1 : 1][FS];
    alignas(16) __half feath[(TC && !DIRECT_B) ? NST : 1][(TC && !DIRECT_B) ? SE + 1 : 1][(TC && !DIRECT_B) ? FSH : 8];
    alignas(16) float wbuf[WSTAGE ? NCW : 1][WSTAGE ? WB_ROWS : 1][WB_STRIDE]; // per-warp weights [k][pixel]
    uint32_t slots[CONTRIB ? NST * (SE + 1) : 1];  // record slot of each ring row (contributions)
    alignas(16) int ent[NCW][2 * SE + 2];            // per-warp compacted ballot list of a stage pair (flat rows)
    int kent[NCW][WB_ROWS];                          // ring row of each pending weight row
    StageMeta meta[NST];
    uint64_t full[NST];
    uint64_t empty[NST];
    // tcgen05 path: per-warp double-buffered B tile (16 x D fp16, canonical MN-major,
    // no swizzle) and the MMA-completion barriers of its two buffers
    alignas(128) __half bbuf[TC ? NCW : 1][2][TC ? 16 * D : 8];
    uint64_t mma_bar[TC ? NCW : 1][2];
    uint32_t tmem_base;
};

// 1-ulp reciprocal (MUFU): only locates the stationary point of an edge; the e_cut
// margin absorbs the error, so the cull stays conservative
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;\n" : "=f"(r) : "f"(x));
    return r;
}

// max over the 8x4 pixel-centre rectangle [x0,x1]x[y0,y1] of the log2-unit
// exponent p(d) = ea dx^2 + eb dx dy + ec dy^2 (d = p - mean; ea, ec < 0),
// compared with e_cut (the alpha >= alpha_min ellipse, inflated).
__device__ __forceinline__ bool ellipse_hits_rect(float u, float v, float ea, float eb, float ec, float ecut,
                                                  float x0, float x1, float y0, float y1) {
    // branch-free (the lanes of a warp test different entries): both edge candidates are
    // evaluated and the ones that do not apply are masked
    const bool inx = u >= x0 && u <= x1, iny = v >= y0 && v <= y1;
    float pmax = -3.4e38f;
    {                         // facing vertical edge: best dy = -eb dx / (2 ec), clamped
        const float dx = (u < x0 ? x0 : x1) - u;
        const float dy = fminf(fmaxf(-eb * dx * rcp_approx(2.f * ec), y0 - v), y1 - v);
        const float pe = ea * dx * dx + eb * dx * dy + ec * dy * dy;
        pmax = inx ? pmax : fmaxf(pmax, pe);
    }
    {                         // facing horizontal edge: best dx = -eb dy / (2 ea), clamped
        const float dy = (v < y0 ? y0 : y1) - v;
        const float dx = fminf(fmaxf(-eb * dy * rcp_approx(2.f * ea), x0 - u), x1 - u);
        const float pe = ea * dx * dx + eb * dx * dy + ec * dy * dy;
        pmax = iny ? pmax : fmaxf(pmax, pe);
    }
    return (inx && iny) || pmax >= ecut;
}

// Blackwell packed fp32 (f32x2) arithmetic: each lane rounds exactly like the
// scalar _rn operation, one issue slot for two.  Only used where no multiply feeds
// an add (ptxas contracts f32x2 mul + add regardless of .rn).
__device__ __forceinline__ uint64_t pk2(float x, float y) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};\n" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ float2 upk2(uint64_t r) {
    float2 v;
    asm("mov.b64 {%0, %1}, %2;\n" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
// (a.x - b.x, a.y - b.y), each rounded to nearest
__device__ __forceinline__ float2 sub2_rn(float ax, float ay, float bx, float by) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;\n" : "=l"(r) : "l"(pk2(ax, ay)), "l"(pk2(bx, by)));
    return upk2(r);
}
// (x, y) += w (a, b) as two fmaf
__device__ __forceinline__ void fma2_acc(float& x, float& y, float w, float a, float b) {
    uint64_t acc = pk2(x, y);
    asm("fma.rn.f32x2 %0, %1, %2, %0;\n" : "+l"(acc) : "l"(pk2(w, w)), "l"(pk2(a, b)));
    const float2 v = upk2(acc);
    x = v.x; y = v.y;
}

// o 2^p as the walk evaluates it (ex2.approx + one rounded product): the only
// decision input that differs from the oracle's fp64 2^p; its deviation is
// bounded by the O14 alpha band (reading Q20, checked by gs_probe_alpha).
__device__ __forceinline__ float alpha_raw(float o, float p) { return __fmul_rn(o, ex2_ftz(p)); }

// alpha of entry k at this lane's pixel, or 0 when the oracle skips it (p > 0
// or alpha < alpha_min).  p(d) = dx (ea dx + eb dy) + ec dy dy with the oracle's
// fused multiply-adds (reading Q29); alpha = min(alpha_max, o 2^p).
__device__ __forceinline__ float entry_alpha(const float4& a, const float4& b, float pxf, float pyf,
                                             const gs_params& P) {
    const float2 d = sub2_rn(a.x, a.y, pxf, pyf);
    const float dx = d.x, dy = d.y;
    const float p = __fmaf_rn(dx, __fmaf_rn(a.z, dx, __fmul_rn(a.w, dy)), __fmul_rn(__fmul_rn(b.x, dy), dy));
    const float alpha = fminf(P.alpha_max, alpha_raw(b.y, p));
    // skipped iff p > 0 or alpha < alpha_min (alpha is never NaN: fminf with alpha_max);
    // one compare feeds the other so the pair costs two FSETP and one select
    float r;
    asm("{\n"
        ".reg .pred pp, keep;\n"
        "setp.gt.f32 pp, %1, 0f00000000;\n"
        "setp.ge.and.f32 keep, %2, %3, !pp;\n"
        "selp.f32 %0, %2, 0f00000000, keep;\n"
        "}\n"
        : "=f"(r)
        : "f"(p), "f"(alpha), "f"(P.alpha_min));
    return r;
}

// Persistent kernel: each CTA renders a sequence of tiles handed out in order by
// a dynamic scheduler.  The producer warp runs ahead across tile boundaries so
// the consumers never wait for a tile's first records.
// back-off of a warp waiting on the stage ring (ns): the producer when the ring is
// full, a consumer warp that ran ahead of its CTA's slowest warp
#ifndef GS_PROD_SLEEP
#define GS_PROD_SLEEP 64
#endif
#ifndef GS_CONS_SLEEP
#define GS_CONS_SLEEP 64
#endif
#ifndef GS_TC_MIN_BLOCKS
#define GS_TC_MIN_BLOCKS 3
#endif
template <int D, bool CONTRIB, bool TC>
__global__ void __launch_bounds__(RT_THREADS, (TC ? (D > 32 ? 1 : GS_TC_MIN_BLOCKS) : (D > 32 ? 1 : (D > 0 ? 2 : 4))))
rasterize_kernel(const gs_view* __restrict__ views, int n_views, const gs_record* __restrict__ rec,
                 const uint32_t* __restrict__ sorted_rec, const uint32_t* __restrict__ sorted_gid,
                 const uint32_t* __restrict__ ranges, uint32_t n_tiles, uint32_t* __restrict__ tile_sched,
                 const float* __restrict__ feat, const __half* __restrict__ feat_h,
                 gs_params P, float* __restrict__ out_rgb, float* __restrict__ out_depth,
                 float* __restrict__ out_alpha, float* __restrict__ out_feat,
                 unsigned long long* __restrict__ contrib, const uint32_t* __restrict__ status, float a_min,
                 float* __restrict__ out_xyz, uint8_t* __restrict__ out_valid) {
    static_assert(!TC || TcCfg<D>::eligible, "tcgen05 feature path needs D in {16, 32, 48, 64}");
    using Smem = RasterSmem<D, CONTRIB, TC>;
    constexpr bool WB = Smem::WB;
    constexpr int NST = Smem::NST;
    constexpr int SE = Smem::SE;
    constexpr int SPL = Smem::SPL;
    constexpr bool HOLD = WB && !Smem::DIRECT_B;   // pending weight rows pin the ring stages of their features
    if (*status) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < NST * 4; i += blockDim.x) sm.rec[i / 4][SE][i % 4] = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (Smem::DIRECT_B) {
        // padding rows of a k-step keep the buffer's previous (finite) rows under zero
        // weights; start from zeros so no uninitialised pattern (NaN) is ever multiplied
        __half* bb = &sm.bbuf[0][0][0];
        for (int i = threadIdx.x; i < (int)(sizeof(sm.bbuf) / sizeof(__half)); i += blockDim.x) bb[i] = __float2half_rn(0.f);
    } else if constexpr (TC)
        for (int i = threadIdx.x; i < NST * Smem::FSH; i += blockDim.x)
            sm.feath[i / Smem::FSH][SE][i % Smem::FSH] = __float2half_rn(0.f);
    else if constexpr (D > 0)
        for (int i = threadIdx.x; i < NST * Smem::FS; i += blockDim.x) sm.feat[i / Smem::FS][SE][i % Smem::FS] = 0.f;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&sm.full[s], 33);     // 32 cp.async arrivals + 1 metadata arrival
            mbar_init(&sm.empty[s], NCW);
        }
        if constexpr (TC)
            for (int w = 0; w < NCW; ++w) { mbar_init(&sm.mma_bar[w][0], 1); mbar_init(&sm.mma_bar[w][1], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if constexpr (TC) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_u32(&sm.tmem_base)),
                         "r"(TcCfg<D>::cols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
        }
        tc_fence_before();
    }
    __syncthreads();
    if constexpr (TC) tc_fence_after();

    if (warp == NCW) {
        // ------------------------------------------------------------ producer
        // Stage iterator over this CTA's tiles; the index loads (sorted slot / gid) of
        // stage s+1 are issued before waiting for stage s's ring slot, so their
        // latency hides behind the wait and the gathers of stage s.
        uint32_t tile = blockIdx.x, rs = 0, re = 0, k = 0, nst = 1;
        int view = 0;
        bool end = false;
        // Dynamic tile scheduler: chunks of SCHED_CHUNK consecutive tiles are handed
        // out in order from a global counter, so all CTAs work on one compact window
        // of tiles (records / feature rows stay L2-resident); the next chunk is
        // claimed one chunk ahead to hide the atomic's latency.  CTA c's first chunk
        // is static.  Without a counter: static round-robin chunks.
        uint32_t ch_base = blockIdx.x * SCHED_CHUNK, ch_i = 0;
        auto claim = [&]() -> uint32_t {
            uint32_t b = 0;
            if (lane == 0) b = atomicAdd(tile_sched, SCHED_CHUNK);
            return gridDim.x * SCHED_CHUNK + __shfl_sync(0xffffffffu, b, 0);
        };
        uint32_t ch_next = tile_sched ? claim() : ch_base + gridDim.x * SCHED_CHUNK;
        auto next_tile = [&]() -> uint32_t {
            if (++ch_i < SCHED_CHUNK) return ch_base + ch_i;
            ch_base = ch_next;
            ch_i = 0;
            ch_next = tile_sched ? (ch_base < n_tiles ? claim() : ch_base) : ch_base + gridDim.x * SCHED_CHUNK;
            return ch_base;
        };
        auto tile_begin = [&](uint32_t t) {
            tile = t;
            end = t >= n_tiles;
            k = 0;
            if (!end) {
                rs = __ldg(&ranges[2 * t]);
                re = __ldg(&ranges[2 * t + 1]);
                view = find_view_by_tile(views, n_views, t);
                nst = max(1u, (re - rs + SE - 1) / SE);
            } else {
                rs = re = 0;
                nst = 1;
            }
        };
        auto load_idx = [&](uint32_t c0, int cnt, uint32_t (&sl)[SE / 32], uint32_t (&gd)[SE / 32]) {
#pragma unroll
            for (int q = 0; q < SE / 32; ++q) {
                const int j = q * 32 + (int)lane;
                sl[q] = j < cnt ? __ldg(&sorted_rec[c0 + j]) : 0u;
                gd[q] = (D > 0 && !Smem::DIRECT_B && j < cnt)
                            ? (sorted_gid ? __ldg(&sorted_gid[c0 + j]) : __ldg(&rec[sl[q]].gid)) : 0u;
            }
        };
        tile_begin(ch_base);
        const uint64_t pol = l2_evict_last_policy();
        uint32_t slot[SE / 32], gid[SE / 32];
        uint32_t c0 = rs;
        int cnt = end ? 0 : (int)min((uint32_t)SE, re - c0);
        load_idx(c0, cnt, slot, gid);
        uint32_t s = 0;
        for (;; ++s) {
            const uint32_t buf = s % NST;
            // descriptor of this stage
            const uint32_t ctile = tile, cc0 = c0;
            const int ccnt = cnt, cview = view;
            const uint32_t flags = (k == 0 ? ST_FIRST : 0u) | (k == nst - 1 ? ST_LAST : 0u) | (end ? ST_END : 0u);
            const bool cend = end;
            // advance the iterator and prefetch the next stage's indices
            uint32_t nslot[SE / 32], ngid[SE / 32];
            if (!cend) {
                if (++k == nst) tile_begin(next_tile());
                c0 = rs + k * SE;
                cnt = end ? 0 : (int)min((uint32_t)SE, re - c0);
                load_idx(c0, cnt, nslot, ngid);
            }
            if (s >= NST) mbar_wait_sleep(&sm.empty[buf], ((s / NST) & 1u) ^ 1u, GS_PROD_SLEEP);
#pragma unroll
            for (int q = 0; q < SE / 32; ++q) {
                const int j = q * 32 + (int)lane;
                if (j < ccnt) {
                    const float4* src = reinterpret_cast<const float4*>(rec + slot[q]);
                    if constexpr (CONTRIB) sm.slots[buf * (SE + 1) + j] = slot[q];
#pragma unroll
                    for (int e = 0; e < 4; ++e) cp_async16(&sm.rec[buf][j][e], src + e, pol);
                    if constexpr (TC && !Smem::DIRECT_B) {
                        const uint4* fs = reinterpret_cast<const uint4*>(feat_h + (int64_t)gid[q] * D);
#pragma unroll
                        for (int e = 0; e < D / 8; ++e) cp_async16(&sm.feath[buf][j][e * 8], fs + e, pol);
                    } else if constexpr (D > 0 && !TC) {
                        const float4* fs = reinterpret_cast<const float4*>(feat + (int64_t)gid[q] * D);
#pragma unroll
                        for (int e = 0; e < D / 4; ++e) cp_async16(&sm.feat[buf][j][e * 4], fs + e, pol);
                    }
                }
            }
            cp_async_mbar_arrive(&sm.full[buf]);
            __syncwarp();   // order the lanes' slot writes before lane 0's release arrival
            if (lane == 0) {
                StageMeta m;
                m.tile = ctile; m.c0 = cc0; m.cnt = ccnt; m.view = cview; m.flags = flags;
                m.pad0 = m.pad1 = m.pad2 = 0;
                sm.meta[buf] = m;
                mbar_arrive(&sm.full[buf]);
            }
            if (cend) break;
#pragma unroll
            for (int q = 0; q < SE / 32; ++q) { slot[q] = nslot[q]; gid[q] = ngid[q]; }
        }
        ++s;
        // drain: the CTA must not retire while copies into its smem are in flight
        for (uint32_t q = (s > NST ? s - NST : 0u); q < s; ++q) mbar_wait(&sm.full[q % NST], (q / NST) & 1u);
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int g = (int)(lane >> 2), t4 = (int)(lane & 3u);
    constexpr int NTP = (D > 0 && !TC) ? (D + 7) / 8 : 1;
    float acc[TC ? 1 : 2][NTP][4];
    // tcgen05 state: TMEM addresses of this warp's accumulator / A buffers, k-step count
    const uint32_t tq = warp & 3u, tgrp = warp >> 2;
    const uint32_t tmem = TC ? sm.tmem_base : 0u;
    const uint32_t tD = tmem + tgrp * (uint32_t)D;                     // MMA operand address (lane field 0)
    const uint32_t tA = tmem + 2u * (uint32_t)D + tgrp * 32u;
    const uint32_t my_lanes = (tq * 32u) << 16;
    constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(D >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint32_t kstep = 0, tile_acc = 0;
    uint32_t tnext = tA + my_lanes;   // DIRECT: TMEM column of the next weight pair (hi; lo at +8)
    // per-tile state
    const gs_view* V = nullptr;
    int W = 0, H = 0, sx = 0, sy = 0, px = 0, py = 0;
    bool inside = false, done = true, warp_done = true;
    float pxf = 0.f, pyf = 0.f, rx0 = 0.f, rx1 = 0.f, ry0 = 0.f, ry1 = 0.f;
    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Dz = 0.f;

    // F[px][:] += W[px][0..nk) F_entries[0..nk)[:] on the tensor cores (nk multiple of 8)
    auto mma_block = [&](int kb, int ke) {
        if constexpr (TC) {
            // one k-step of 16 weight rows on tcgen05: A (this warp's 32 pixel rows, fp16
            // hi + lo weight pairs) -> TMEM, B (16 feature rows -> fp16) -> the canonical
            // smem tile, then two lane-masked M=128 N=D K=16 MMAs issued by lane 0
            const uint32_t b = kstep & 1u;
            if constexpr (!Smem::DIRECT) {
                if (kstep >= 2) mbar_wait(&sm.mma_bar[warp][b], ((kstep >> 1) - 1u) & 1u);
                uint32_t hi[8], lo[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float w0 = sm.wbuf[warp][2 * c][lane], w1 = sm.wbuf[warp][2 * c + 1][lane];
                    const __half2 h = __floats2half2_rn(w0, w1);
                    const float2 hf = __half22float2(h);
                    const __half2 l = __floats2half2_rn(w0 - hf.x, w1 - hf.y);
                    hi[c] = *reinterpret_cast<const uint32_t*>(&h);
                    lo[c] = *reinterpret_cast<const uint32_t*>(&l);
                }
                tmem_st8(tA + my_lanes + b * 16u, hi);
                tmem_st8(tA + my_lanes + b * 16u + 8u, lo);
            }
            __half* bt = &sm.bbuf[warp][b][0];
            if constexpr (Smem::DIRECT_B) {
                // the k-step's feature rows were cp.async'd into this B tile as its entries
                // were walked (feed_rows): wait for this lane's copies
                asm volatile("cp.async.wait_all;\n" ::: "memory");
            } else {
                // the B tile is built while the TMEM stores are in flight
                constexpr int NC8 = D / 8;
                const __half* fb = &sm.feath[0][0][0];
#pragma unroll
                for (int c = (int)lane; c < 16 * NC8; c += 32) {
                    const int k = c / NC8, n8 = c % NC8;
                    GS_DCHECK(sm.kent[warp][k] >= 0 && sm.kent[warp][k] < NST * (SE + 1));
                    const uint4 o = *reinterpret_cast<const uint4*>(fb + sm.kent[warp][k] * Smem::FSH + n8 * 8);
                    // element (k, n) at n8*64 + (k%8)*8 + (k/8)*8*D halves (SBO = 128 B, LBO = 16 D B)
                    *reinterpret_cast<uint4*>(bt + n8 * 64 + (k & 7) * 8 + (k >> 3) * 8 * D) = o;
                }
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                tc_fence_after();
                const uint64_t desc = (uint64_t)((smem_u32(bt) >> 4) & 0x3FFFu) |
                                      ((uint64_t)(((16u * D) >> 4) & 0x3FFFu) << 16) |
                                      ((uint64_t)((128u >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
                tc_mma_f16(tD, tA + b * 16u, desc, IDESC, tile_acc, tq);
                tc_mma_f16(tD, tA + b * 16u + 8u, desc, IDESC, 1u, tq);
                tc_commit(&sm.mma_bar[warp][b]);
            }
            __syncwarp();
            tile_acc = 1;
            ++kstep;
            // DIRECT: the walk writes the next k-step's weights into the other buffer as it
            // goes, so wait here (not per entry pair) for that buffer's MMA, issued one
            // k-step ago and long finished
            if constexpr (Smem::DIRECT) {
                if (kstep >= 2) mbar_wait(&sm.mma_bar[warp][kstep & 1u], ((kstep >> 1) - 1u) & 1u);
                tnext = tA + my_lanes + (kstep & 1u) * 16u;
            }
        } else if constexpr (D > 0) {
            // m16n8k16 FP16 MMAs: weights split hi + lo (fp16 pairs, ~2^-22 exact), feature
            // rows rounded once to fp16 (error <= 2^-11 sum w|f|, inside 1e-3 max(1,|f|))
            for (int k0 = kb; k0 < ke; k0 += 16) {
                uint32_t ahi[2][4], alo[2][4];
#pragma unroll
                for (int m = 0; m < 2; ++m) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int px = m * 16 + g + ((i & 1) ? 8 : 0);
                        const int k = k0 + 2 * t4 + ((i & 2) ? 8 : 0);
                        const float w0 = sm.wbuf[warp][k][px], w1 = sm.wbuf[warp][k + 1][px];
                        const __half2 h = __floats2half2_rn(w0, w1);
                        const float2 hf = __half22float2(h);
                        const __half2 l = __floats2half2_rn(w0 - hf.x, w1 - hf.y);
                        ahi[m][i] = *reinterpret_cast<const uint32_t*>(&h);
                        alo[m][i] = *reinterpret_cast<const uint32_t*>(&l);
                    }
                }
                const float* fb = &sm.feat[0][0][0];
                constexpr int FS = Smem::FS;
                const float* f0 = fb + sm.kent[warp][k0 + 2 * t4] * FS;
                const float* f1 = fb + sm.kent[warp][k0 + 2 * t4 + 1] * FS;
                const float* f2 = fb + sm.kent[warp][k0 + 2 * t4 + 8] * FS;
                const float* f3 = fb + sm.kent[warp][k0 + 2 * t4 + 9] * FS;
#pragma unroll
                for (int n = 0; n < NTP; ++n) {
                    const int ch = n * 8 + g;
                    const bool in = ch < D;
                    const __half2 b0h = __floats2half2_rn(in ? f0[ch] : 0.f, in ? f1[ch] : 0.f);
                    const __half2 b1h = __floats2half2_rn(in ? f2[ch] : 0.f, in ? f3[ch] : 0.f);
                    const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&b0h);
                    const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&b1h);
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        mma_f16(acc[m][n], ahi[m], b0, b1);
                        mma_f16(acc[m][n], alo[m], b0, b1);
                    }
                }
            }
        }
    };
    // N1: each walked entry's blend weights summed over the warp's 32 pixels with one
    // integer warp reduction (REDUX) in 2^-27 fixed point (w <= alpha_max = 0.99, so 32
    // lanes stay below 2^32); the sum of the entry at compacted-list index idx is kept
    // by lane idx % 32 and every 32 entries the lanes add theirs to the records'
    // contributions (2^-32 units) with one 64-bit atomic each: order-independent, hence
    // run-to-run deterministic, and no per-entry divergent atomics
    uint32_t csum = 0;
    auto contrib_put = [&](int idx, float w1, float w2) {
        if constexpr (CONTRIB) {
            const uint32_t c1 = __reduce_add_sync(0xffffffffu, __float2uint_rn(w1 * 134217728.0f));
            const uint32_t c2 = __reduce_add_sync(0xffffffffu, __float2uint_rn(w2 * 134217728.0f));
            csum = ((uint32_t)idx & 31u) == lane ? c1 : csum;
            csum = ((uint32_t)(idx + 1) & 31u) == lane ? c2 : csum;
        }
    };
    auto contrib_flush = [&](int base, int cnt) {   // entries [base, base + cnt) of the list, cnt <= 32
        if constexpr (CONTRIB) {
            if ((int)lane < cnt && csum) {
                const int row = sm.ent[warp][base + (int)lane];
                if ((row % (SE + 1)) != SE)
                    atomicAdd(&contrib[sm.slots[row]], (unsigned long long)csum << 5);
            }
            csum = 0;
        }
    };
    // apply one evaluated entry to this lane's pixel, branch-free (om = 1 - a).  A
    // skipped entry (power > 0 or alpha < alpha_min) arrives as alpha = 0, an exact
    // no-op: Tn = T(1 - 0) = T >= t_min, w = 0.  A pixel that already stopped keeps
    // T and gets weight 0 whatever a is.
    auto blend_om = [&](float a, float om, const float4& c) -> float {
        const float Tn = __fmul_rn(T, om);
        const bool stop = done || Tn < P.t_min;
        const float wgt = stop ? 0.0f : __fmul_rn(a, T);
        fma2_acc(C0, C1, wgt, c.x, c.y);
        fma2_acc(C2, Dz, wgt, c.z, c.w);
        T = stop ? T : Tn;
        done = stop;
        return wgt;
    };

    // Weights of walked entries are fed to the tensor cores 8 at a time; fewer than
    // 8 may stay pending across stages, so a stage's ring slot is released only when
    // no pending row references it.  Ring rows are addressed flat: stage buffer b,
    // entry j -> b * (SE + 1) + j (row SE of every buffer is the null record).
    const float4* recf = &sm.rec[0][0][0];
    int pend = 0;             // pending weight rows (< WB_ROWS between stages)
    uint32_t hold = 0;        // oldest stage a pending row references
    uint32_t rel = 0;         // next stage to release
    // DIRECT: weights of entries (2q, 2q+1) of the current k-step -> A column q (hi) and
    // 8 + q (lo) of TMEM buffer kstep & 1 (free: mma_block waited for its previous MMA)
    auto store_pair = [&](float w1, float w2, int q) {
        if constexpr (Smem::DIRECT) {
            (void)q;   // column q of the k-step = tnext
            const __half2 h = __floats2half2_rn(w1, w2);
            const float2 hf = __half22float2(h);
            const float2 r = sub2_rn(w1, w2, hf.x, hf.y);
            const __half2 l = __floats2half2_rn(r.x, r.y);
            GS_DCHECK((tnext & 0xffffu) >= (tA & 0xffffu) && (tnext & 0xffffu) < (tA & 0xffffu) + 24u);
            tmem_st1(tnext, *reinterpret_cast<const uint32_t*>(&h));
            tmem_st1(tnext + 8u, *reinterpret_cast<const uint32_t*>(&l));
            ++tnext;
        }
    };
    // direct B: entries [i, i + m) of the compacted list become rows pend.. of the k-step
    // being filled; lane l < m copies entry i + l's fp16 feature row (D / 8 16-B chunks) into
    // the canonical B tile (element (k, n) at n8*64 + (k%8)*8 + (k/8)*8*D halves); the null
    // record (odd-tail padding) gets a zero row
    auto feed_rows = [&](int i, int m) {
        if constexpr (Smem::DIRECT_B) {
            if (lane < (uint32_t)m) {
                const int row = sm.ent[warp][i + (int)lane];
                GS_DCHECK(row >= 0 && row < NST * (SE + 1));
                const bool real = (row % (SE + 1)) != SE;
                const uint32_t g = __float_as_uint(recf[4 * row + 3].x);   // record gid
                const uint4* src = reinterpret_cast<const uint4*>(feat_h + (int64_t)(real ? g : 0u) * D);
                const int k = pend + (int)lane;
                GS_DCHECK(k < WB_ROWS && (!real || g < 0x10000000u));
                __half* dst = &sm.bbuf[warp][kstep & 1u][0] + (k & 7) * 8 + (k >> 3) * 8 * D;
#pragma unroll
                for (int n8 = 0; n8 < D / 8; ++n8) cp_async16_zfill(dst + n8 * 64, src + n8, real);
            }
        }
    };
    auto flush_pending = [&]() {
        if constexpr (WB) {
            if (pend > 0) {
                if constexpr (Smem::DIRECT)
                    for (int q = pend >> 1; q < WB_ROWS / 2; ++q) store_pair(0.f, 0.f, q);
                else
                    for (int r = pend; r < WB_ROWS; ++r) sm.wbuf[warp][r][lane] = 0.f;
                if (!Smem::DIRECT_B && lane < (uint32_t)(WB_ROWS - pend)) sm.kent[warp][pend + lane] = SE;   // null row
                __syncwarp();
                mma_block(0, WB_ROWS);
                __syncwarp();
                pend = 0;
            }
        }
    };

    // Consumers take the ring two stages at a time when both belong to the same tile
    // (SE-entry stages): one wait / cull-compaction / walk / release
    // cycle per 64 entries halves the per-stage bookkeeping.
    for (uint32_t s = 0;;) {
        const int buf = (int)(s % NST);
        mbar_wait_sleep(&sm.full[buf], (s / NST) & 1u, GS_CONS_SLEEP);
        const StageMeta m = sm.meta[buf];
        if (m.flags & ST_END) break;
        const bool pair = !(m.flags & ST_LAST);   // a non-last stage is followed by one of its tile
        const uint32_t s2 = pair ? s + 1 : s;
        const int buf2 = (int)(s2 % NST);
        int cnt2 = 0;
        uint32_t last_flags = m.flags;
        if (pair) {
            mbar_wait_sleep(&sm.full[buf2], (s2 / NST) & 1u, GS_CONS_SLEEP);
            cnt2 = sm.meta[buf2].cnt;
            last_flags = sm.meta[buf2].flags;
        }
        if (m.flags & ST_FIRST) {
            V = &views[m.view];
            W = V->width;
            H = V->height;
            const int TX = (W + GS_TILE - 1) / GS_TILE;
            const uint32_t lt = m.tile - V->tile_offset;
            const int tx = (int)(lt % (uint32_t)TX), ty = (int)(lt / (uint32_t)TX);
            sx = tx * 16 + (int)(warp & 1u) * 8;
            sy = ty * 16 + (int)(warp >> 1) * 4;
            px = sx + (int)(lane & 7u);
            py = sy + (int)(lane >> 3);
            inside = px < W && py < H;
            pxf = (float)px; pyf = (float)py;
            rx0 = (float)sx; rx1 = (float)(sx + 7); ry0 = (float)sy; ry1 = (float)(sy + 3);
            T = 1.0f; C0 = C1 = C2 = Dz = 0.f;
            done = !inside;
            warp_done = __all_sync(0xffffffffu, done);
            tile_acc = 0;
            if constexpr (!TC) {
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int n = 0; n < NTP; ++n) acc[a][n][0] = acc[a][n][1] = acc[a][n][2] = acc[a][n][3] = 0.f;
            }
        }
        if (!warp_done && (m.cnt > 0 || cnt2 > 0)) {
            const int flat0 = buf * (SE + 1), flat2 = buf2 * (SE + 1);
            bool hit[2 * SPL];
            uint32_t mk[2 * SPL];
#pragma unroll
            for (int h = 0; h < 2 * SPL; ++h) {
                const int j = (int)lane + 32 * (h % SPL);
                const int b = h < SPL ? buf : buf2;
                hit[h] = false;
                if (j < (h < SPL ? m.cnt : cnt2)) {
                    const float4 a = sm.rec[b][j][0];   // u, v, ea, eb
                    const float4 q = sm.rec[b][j][1];   // ec, o, e_cut, -
                    hit[h] = ellipse_hits_rect(a.x, a.y, a.z, a.w, q.x, q.z, rx0, rx1, ry0, ry1);
                }
            }
            int off[2 * SPL + 1];
            off[0] = 0;
#pragma unroll
            for (int h = 0; h < 2 * SPL; ++h) {
                mk[h] = __ballot_sync(0xffffffffu, hit[h]);
                off[h + 1] = off[h] + __popc(mk[h]);
            }
            const int n = off[2 * SPL];
            if (n > 0) {
                // compacted in-order entry list; an odd tail is padded with the null record
                const uint32_t below = (1u << lane) - 1u;
#pragma unroll
                for (int h = 0; h < 2 * SPL; ++h)
                    if (hit[h])
                        sm.ent[warp][off[h] + __popc(mk[h] & below)] =
                            (h < SPL ? flat0 : flat2) + (int)lane + 32 * (h % SPL);
                if (lane == 0 && (n & 1)) sm.ent[warp][n] = flat0 + SE;
                __syncwarp();
                // walk one entry pair: independent alphas (ILP 2), transmittance in list order
                auto walk_pair = [&](const int2 kk, float& w1, float& w2) {
#ifdef GS_RASTER_STATS
                    {
                        const unsigned live = __ballot_sync(0xffffffffu, !done);
                        if (lane == 0) {
                            atomicAdd(&g_raster_stats[0], 2ull);                       // entry-walks
                            atomicAdd(&g_raster_stats[1], 2ull * __popc(live));       // live lane-walks
                        }
                    }
#endif
                    GS_DCHECK(kk.x >= 0 && kk.x < NST * (SE + 1) && kk.y >= 0 && kk.y < NST * (SE + 1));
                    const float4* r1 = recf + 4 * kk.x;
                    const float4* r2 = recf + 4 * kk.y;
                    const float a1 = entry_alpha(r1[0], r1[1], pxf, pyf, P);
                    const float a2 = entry_alpha(r2[0], r2[1], pxf, pyf, P);
                    // 1 - alpha of both entries at once
                    const float2 om = sub2_rn(1.0f, 1.0f, a1, a2);
                    w1 = blend_om(a1, om.x, r1[2]);
                    w2 = blend_om(a2, om.y, r2[2]);
#ifdef GS_RASTER_STATS
                    {
                        const unsigned any1 = __ballot_sync(0xffffffffu, a1 > 0.f), any2 = __ballot_sync(0xffffffffu, a2 > 0.f);
                        const unsigned b1 = __ballot_sync(0xffffffffu, w1 > 0.f), b2 = __ballot_sync(0xffffffffu, w2 > 0.f);
                        if (lane == 0) {
                            // entries with alpha >= alpha_min at some pixel of the warp; lane blends
                            atomicAdd(&g_raster_stats[2], (unsigned long long)((any1 != 0) + (any2 != 0)));
                            atomicAdd(&g_raster_stats[3], (unsigned long long)(__popc(b1) + __popc(b2)));
                        }
                    }
#endif
                };
                // two entry pairs: four independent alphas (ILP 4), then the transmittance chain
                auto walk_quad = [&](const int2 ka, const int2 kb, float (&w)[4]) {
                    const float4* r0 = recf + 4 * ka.x;
                    const float4* r1 = recf + 4 * ka.y;
                    const float4* r2 = recf + 4 * kb.x;
                    const float4* r3 = recf + 4 * kb.y;
                    const float a0 = entry_alpha(r0[0], r0[1], pxf, pyf, P);
                    const float a1 = entry_alpha(r1[0], r1[1], pxf, pyf, P);
                    const float a2 = entry_alpha(r2[0], r2[1], pxf, pyf, P);
                    const float a3 = entry_alpha(r3[0], r3[1], pxf, pyf, P);
                    const float2 om01 = sub2_rn(1.0f, 1.0f, a0, a1), om23 = sub2_rn(1.0f, 1.0f, a2, a3);
                    w[0] = blend_om(a0, om01.x, r0[2]);
                    w[1] = blend_om(a1, om01.y, r1[2]);
                    w[2] = blend_om(a2, om23.x, r2[2]);
                    w[3] = blend_om(a3, om23.y, r3[2]);
                };
                const int ne = (n + 1) & ~1;   // entry pairs (an odd tail pairs with the null record)
                if constexpr (WB) {
                    // chunks that end at a k-step boundary: the pending-row bookkeeping (ring rows
                    // of the weight rows, the oldest referenced stage) is done once per chunk
                    for (int i = 0; i < ne;) {
                        if (pend == 0) hold = s;
                        const int m = min(ne - i, WB_ROWS - pend);
                        if constexpr (Smem::DIRECT_B) feed_rows(i, m);
                        else if (lane < (uint32_t)m) sm.kent[warp][pend + (int)lane] = sm.ent[warp][i + (int)lane];
                        int j = 0;
#if GS_WALK4
#pragma unroll 1
                        for (; j + 4 <= m; j += 4) {
                            const int2 ka = *reinterpret_cast<const int2*>(&sm.ent[warp][i + j]);   // i + j even
                            const int2 kb = *reinterpret_cast<const int2*>(&sm.ent[warp][i + j + 2]);
                            float w[4];
                            walk_quad(ka, kb, w);
                            contrib_put(i + j, w[0], w[1]);
                            if (((i + j + 2) & 31) == 0) contrib_flush(i + j - 30, 32);
                            contrib_put(i + j + 2, w[2], w[3]);
                            if (((i + j + 4) & 31) == 0) contrib_flush(i + j - 28, 32);
                            if constexpr (Smem::DIRECT) {
                                store_pair(w[0], w[1], (pend + j) >> 1);
                                store_pair(w[2], w[3], (pend + j + 2) >> 1);
                            } else {
#pragma unroll
                                for (int q = 0; q < 4; ++q) sm.wbuf[warp][pend + j + q][lane] = w[q];
                            }
                        }
#endif
#pragma unroll 1
                        for (; j < m; j += 2) {
                            const int2 kk = *reinterpret_cast<const int2*>(&sm.ent[warp][i + j]);   // i + j even
                            float w1, w2;
                            walk_pair(kk, w1, w2);
                            contrib_put(i + j, w1, w2);
                            if (((i + j + 2) & 31) == 0) contrib_flush(i + j - 30, 32);
                            if constexpr (Smem::DIRECT) {
                                store_pair(w1, w2, (pend + j) >> 1);
                            } else {
                                sm.wbuf[warp][pend + j][lane] = w1;
                                sm.wbuf[warp][pend + j + 1][lane] = w2;
                            }
                        }
                        pend += m;
                        i += m;
                        if (i >= ne && (ne & 31)) contrib_flush(ne & ~31, ne & 31);
                        if (pend == WB_ROWS) {             // a full k-step: feed the tensor cores
                            __syncwarp();
                            mma_block(0, WB_ROWS);
                            __syncwarp();
                            pend = 0;
                        }
                    }
                } else {
                    int i = 0;
#if GS_WALK4
#pragma unroll 1
                    for (; i + 4 <= ne; i += 4) {
                        const int2 ka = *reinterpret_cast<const int2*>(&sm.ent[warp][i]);
                        const int2 kb = *reinterpret_cast<const int2*>(&sm.ent[warp][i + 2]);
                        float w[4];
                        walk_quad(ka, kb, w);
                        contrib_put(i, w[0], w[1]);
                        if (((i + 2) & 31) == 0) contrib_flush(i - 30, 32);
                        contrib_put(i + 2, w[2], w[3]);
                        if (((i + 4) & 31) == 0) contrib_flush(i - 28, 32);
                    }
#endif
#pragma unroll 1
                    for (; i < ne; i += 2) {
                        float w1, w2;
                        const int2 kk = *reinterpret_cast<const int2*>(&sm.ent[warp][i]);
                        walk_pair(kk, w1, w2);
                        contrib_put(i, w1, w2);
                        if (((i + 2) & 31) == 0) contrib_flush(i - 30, 32);
                    }
                    if (ne & 31) contrib_flush(ne & ~31, ne & 31);
                }
                warp_done = __all_sync(0xffffffffu, done);
            }
        }
        // never pin more than half the ring: the producer must be able to refill
        if (HOLD && pend > 0 && s2 - hold >= NST / 2) flush_pending();
        if (last_flags & ST_LAST) {
            flush_pending();
            // -------------------------------------------------------- outputs
            const int64_t HW = (int64_t)W * H;
            const int64_t po = V->pix_offset;
            if (inside) {
                const int64_t loc = (int64_t)py * W + px;
                GS_DCHECK(loc >= 0 && loc < HW && m.view < n_views);
                // streaming stores (evict-first in L2): the 37-plane output stream must not
                // evict the records / feature rows that neighbouring tiles re-read
                __stcs(&out_rgb[3 * po + loc], C0);
                __stcs(&out_rgb[3 * po + HW + loc], C1);
                __stcs(&out_rgb[3 * po + 2 * HW + loc], C2);
                __stcs(&out_depth[po + loc], Dz);
                __stcs(&out_alpha[po + loc], 1.0f - T);
                if (out_xyz) {   // fused O13 (gs_rasterize_backproject)
                    float X, Y, Z;
                    uint8_t ok;
                    bp_pixel(*V, Dz, 1.0f - T, a_min, px, py, X, Y, Z, ok);
                    __stcs(&out_xyz[3 * po + loc], X);
                    __stcs(&out_xyz[3 * po + HW + loc], Y);
                    __stcs(&out_xyz[3 * po + 2 * HW + loc], Z);
                    out_valid[po + loc] = ok;
                }
            }
            if constexpr (TC) {
                // this lane's pixel row of the group accumulator: D channels
                float f[D];
                if (tile_acc) {
                    const uint32_t jl = kstep - 1u;
                    mbar_wait(&sm.mma_bar[warp][jl & 1u], (jl >> 1) & 1u);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < D; c += 16) tmem_ld16(tD + my_lanes + (uint32_t)c, f + c);
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                } else {
#pragma unroll
                    for (int c = 0; c < D; ++c) f[c] = 0.f;
                }
                if (inside) {
                    // byte address stepped by one plane per channel (64-bit add + store per
                    // channel; the float-index form compiled to index arithmetic + LEA pairs)
                    uint64_t qa = reinterpret_cast<uint64_t>(out_feat + (int64_t)D * po + (int64_t)py * W + px);
                    const uint64_t step = 4ull * (uint64_t)HW;
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        __stcs(reinterpret_cast<float*>(qa), f[c]);
                        qa += step;
                    }
                }
            } else if constexpr (D > 0) {
                // accumulator (a, n, i): pixel (sx + g, sy + 2a + (i >> 1)), channel 8n + 2 t4 + (i & 1);
                // one 64-bit base pointer per (a, i) and a plain pointer walk over the channel planes
                const int fx = sx + g;
                float* fbase = out_feat + (int64_t)D * po + (int64_t)(2 * t4) * HW + fx;
                const int64_t step8 = 8 * HW;
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int fy = sy + 2 * a + (i >> 1);
                        if (fx < W && fy < H) {
                            float* q = fbase + (int64_t)fy * W + ((i & 1) ? HW : 0);
#pragma unroll
                            for (int n = 0; n < NTP; ++n) {
                                if (n * 8 + 2 * t4 + (i & 1) < D) __stcs(q, acc[a][n][i]);
                                q += step8;
                            }
                        }
                    }
            }
        }
        // release every stage no pending row references, in order
        const uint32_t lim = (HOLD && pend > 0) ? hold : s2 + 1;
        __syncwarp();
        for (; rel < lim; ++rel)
            if (lane == 0) mbar_arrive(&sm.empty[rel % NST]);
        s = s2 + 1;
    }
    if constexpr (TC) {
        // every MMA was waited for at its tile's epilogue; free TMEM once all consumers are done
        tc_fence_before();
        asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32) : "memory");
        if (warp == 0) {
            tc_fence_after();
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TcCfg<D>::cols)
                         : "memory");
        }
    }
}

template <int D, bool CONTRIB, bool TC>
gs_status launch(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins, const gs_view* views_dev,
                 int n_views, int64_t T, const gs_params* P, gs_images* out, cudaStream_t s, float a_min,
                 float* xyz, uint8_t* valid) {
    const int smem = (int)sizeof(RasterSmem<D, CONTRIB, TC>);
    // kernel attributes are per device: set on every call (cheap); the occupancy is
    // cached per device
    cudaFuncSetAttribute(rasterize_kernel<D, CONTRIB, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(rasterize_kernel<D, CONTRIB, TC>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    static std::atomic<int> bps_cache[GS_MAX_DEVICES];
    const int cur_dev = current_device();
    const bool cacheable = cur_dev >= 0 && cur_dev < GS_MAX_DEVICES;
    int blocks_per_sm = cacheable ? bps_cache[cur_dev].load(std::memory_order_relaxed) : 0;
    if (blocks_per_sm == 0) {
        const cudaError_t e =
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, rasterize_kernel<D, CONTRIB, TC>, RT_THREADS, smem);
        if (TC) {
            // the occupancy calculator reports 1 CTA/SM for kernels that allocate TMEM;
            // the real limits are shared memory, registers and the 512 TMEM columns
            int dev = 0, smem_sm = 0, regs_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
            cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, rasterize_kernel<D, CONTRIB, TC>);
            const int by_smem = smem_sm / (smem + 1024);
            const int by_regs = regs_sm / (std::max(fa.numRegs, 1) * RT_THREADS);
            const int by_tmem = 512 / (int)TcCfg<D>::cols;
            blocks_per_sm = std::min(std::min(by_smem, by_regs), by_tmem);
        }
        if (const char* o = getenv("GS_RASTER_CTAS_PER_SM")) blocks_per_sm = atoi(o);
        if (getenv("GS_DEBUG"))
            fprintf(stderr, "[gs] rasterize<%d,%d>: smem %d B, occupancy %d CTAs/SM (%s)\n", D, (int)CONTRIB, smem,
                    blocks_per_sm, cudaGetErrorString(e));
        if (blocks_per_sm < 1) blocks_per_sm = 1;
        if (cacheable) bps_cache[cur_dev].store(blocks_per_sm, std::memory_order_relaxed);
    }
    const int64_t grid =
        std::min<int64_t>((T + SCHED_CHUNK - 1) / SCHED_CHUNK, (int64_t)num_sms() * blocks_per_sm);
    if (grid <= 0) return GS_OK;
    if (bins->tile_sched) cudaMemsetAsync(bins->tile_sched, 0, sizeof(uint32_t), s);
    if (CONTRIB) cudaMemsetAsync(proj->contrib, 0, sizeof(unsigned long long) * (size_t)n_views * proj->rec_capacity, s);
    rasterize_kernel<D, CONTRIB, TC><<<(unsigned)grid, RT_THREADS, smem, s>>>(
        views_dev, n_views, proj->rec, bins->sorted_rec, bins->sorted_gid, bins->ranges, (uint32_t)T, bins->tile_sched,
        scene->feat, reinterpret_cast<const __half*>(scene->feat_h),
        *P, out->rgb, out->depth, out->alpha, out->feat, proj->contrib, proj->status, a_min, xyz, valid);
    return check_launch("rasterize_kernel");
}

// ---------------------------------------------------------------- N4 backward
// Feature-field backward of Eq. 2 with the geometry frozen:
// dL/df_g += sum over pixels of w_g(px) * dL/dF(px).  One CTA per tile (8 warps
// x 8x4 pixels, the forward's exact per-pixel walk: same cull, exponent, alpha,
// stop rule), the tile list in chunks of BW_CHUNK entries.  Per warp, the
// weights of 16 walked entries feed m16n8k16 MMAs G[entry][ch] = W[entry][px] .
// g[px][ch] (fp16 hi + lo operands, 3 products; the warp's upstream gradients
// live in registers as B fragments for the whole tile), reduced over the 8
// warps in shared memory, then one global atomic per (entry, channel) per chunk.
constexpr int BW_CHUNK = 64;

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

template <int D>
__global__ void __launch_bounds__(256)
feature_backward_kernel(const gs_view* __restrict__ views, int n_views, const gs_record* __restrict__ rec,
                        const uint32_t* __restrict__ sorted_rec, const uint32_t* __restrict__ ranges, gs_params P,
                        const float* __restrict__ gimg, float* __restrict__ grad, const uint32_t* __restrict__ status) {
    if (*status) return;
    constexpr int NT = D / 8;
    __shared__ float4 srec[BW_CHUNK + 1][2];      // u, v, ea, eb | ec, o, e_cut, - ; row BW_CHUNK = null
    __shared__ uint32_t sgid[BW_CHUNK];
    __shared__ float acc[BW_CHUNK][D + 1];
    __shared__ __align__(16) float wbuf[8][16][36];
    __shared__ int ent[8][BW_CHUNK + 18];
    const uint32_t tile = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int vi = find_view_by_tile(views, n_views, tile);
    const gs_view& V = views[vi];
    const int W = V.width, H = V.height, TX = (W + GS_TILE - 1) / GS_TILE;
    const uint32_t lt = tile - V.tile_offset;
    const int sx = (int)(lt % (uint32_t)TX) * 16 + (warp & 1) * 8, sy = (int)(lt / (uint32_t)TX) * 16 + (warp >> 1) * 4;
    const int px = sx + (lane & 7), py = sy + (lane >> 3);
    const bool inside = px < W && py < H;
    const float pxf = (float)px, pyf = (float)py;
    const float rx0 = (float)sx, rx1 = (float)(sx + 7), ry0 = (float)sy, ry1 = (float)(sy + 3);
    const int64_t HW = (int64_t)W * H;
    const float* G = gimg + (int64_t)D * V.pix_offset;
    // B fragments of this warp's upstream gradients: k = pixel p (p -> (p & 7, p >> 3)), n = channel
    auto gval = [&](int p, int ch) -> float {
        const int x = sx + (p & 7), y = sy + (p >> 3);
        return (x < W && y < H) ? __ldg(&G[(int64_t)ch * HW + (int64_t)y * W + x]) : 0.f;
    };
    uint32_t bh[NT][2][2], bl[NT][2][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int p = 16 * ks + 8 * r + 2 * t4, ch = 8 * nt + g;
                const float v0 = gval(p, ch), v1 = gval(p + 1, ch);
                const __half2 h = __floats2half2_rn(v0, v1);
                const float2 hf = __half22float2(h);
                bh[nt][ks][r] = *reinterpret_cast<const uint32_t*>(&h);
                bl[nt][ks][r] = pack_h2(v0 - hf.x, v1 - hf.y);
            }
    for (int i = tid; i < BW_CHUNK * (D + 1); i += 256) (&acc[0][0])[i] = 0.f;
    if (tid < 2) srec[BW_CHUNK][tid] = make_float4(0.f, 0.f, 0.f, 0.f);
    float T = 1.0f;
    bool done = !inside;
    bool warp_done = __all_sync(0xffffffffu, done);
    const uint32_t rs = ranges[2 * tile], re = ranges[2 * tile + 1];
    // 16 walked entries -> G rows added to acc[chunk entry][ch]
    auto kstep = [&](int eb) {
        float d[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            uint32_t ah[4], al[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = g + ((i & 1) ? 8 : 0), p = 16 * ks + 2 * t4 + ((i & 2) ? 8 : 0);
                const float w0 = wbuf[warp][row][p], w1 = wbuf[warp][row][p + 1];
                const __half2 h = __floats2half2_rn(w0, w1);
                const float2 hf = __half22float2(h);
                ah[i] = *reinterpret_cast<const uint32_t*>(&h);
                al[i] = pack_h2(w0 - hf.x, w1 - hf.y);
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                mma_f16(d[nt], ah, bh[nt][ks][0], bh[nt][ks][1]);
                mma_f16(d[nt], ah, bl[nt][ks][0], bl[nt][ks][1]);
                mma_f16(d[nt], al, bh[nt][ks][0], bh[nt][ks][1]);
            }
        }
        const int e0 = ent[warp][eb + g], e1 = ent[warp][eb + g + 8];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int ch = 8 * nt + 2 * t4;
            if (e0 < BW_CHUNK) { atomicAdd(&acc[e0][ch], d[nt][0]); atomicAdd(&acc[e0][ch + 1], d[nt][1]); }
            if (e1 < BW_CHUNK) { atomicAdd(&acc[e1][ch], d[nt][2]); atomicAdd(&acc[e1][ch + 1], d[nt][3]); }
        }
    };
    __syncthreads();
    for (uint32_t c0 = rs; c0 < re; c0 += BW_CHUNK) {
        const int cnt = (int)min((uint32_t)BW_CHUNK, re - c0);
        for (int i = tid; i < 2 * cnt; i += 256) {
            const uint32_t slot = __ldg(&sorted_rec[c0 + i / 2]);
            srec[i / 2][i & 1] = __ldg(reinterpret_cast<const float4*>(rec + slot) + (i & 1));
            if ((i & 1) == 0) sgid[i / 2] = __ldg(&rec[slot].gid);
        }
        __syncthreads();
        if (!warp_done) {
            bool hit[2] = {false, false};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = lane + 32 * h;
                if (j < cnt) {
                    const float4 a = srec[j][0], b = srec[j][1];
                    hit[h] = ellipse_hits_rect(a.x, a.y, a.z, a.w, b.x, b.z, rx0, rx1, ry0, ry1);
                }
            }
            const uint32_t m0 = __ballot_sync(0xffffffffu, hit[0]), m1 = __ballot_sync(0xffffffffu, hit[1]);
            const int n0 = __popc(m0), n = n0 + __popc(m1);
            const uint32_t below = (1u << lane) - 1u;
            if (hit[0]) ent[warp][__popc(m0 & below)] = lane;
            if (hit[1]) ent[warp][n0 + __popc(m1 & below)] = lane + 32;
            const int np = (n + 15) & ~15;                     // padded to whole K steps
            if (lane < np - n) ent[warp][n + lane] = BW_CHUNK;  // null rows
            __syncwarp();
            for (int i = 0; i < np; ++i) {
                const int k = ent[warp][i];
                float a = entry_alpha(srec[k][0], srec[k][1], pxf, pyf, P);
                a = (done || k == BW_CHUNK) ? 0.0f : a;
                const float Tn = __fmul_rn(T, __fsub_rn(1.0f, a));
                const bool stop = Tn < P.t_min;
                const float wgt = stop ? 0.0f : __fmul_rn(a, T);
                T = stop ? T : Tn;
                done = done || stop;
                wbuf[warp][i & 15][lane] = wgt;
                if ((i & 15) == 15) {
                    __syncwarp();
                    kstep(i - 15);
                    __syncwarp();
                }
            }
            warp_done = __all_sync(0xffffffffu, done);
        }
        __syncthreads();
        for (int i = tid; i < cnt * D; i += 256) {
            const int e = i / D, ch = i % D;
            const float v = acc[e][ch];
            if (v != 0.f) {
                atomicAdd(&grad[(int64_t)sgid[e] * D + ch], v);
                acc[e][ch] = 0.f;
            }
        }
        __syncthreads();
    }
}

template <int D>
gs_status launch_backward(const gs_projected* proj, const gs_bins* bins, const gs_view* views_dev, int n_views,
                          int64_t T, const gs_params* P, const float* gimg, float* grad, cudaStream_t s) {
    if (T <= 0) return GS_OK;
    feature_backward_kernel<D><<<(unsigned)T, 256, 0, s>>>(views_dev, n_views, proj->rec, bins->sorted_rec,
                                                           bins->ranges, *P, gimg, grad, proj->status);
    return check_launch("feature_backward_kernel");
}

// Radiance backward: per record slot, the gradient of
// L = sum_px gC . C + gD Dz + gA A w.r.t. {u, v, ea, eb, ec, opacity, r, g, b, z},
// front to back from the forward's outputs (no division by T):
//   dC/dalpha_k = T_k c_k - (C_f - C_<=k) / (1 - alpha_k),  dA/dalpha_k = T_f / (1 - alpha_k).
// Same tile / chunk / warp structure as the feature backward; the 10 per-pixel
// terms of each walked entry are warp-reduced, summed over the warps in shared
// memory and flushed with one global atomic per (entry, field) per chunk.
// DF > 0 (gs_joint_backward, Eq. 1 with Eq. 2's feature term through the geometry):
// the rendered feature vector F = sum_k w_k f_k enters like a colour channel with
// the pixel's upstream gradient gF: dL/dalpha_k += T_k (gF . f_k) - (gF . F -
// sum_{j<=k} w_j gF . f_j) / (1 - alpha_k)  (the scalar gF . f_k per walked entry
// and pixel, fp32 from the scene's fp32 feature rows staged per chunk).
constexpr int NGRAD = 10;

template <int DF>
__global__ void __launch_bounds__(256, DF > 0 ? 3 : 4)
radiance_backward_kernel(const gs_view* __restrict__ views, int n_views, const gs_record* __restrict__ rec,
                         const uint32_t* __restrict__ sorted_rec, const uint32_t* __restrict__ ranges, gs_params P,
                         const float* __restrict__ img_rgb, const float* __restrict__ img_depth,
                         const float* __restrict__ img_alpha, const float* __restrict__ g_rgb,
                         const float* __restrict__ g_depth, const float* __restrict__ g_alpha,
                         float* __restrict__ grec, const uint32_t* __restrict__ status,
                         const float* __restrict__ feat, const float* __restrict__ img_feat,
                         const float* __restrict__ g_feat) {
    if (*status) return;
    __shared__ float4 srec[BW_CHUNK + 1][3];
    __shared__ __align__(16) float sfeat[DF > 0 ? BW_CHUNK + 1 : 1][DF > 0 ? DF : 4];   // row BW_CHUNK = 0
    // gF . f_k of 16 walked entries x the warp's 32 pixels (tensor-core dots, below)
    __shared__ float sdot[DF > 0 ? 8 : 1][DF > 0 ? 16 : 1][DF > 0 ? 33 : 1];
    __shared__ uint32_t sslot[BW_CHUNK];
    __shared__ float acc[BW_CHUNK][NGRAD + 1];
    __shared__ int ent[8][2 * 32 + 2];
    const uint32_t tile = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vi = find_view_by_tile(views, n_views, tile);
    const gs_view& V = views[vi];
    const int W = V.width, H = V.height, TX = (W + GS_TILE - 1) / GS_TILE;
    const uint32_t lt = tile - V.tile_offset;
    const int sx = (int)(lt % (uint32_t)TX) * 16 + (warp & 1) * 8, sy = (int)(lt / (uint32_t)TX) * 16 + (warp >> 1) * 4;
    const int px = sx + (lane & 7), py = sy + (lane >> 3);
    const bool inside = px < W && py < H;
    const float pxf = (float)px, pyf = (float)py;
    const float rx0 = (float)sx, rx1 = (float)(sx + 7), ry0 = (float)sy, ry1 = (float)(sy + 3);
    const int64_t HW = (int64_t)W * H, po = V.pix_offset, loc = (int64_t)py * W + px;
    float Cf[3] = {0.f, 0.f, 0.f}, Df = 0.f, Tf = 1.f, gC[3] = {0.f, 0.f, 0.f}, gD = 0.f, gA = 0.f;
    if (inside) {
        for (int q = 0; q < 3; ++q) {
            Cf[q] = __ldg(&img_rgb[3 * po + q * HW + loc]);
            gC[q] = __ldg(&g_rgb[3 * po + q * HW + loc]);
        }
        Df = __ldg(&img_depth[po + loc]);
        Tf = 1.0f - __ldg(&img_alpha[po + loc]);
        gD = __ldg(&g_depth[po + loc]);
        gA = __ldg(&g_alpha[po + loc]);
    }
    // feature term: gF . F of the forward's map at this pixel, and the warp's upstream
    // gradients as fp16 hi / lo B fragments of m16n8k16 MMAs (k = channel, n = pixel
    // 8 nt + g of the warp's 8x4 block, the same pixel numbering as the lanes)
    float SF = 0.f, Sacc = 0.f;
    constexpr int KS = DF > 0 ? (DF + 15) / 16 : 1;
    uint32_t gbh[DF > 0 ? 4 : 1][KS][2], gbl[DF > 0 ? 4 : 1][KS][2];
    if constexpr (DF > 0) {
        const int g8 = lane >> 2, t4 = lane & 3;
        const float* GF = g_feat + (int64_t)DF * po;
#pragma unroll
        for (int c = 0; c < DF; ++c)
            if (inside) SF = fmaf(__ldg(&GF[(int64_t)c * HW + loc]), __ldg(&img_feat[(int64_t)DF * po + (int64_t)c * HW + loc]), SF);
        auto gv = [&](int p, int c) -> float {
            const int x = sx + (p & 7), y = sy + (p >> 3);
            return (c < DF && x < W && y < H) ? __ldg(&GF[(int64_t)c * HW + (int64_t)y * W + x]) : 0.f;
        };
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const int p = 8 * nt + g8, c = 16 * ks + 2 * t4 + 8 * r;
                    const float v0 = gv(p, c), v1 = gv(p, c + 1);
                    const __half2 h = __floats2half2_rn(v0, v1);
                    const float2 hf = __half22float2(h);
                    gbh[nt][ks][r] = *reinterpret_cast<const uint32_t*>(&h);
                    gbl[nt][ks][r] = pack_h2(v0 - hf.x, v1 - hf.y);
                }
    }
    // dots of the walked entries ent[eb .. eb + 16) (row BW_CHUNK beyond the list) with
    // the 32 pixels' gF: A = feature rows (fp16 hi / lo), 3 products per k-step (~2^-22)
    auto dots16 = [&](int eb, int n_ent) {
        if constexpr (DF > 0) {
            const int g8 = lane >> 2, t4 = lane & 3;
            const int e0 = eb + g8 < n_ent ? ent[warp][eb + g8] : BW_CHUNK;
            const int e1 = eb + g8 + 8 < n_ent ? ent[warp][eb + g8 + 8] : BW_CHUNK;
            float d[4][4];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                uint32_t ah[4], al[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int e = (i & 1) ? e1 : e0, c = 16 * ks + 2 * t4 + ((i & 2) ? 8 : 0);
                    const float f0 = c < DF ? sfeat[e][c] : 0.f, f1 = c + 1 < DF ? sfeat[e][c + 1] : 0.f;
                    const __half2 h = __floats2half2_rn(f0, f1);
                    const float2 hf = __half22float2(h);
                    ah[i] = *reinterpret_cast<const uint32_t*>(&h);
                    al[i] = pack_h2(f0 - hf.x, f1 - hf.y);
                }
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    mma_f16(d[nt], ah, gbh[nt][ks][0], gbh[nt][ks][1]);
                    mma_f16(d[nt], ah, gbl[nt][ks][0], gbl[nt][ks][1]);
                    mma_f16(d[nt], al, gbh[nt][ks][0], gbh[nt][ks][1]);
                }
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int px0 = 8 * nt + 2 * t4;
                sdot[warp][g8][px0] = d[nt][0];
                sdot[warp][g8][px0 + 1] = d[nt][1];
                sdot[warp][g8 + 8][px0] = d[nt][2];
                sdot[warp][g8 + 8][px0 + 1] = d[nt][3];
            }
            __syncwarp();
        }
    };
    for (int i = tid; i < BW_CHUNK * (NGRAD + 1); i += 256) (&acc[0][0])[i] = 0.f;
    if constexpr (DF > 0)
        for (int i = tid; i < DF; i += 256) sfeat[BW_CHUNK][i] = 0.f;
    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Dz = 0.f;
    bool done = !inside;
    bool warp_done = __all_sync(0xffffffffu, done);
    const uint32_t rs = ranges[2 * tile], re = ranges[2 * tile + 1];
    __syncthreads();
    for (uint32_t c0 = rs; c0 < re; c0 += BW_CHUNK) {
        const int cnt = (int)min((uint32_t)BW_CHUNK, re - c0);
        for (int i = tid; i < 3 * cnt; i += 256) {
            const uint32_t slot = __ldg(&sorted_rec[c0 + i / 3]);
            srec[i / 3][i % 3] = __ldg(reinterpret_cast<const float4*>(rec + slot) + (i % 3));
            if (i % 3 == 0) sslot[i / 3] = slot;
        }
        if constexpr (DF > 0) {
            // the chunk's feature rows (gid of each entry read once, then coalesced float4 rows)
            __syncthreads();
            for (int i = tid; i < cnt * (DF / 4); i += 256) {
                const int e = i / (DF / 4), q = i % (DF / 4);
                const uint32_t g = __ldg(&rec[sslot[e]].gid);
                reinterpret_cast<float4*>(&sfeat[e][0])[q] = __ldg(reinterpret_cast<const float4*>(feat + (int64_t)g * DF) + q);
            }
        }
        __syncthreads();
        if (!warp_done) {
            bool hit[2] = {false, false};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = lane + 32 * h;
                if (j < cnt) {
                    const float4 a = srec[j][0], b = srec[j][1];
                    hit[h] = ellipse_hits_rect(a.x, a.y, a.z, a.w, b.x, b.z, rx0, rx1, ry0, ry1);
                }
            }
            const uint32_t m0 = __ballot_sync(0xffffffffu, hit[0]), m1 = __ballot_sync(0xffffffffu, hit[1]);
            const int n0 = __popc(m0), n = n0 + __popc(m1);
            const uint32_t below = (1u << lane) - 1u;
            if (hit[0]) ent[warp][__popc(m0 & below)] = lane;
            if (hit[1]) ent[warp][n0 + __popc(m1 & below)] = lane + 32;
            __syncwarp();
            for (int i = 0; i < n; ++i) {
                if constexpr (DF > 0)
                    if ((i & 15) == 0) dots16(i, n);
                const int k = ent[warp][i];
                const float4 a4 = srec[k][0], b4 = srec[k][1], c4 = srec[k][2];
                // the forward's exponent / alpha (entry_alpha), keeping 2^p and the raw alpha
                const float dx = __fsub_rn(a4.x, pxf), dy = __fsub_rn(a4.y, pyf);
                const float p = __fmaf_rn(dx, __fmaf_rn(a4.z, dx, __fmul_rn(a4.w, dy)), __fmul_rn(__fmul_rn(b4.x, dy), dy));
                const float e2p = ex2_ftz(p);
                const float araw = __fmul_rn(b4.y, e2p);
                float alpha = fminf(P.alpha_max, araw);
                alpha = ((p > 0.0f) || (alpha < P.alpha_min) || done) ? 0.0f : alpha;
                const float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                const bool stop = Tn < P.t_min;
                const float wgt = stop ? 0.0f : __fmul_rn(alpha, T);
                float g[16];   // NGRAD fields, padded for the halving reduction
#pragma unroll
                for (int q = 0; q < 16; ++q) g[q] = 0.f;
                const bool blended = wgt > 0.f;
                float dot = 0.f;                       // gF . f_k (feature term)
                if constexpr (DF > 0) dot = sdot[warp][i & 15][lane];
                if (blended) {
                    C0 = fmaf(wgt, c4.x, C0); C1 = fmaf(wgt, c4.y, C1); C2 = fmaf(wgt, c4.z, C2); Dz = fmaf(wgt, c4.w, Dz);
                    const float iom = __frcp_rn(1.0f - alpha);
                    float dLda = gC[0] * (T * c4.x - (Cf[0] - C0) * iom) + gC[1] * (T * c4.y - (Cf[1] - C1) * iom) +
                                 gC[2] * (T * c4.z - (Cf[2] - C2) * iom) + gD * (T * c4.w - (Df - Dz) * iom) +
                                 gA * (Tf * iom);
                    if constexpr (DF > 0) {
                        Sacc = fmaf(wgt, dot, Sacc);
                        dLda += T * dot - (SF - Sacc) * iom;
                    }
                    g[6] = wgt * gC[0]; g[7] = wgt * gC[1]; g[8] = wgt * gC[2]; g[9] = wgt * gD;
                    if (araw <= P.alpha_max) {
                        g[5] = dLda * e2p;
                        const float dLdp = dLda * araw * 0.6931471805599453f;
                        g[2] = dLdp * dx * dx; g[3] = dLdp * dx * dy; g[4] = dLdp * dy * dy;
                        g[0] = dLdp * (2.f * a4.z * dx + a4.w * dy);
                        g[1] = dLdp * (a4.w * dx + 2.f * b4.x * dy);
                    }
                }
                T = stop ? T : Tn;
                done = done || stop;
                if (!__any_sync(0xffffffffu, blended)) continue;
                // halving butterfly: 16 values over 32 lanes in 16 shuffles; afterwards lanes
                // 2q and 2q + 1 hold the warp sum of field q
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const bool up = lane & 16;
                    const float send = up ? g[j] : g[j + 8], keep = up ? g[j + 8] : g[j];
                    g[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const bool up = lane & 8;
                    const float send = up ? g[j] : g[j + 4], keep = up ? g[j + 4] : g[j];
                    g[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const bool up = lane & 4;
                    const float send = up ? g[j] : g[j + 2], keep = up ? g[j + 2] : g[j];
                    g[j] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                }
                {
                    const bool up = lane & 2;
                    const float send = up ? g[0] : g[1], keep = up ? g[1] : g[0];
                    g[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
                }
                g[0] += __shfl_xor_sync(0xffffffffu, g[0], 1);
                const int q = lane >> 1;
                if ((lane & 1) == 0 && q < NGRAD && g[0] != 0.f) atomicAdd(&acc[k][q], g[0]);
            }
            warp_done = __all_sync(0xffffffffu, done);
        }
        __syncthreads();
        for (int i = tid; i < cnt * NGRAD; i += 256) {
            const int e = i / NGRAD, q = i % NGRAD;
            const float v = acc[e][q];
            if (v != 0.f) {
                atomicAdd(&grec[(int64_t)sslot[e] * NGRAD + q], v);
                acc[e][q] = 0.f;
            }
        }
        __syncthreads();
    }
}

// N4 training helpers: L1 loss of Eq. 2 and a plain gradient step
__global__ void l1_grad_kernel(const float* __restrict__ F, const float* __restrict__ Ft, int64_t n, float scale,
                               float* __restrict__ gF, double* __restrict__ loss) {
    double part = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float d = F[i] - Ft[i];
        gF[i] = d > 0.f ? scale : (d < 0.f ? -scale : 0.f);
        part += (double)fabsf(d) * scale;
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(loss, part);
}

// Eq. 3's L1 term against the appearance-varied rendering (reading Q38): plane p of
// hw pixels, I^a = a[p] I^r + b[p]; grad = scale sign(I^a - I) a[p] (written), and
// per plane dL/da = scale sum sign * I^r, dL/db = scale sum sign (accumulated).
__global__ void appearance_l1_kernel(const float* __restrict__ r, const float* __restrict__ t, int64_t hw,
                                     const float* __restrict__ a, const float* __restrict__ b, float scale,
                                     float* __restrict__ g, float* __restrict__ ga, float* __restrict__ gb,
                                     double* __restrict__ loss) {
    const int p = blockIdx.y;
    const float ap = a[p], bp = b[p];
    const int64_t base = (int64_t)p * hw;
    float sa = 0.f, sb = 0.f;
    double ls = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = r[base + i];
        const float d = fmaf(ap, x, bp) - t[base + i];
        const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
        g[base + i] = scale * sg * ap;
        sa = fmaf(sg, x, sa);
        sb += sg;
        ls += (double)fabsf(d);
    }
    for (int o = 16; o; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
        ls += __shfl_xor_sync(0xffffffffu, ls, o);
    }
    __shared__ float s_a[32], s_b[32];
    __shared__ double s_l[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { s_a[w] = sa; s_b[w] = sb; s_l[w] = ls; }
    __syncthreads();
    if (threadIdx.x == 0) {
        float ta = 0.f, tb = 0.f;
        double tl = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { ta += s_a[k]; tb += s_b[k]; tl += s_l[k]; }
        atomicAdd(&ga[p], scale * ta);
        atomicAdd(&gb[p], scale * tb);
        atomicAdd(loss, (double)scale * tl);
    }
}

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float bc1,
                            float bc2, __half* __restrict__ ph) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float gi = g[i];
        const float mi = b1 * m[i] + (1.0f - b1) * gi;
        const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const float pi = p[i] - lr * (mi * bc1) / (sqrtf(vi * bc2) + eps);
        p[i] = pi;
        if (ph) ph[i] = __float2half_rn(pi);
    }
}

__global__ void sgd_kernel(float* __restrict__ feat, const float* __restrict__ grad, int64_t n, float lr,
                           __half* __restrict__ feat_h) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float f = feat[i] - lr * grad[i];
        feat[i] = f;
        if (feat_h) feat_h[i] = __float2half_rn(f);
    }
}

}  // namespace
}  // namespace gs

using namespace gs;

static gs_status rasterize_impl(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                                const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                                const gs_params* params, gs_images* out, void* stream, float a_min, float* xyz,
                                uint8_t* valid) {
    gs_status st = validate_scene(scene, false);
    if (st != GS_OK) return st;
    int64_t total_pixels = 0, T = 0;
    st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(params != nullptr, GS_INVALID_ARG, "params is NULL");
    GS_REQUIRE(proj && proj->rec && proj->status, GS_INVALID_ARG, "proj has a NULL pointer");
    GS_REQUIRE(bins && bins->ranges && bins->sorted_rec, GS_INVALID_ARG, "bins has a NULL pointer");
    GS_REQUIRE(out && out->rgb && out->depth && out->alpha, GS_INVALID_ARG, "images has a NULL pointer");
    GS_REQUIRE(scene->feat_dim == 0 || out->feat != nullptr, GS_INVALID_ARG, "feat_dim = %d but images.feat is NULL",
               scene->feat_dim);
    GS_REQUIRE(scene->feat_dim == 0 || scene->feat != nullptr, GS_INVALID_ARG, "scene feat is NULL");
    GS_REQUIRE(((uintptr_t)proj->rec & 15) == 0 && (scene->feat_dim == 0 || ((uintptr_t)scene->feat & 15) == 0),
               GS_INVALID_ARG, "records and features must be 16-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    const bool tc = scene->feat_h != nullptr;
    GS_REQUIRE(!tc || ((uintptr_t)scene->feat_h & 15) == 0, GS_INVALID_ARG, "feat_h must be 16-byte aligned");
    switch (scene->feat_dim) {
#define GS_CASE(d) \
    case d:                                                                                       \
        return proj->contrib ? launch<d, true, false>(scene, proj, bins, views_dev, n_views, T, params, out, s, a_min, xyz, valid) \
                             : launch<d, false, false>(scene, proj, bins, views_dev, n_views, T, params, out, s, a_min, xyz, valid);
#define GS_CASE_TC(d) \
    case d:                                                                                              \
        if (tc)                                                                                          \
            return proj->contrib ? launch<d, true, true>(scene, proj, bins, views_dev, n_views, T, params, out, s, a_min, xyz, valid) \
                                 : launch<d, false, true>(scene, proj, bins, views_dev, n_views, T, params, out, s, a_min, xyz, valid); \
        return proj->contrib ? launch<d, true, false>(scene, proj, bins, views_dev, n_views, T, params, out, s, a_min, xyz, valid) \
                             : launch<d, false, false>(scene, proj, bins, views_dev, n_views, T, params, out, s, a_min, xyz, valid);
        GS_CASE(0) GS_CASE(4) GS_CASE(8) GS_CASE(12) GS_CASE_TC(16) GS_CASE(20) GS_CASE(24) GS_CASE(28)
        GS_CASE_TC(32) GS_CASE(36) GS_CASE(40) GS_CASE(44) GS_CASE_TC(48) GS_CASE(52) GS_CASE(56) GS_CASE(60)
        GS_CASE_TC(64)
#undef GS_CASE
#undef GS_CASE_TC
        default:
            gs::set_error("feat_dim = %d unsupported", scene->feat_dim);
            return GS_UNSUPPORTED;
    }
}

extern "C" gs_status gs_rasterize(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                                  const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                                  const gs_params* params, gs_images* out, void* stream) {
    return rasterize_impl(scene, proj, bins, views_host, views_dev, n_views, params, out, stream, 0.0f, nullptr,
                          nullptr);
}

extern "C" gs_status gs_rasterize_backproject(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                                              const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                                              const gs_params* params, gs_images* out, float a_min, float* xyz,
                                              uint8_t* valid, void* stream) {
    GS_REQUIRE(xyz && valid, GS_INVALID_ARG, "xyz/valid is NULL");
    GS_REQUIRE(a_min == a_min, GS_INVALID_ARG, "a_min is NaN");
    return rasterize_impl(scene, proj, bins, views_host, views_dev, n_views, params, out, stream, a_min, xyz, valid);
}

namespace gs {
namespace {
__global__ void probe_alpha_kernel(const float* __restrict__ o, const float* __restrict__ p, int64_t n,
                                   float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = alpha_raw(o[i], p[i]);
}

__global__ void features_f16_kernel(const float4* __restrict__ f, uint2* __restrict__ out, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 x = f[i];
        const __half2 a = __floats2half2_rn(x.x, x.y), b = __floats2half2_rn(x.z, x.w);
        out[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
}
}  // namespace
}  // namespace gs

extern "C" gs_status gs_probe_alpha(const float* opacity, const float* power, int64_t n, float* alpha_out,
                                    void* stream) {
    GS_REQUIRE(n >= 0 && (n == 0 || (opacity && power && alpha_out)), GS_INVALID_ARG, "gs_probe_alpha: bad arguments");
    if (n == 0) return GS_OK;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
    probe_alpha_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(opacity, power, n, alpha_out);
    return check_launch("probe_alpha_kernel");
}

extern "C" gs_status gs_scene_features_f16(const gs_scene* scene, void* feat_h_out, void* stream) {
    gs_status st = validate_scene(scene, false);
    if (st != GS_OK) return st;
    GS_REQUIRE(scene->feat_dim > 0 && scene->feat != nullptr, GS_INVALID_ARG, "scene has no features");
    GS_REQUIRE(feat_h_out != nullptr && ((uintptr_t)feat_h_out & 15) == 0 && ((uintptr_t)scene->feat & 15) == 0,
               GS_INVALID_ARG, "feature buffers must be non-NULL and 16-byte aligned");
    const int64_t n4 = scene->n * scene->feat_dim / 4;
    if (n4 == 0) return GS_OK;
    const int64_t blocks = std::min<int64_t>((n4 + 255) / 256, (int64_t)num_sms() * 8);
    features_f16_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float4*>(scene->feat), reinterpret_cast<uint2*>(feat_h_out), n4);
    return check_launch("features_f16_kernel");
}

extern "C" gs_status gs_feature_backward(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                                         const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                                         const gs_params* params, const float* grad_image, float* grad_feat,
                                         void* stream) {
    gs_status st = validate_scene(scene, false);
    if (st != GS_OK) return st;
    int64_t total_pixels = 0, T = 0;
    st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(params && proj && proj->rec && proj->status && bins && bins->ranges && bins->sorted_rec && grad_image &&
                   grad_feat,
               GS_INVALID_ARG, "gs_feature_backward: NULL pointer");
    cudaStream_t s = (cudaStream_t)stream;
    switch (scene->feat_dim) {
        case 8: return launch_backward<8>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        case 16: return launch_backward<16>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        case 24: return launch_backward<24>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        case 32: return launch_backward<32>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        case 40: return launch_backward<40>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        case 48: return launch_backward<48>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        case 56: return launch_backward<56>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        case 64: return launch_backward<64>(proj, bins, views_dev, n_views, T, params, grad_image, grad_feat, s);
        default:
            gs::set_error("gs_feature_backward: feat_dim = %d (need a multiple of 8, 8..64)", scene->feat_dim);
            return GS_UNSUPPORTED;
    }
}

extern "C" gs_status gs_feature_l1_grad(const float* rendered, const float* target, int64_t n, float scale,
                                        float* grad_image, double* loss, void* stream) {
    GS_REQUIRE(rendered && target && grad_image && loss && n >= 0, GS_INVALID_ARG, "gs_feature_l1_grad: bad args");
    if (n == 0) return GS_OK;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    l1_grad_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(rendered, target, n, scale, grad_image, loss);
    return check_launch("l1_grad_kernel");
}

extern "C" gs_status gs_appearance_l1_grad(const float* rendered, const float* target, int32_t n_planes,
                                           int64_t plane_pixels, const float* a, const float* b, float scale,
                                           float* grad_image, float* grad_a, float* grad_b, double* loss,
                                           void* stream) {
    GS_REQUIRE(n_planes >= 0 && n_planes <= 65535 && plane_pixels >= 0, GS_INVALID_ARG,
               "gs_appearance_l1_grad: bad sizes");
    if (n_planes == 0 || plane_pixels == 0) return GS_OK;
    GS_REQUIRE(rendered && target && a && b && grad_image && grad_a && grad_b && loss, GS_INVALID_ARG,
               "gs_appearance_l1_grad: NULL pointer");
    const int64_t bx = std::max<int64_t>(1, std::min<int64_t>((plane_pixels + 1023) / 1024,
                                                              (int64_t)num_sms() * 8 / n_planes + 1));
    appearance_l1_kernel<<<dim3((unsigned)bx, (unsigned)n_planes), 256, 0, (cudaStream_t)stream>>>(
        rendered, target, plane_pixels, a, b, scale, grad_image, grad_a, grad_b, loss);
    return check_launch("appearance_l1_kernel");
}

extern "C" gs_status gs_feature_sgd(float* feat, const float* grad_feat, int64_t n, float lr, void* feat_h,
                                    void* stream) {
    GS_REQUIRE(feat && grad_feat && n >= 0, GS_INVALID_ARG, "gs_feature_sgd: bad args");
    if (n == 0) return GS_OK;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    sgd_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(feat, grad_feat, n, lr,
                                                                   reinterpret_cast<__half*>(feat_h));
    return check_launch("sgd_kernel");
}

extern "C" gs_status gs_adam(float* param, const float* grad, float* m, float* v, int64_t n, float lr, float beta1,
                              float beta2, float eps, int32_t step, void* param_h, void* stream) {
    GS_REQUIRE(param && grad && m && v && n >= 0 && step >= 1, GS_INVALID_ARG, "gs_adam: bad args");
    if (n == 0) return GS_OK;
    const float bc1 = (float)(1.0 / (1.0 - std::pow((double)beta1, step)));
    const float bc2 = (float)(1.0 / (1.0 - std::pow((double)beta2, step)));
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    adam_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(param, grad, m, v, n, lr, beta1, beta2, eps, bc1,
                                                                    bc2, reinterpret_cast<__half*>(param_h));
    return check_launch("adam_kernel");
}

extern "C" gs_status gs_radiance_backward(const gs_projected* proj, const gs_bins* bins, const gs_view* views_host,
                                          const gs_view* views_dev, int32_t n_views, const gs_params* params,
                                          const gs_images* fwd, const gs_images* grad_out, float* grad_rec,
                                          void* stream) {
    int64_t total_pixels = 0, T = 0;
    gs_status st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(params && proj && proj->rec && proj->status && bins && bins->ranges && bins->sorted_rec && fwd &&
                   fwd->rgb && fwd->depth && fwd->alpha && grad_out && grad_out->rgb && grad_out->depth &&
                   grad_out->alpha && grad_rec,
               GS_INVALID_ARG, "gs_radiance_backward: NULL pointer");
    if (T <= 0) return GS_OK;
    radiance_backward_kernel<0><<<(unsigned)T, 256, 0, (cudaStream_t)stream>>>(
        views_dev, n_views, proj->rec, bins->sorted_rec, bins->ranges, *params, fwd->rgb, fwd->depth, fwd->alpha,
        grad_out->rgb, grad_out->depth, grad_out->alpha, grad_rec, proj->status, nullptr, nullptr, nullptr);
    return check_launch("radiance_backward_kernel");
}

extern "C" gs_status gs_joint_backward(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                                       const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                                       const gs_params* params, const gs_images* fwd, const gs_images* grad_out,
                                       float* grad_rec, void* stream) {
    if (grad_out == nullptr || grad_out->feat == nullptr || scene == nullptr || scene->feat_dim == 0)
        return gs_radiance_backward(proj, bins, views_host, views_dev, n_views, params, fwd, grad_out, grad_rec,
                                    stream);
    gs_status st = validate_scene(scene, false);
    if (st != GS_OK) return st;
    int64_t total_pixels = 0, T = 0;
    st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(params && proj && proj->rec && proj->status && bins && bins->ranges && bins->sorted_rec && fwd &&
                   fwd->rgb && fwd->depth && fwd->alpha && fwd->feat && grad_out->rgb && grad_out->depth &&
                   grad_out->alpha && grad_rec && scene->feat,
               GS_INVALID_ARG, "gs_joint_backward: NULL pointer");
    GS_REQUIRE(((uintptr_t)scene->feat & 15) == 0, GS_INVALID_ARG, "gs_joint_backward: features must be 16-byte aligned");
    if (T <= 0) return GS_OK;
    cudaStream_t s = (cudaStream_t)stream;
#define GS_JCASE(d)                                                                                                  \
    case d:                                                                                                          \
        radiance_backward_kernel<d><<<(unsigned)T, 256, 0, s>>>(                                                     \
            views_dev, n_views, proj->rec, bins->sorted_rec, bins->ranges, *params, fwd->rgb, fwd->depth, fwd->alpha, \
            grad_out->rgb, grad_out->depth, grad_out->alpha, grad_rec, proj->status, scene->feat, fwd->feat,          \
            grad_out->feat);                                                                                         \
        return check_launch("radiance_backward_kernel");
    switch (scene->feat_dim) {
        GS_JCASE(8) GS_JCASE(16) GS_JCASE(24) GS_JCASE(32) GS_JCASE(48) GS_JCASE(64)
        default:
            gs::set_error("gs_joint_backward: feat_dim = %d (need 8, 16, 24, 32, 48 or 64)", scene->feat_dim);
            return GS_UNSUPPORTED;
    }
#undef GS_JCASE
}

#ifdef GS_RASTER_STATS
extern "C" void gs_debug_raster_stats(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, gs::g_raster_stats, sizeof(unsigned long long) * 4);
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(gs::g_raster_stats, z, sizeof(z));
}
#endif
