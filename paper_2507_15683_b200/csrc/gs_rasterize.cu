// gs_rasterize.cu -- O12: per pixel front-to-back alpha
// compositing of colour, depth (sum w z), opacity (1 - T) and an optional
// D-channel feature.  P:136 "Color attributes c are rasterized ... using alpha
// blending, while feature attributes f are rendered ... through identical
// rasterization"; "render dense feature and depth maps"; S:157;
// readings Q4, Q11, Q14-Q18.
//
// Design (B200):
//   * one CTA per 16x16 tile = 8 consumer warps (one 8x4 sub-tile each) + 1
//     producer warp;
//   * the producer streams the tile's sorted list through a 4-stage
//     shared-memory ring with TMA bulk copies (cp.async.bulk, one 64-B record
//     and one D*4-B feature row per entry) completing on mbarriers; consumers
//     release stages through "empty" mbarriers -- no CTA-wide barrier in the
//     loop;
//   * exact warp-level culling: each lane tests one staged entry: does the
//     entry's alpha >= alpha_min ellipse (q <= q_cut, inflated) touch the warp's
//     8x4 pixel rectangle?  A ballot gives the entries the warp walks
//     (conservative, so it never drops a Gaussian the oracle blends -- Q11);
//   * per pixel the skip / stop decisions (power, alpha, Tn) are evaluated with
//     explicit _rn intrinsics in the oracle's operation order;
//   * the feature blend F[px][:] += w[px][k] f[k][:] -- the one dense
//     contraction of the path -- runs on the tensor cores: each warp compacts
//     the weights of its walked entries into an 8-entry shared buffer and
//     issues m16n8k8 TF32 MMAs (weights split hi+lo, features rounded once:
//     error <= 2^-11 sum w|f|, inside the 1e-3 max(1,|f|) tolerance);
//   * warp-ballot early termination once all 32 pixels have T < t_min.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int NCW = 8;                 // consumer warps
constexpr int RT_THREADS = (NCW + 1) * 32;
constexpr int SE = 64;                 // entries per stage
constexpr int NST = 4;                 // ring stages
constexpr int WB_STRIDE = 40;          // weight-buffer row stride (conflict-free A fragments)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int D>
struct RasterSmem {
    static constexpr int FS = D > 0 ? D + 8 : 1;   // feature row stride (floats)
    float4 rec[NST][SE][4];                        // 64-byte records
    float feat[D > 0 ? NST : 1][D > 0 ? SE : 1][FS];
    float wbuf[D > 0 ? NCW : 1][8][WB_STRIDE];     // per-warp compacted weights [k][pixel]
    int ent[NCW][8];                               // per-warp compacted entry index
    uint64_t full[NST];
    uint64_t empty[NST];
    int view;
};

// min over the 8x4 pixel-centre rectangle [x0,x1]x[y0,y1] of
// q(d) = ca dx^2 + 2 cb dx dy + cc dy^2 (d = p - mean), compared with q_cut.
__device__ __forceinline__ bool ellipse_hits_rect(float u, float v, float ca, float cb, float cc, float qcut,
                                                  float x0, float x1, float y0, float y1) {
    const bool inx = u >= x0 && u <= x1, iny = v >= y0 && v <= y1;
    if (inx && iny) return true;
    float qmin = 3.4e38f;
    if (!inx) {               // facing vertical edge
        const float dx = (u < x0 ? x0 : x1) - u;
        const float dy = fminf(fmaxf(-cb * dx * __frcp_rn(cc), y0 - v), y1 - v);
        qmin = fminf(qmin, ca * dx * dx + 2.f * cb * dx * dy + cc * dy * dy);
    }
    if (!iny) {               // facing horizontal edge
        const float dy = (v < y0 ? y0 : y1) - v;
        const float dx = fminf(fmaxf(-cb * dy * __frcp_rn(ca), x0 - u), x1 - u);
        qmin = fminf(qmin, ca * dx * dx + 2.f * cb * dx * dy + cc * dy * dy);
    }
    return qmin <= qcut;
}

template <int D>
__global__ void __launch_bounds__(RT_THREADS, (D > 32 ? 1 : 2))
rasterize_kernel(const gs_view* __restrict__ views, int n_views, const gs_record* __restrict__ rec,
                 const uint32_t* __restrict__ sorted_rec, const uint32_t* __restrict__ ranges,
                 const float* __restrict__ feat, gs_params P, float* __restrict__ out_rgb,
                 float* __restrict__ out_depth, float* __restrict__ out_alpha, float* __restrict__ out_feat,
                 const uint32_t* __restrict__ status) {
    if (*status) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    RasterSmem<D>& sm = *reinterpret_cast<RasterSmem<D>*>(smem_raw);
    const uint32_t tile = blockIdx.x;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        sm.view = find_view_by_tile(views, n_views, tile);
        for (int s = 0; s < NST; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const uint32_t rs = __ldg(&ranges[2 * tile]), re = __ldg(&ranges[2 * tile + 1]);
    const uint32_t L = re - rs;
    const int nstage = (int)((L + SE - 1) / SE);

    if (warp == NCW) {
        // ------------------------------------------------------------ producer
        for (int s = 0; s < nstage; ++s) {
            const int buf = s % NST;
            if (s >= NST) mbar_wait(&sm.empty[buf], ((s / NST) & 1) ^ 1);
            const uint32_t c0 = rs + (uint32_t)s * SE;
            const int cnt = (int)min((uint32_t)SE, re - c0);
            if (lane == 0) mbar_arrive_expect_tx(&sm.full[buf], (uint32_t)cnt * (64u + 4u * D));
            __syncwarp();
            for (int j = (int)lane; j < cnt; j += 32) {
                const uint32_t slot = __ldg(&sorted_rec[c0 + j]);
                bulk_g2s(&sm.rec[buf][j][0], rec + slot, 64u, &sm.full[buf]);
                if (D > 0) {
                    const uint32_t gid = __ldg(&rec[slot].gid);
                    bulk_g2s(&sm.feat[buf][j][0], feat + (int64_t)gid * D, 4u * D, &sm.full[buf]);
                }
            }
        }
        // drain: the CTA must not retire while bulk copies into its smem are in flight
        for (int s = (nstage > NST ? nstage - NST : 0); s < nstage; ++s)
            mbar_wait(&sm.full[s % NST], (s / NST) & 1);
        return;
    }

    // ---------------------------------------------------------------- consumers
    const gs_view& V = views[sm.view];
    const int W = V.width, H = V.height;
    const int TX = (W + GS_TILE - 1) / GS_TILE;
    const uint32_t lt = tile - V.tile_offset;
    const int tx = (int)(lt % (uint32_t)TX), ty = (int)(lt / (uint32_t)TX);
    const int sx = tx * 16 + (int)(warp & 1u) * 8, sy = ty * 16 + (int)(warp >> 1) * 4;
    const int px = sx + (int)(lane & 7u), py = sy + (int)(lane >> 3);
    const bool inside = px < W && py < H;
    const float pxf = (float)px, pyf = (float)py;
    const float rx0 = (float)sx, rx1 = (float)(sx + 7), ry0 = (float)sy, ry1 = (float)(sy + 3);

    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Dz = 0.f;
    bool done = !inside;
    bool warp_done = __all_sync(0xffffffffu, done);
    constexpr int NT = D > 0 ? D / 8 : 1;   // n-tiles of 8 features (D % 8 == 4 handled by a padded tile)
    constexpr int NTP = D > 0 ? (D + 7) / 8 : 1;
    float acc[2][NTP][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < NTP; ++n) acc[m][n][0] = acc[m][n][1] = acc[m][n][2] = acc[m][n][3] = 0.f;
    (void)NT;
    int nc = 0;   // compacted weights pending in this warp's buffer
    const int g = (int)(lane >> 2), t4 = (int)(lane & 3u);

    auto mma_flush = [&](int buf) {
        if constexpr (D > 0) {
            // pad rows nc..7 with zero weights, point them at a valid entry
            for (int k = nc; k < 8; ++k) {
                sm.wbuf[warp][k][lane] = 0.f;
                if (lane == 0) sm.ent[warp][k] = sm.ent[warp][0];
            }
            __syncwarp();
            uint32_t ahi[2][4], alo[2][4];
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const float a0 = sm.wbuf[warp][t4][m * 16 + g], a1 = sm.wbuf[warp][t4][m * 16 + g + 8];
                const float a2 = sm.wbuf[warp][t4 + 4][m * 16 + g], a3 = sm.wbuf[warp][t4 + 4][m * 16 + g + 8];
                const float av[4] = {a0, a1, a2, a3};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    ahi[m][i] = to_tf32(av[i]);
                    alo[m][i] = to_tf32(av[i] - __uint_as_float(ahi[m][i]));
                }
            }
            const int e0 = sm.ent[warp][t4], e1 = sm.ent[warp][t4 + 4];
            const float* f0 = &sm.feat[buf][e0][0];
            const float* f1 = &sm.feat[buf][e1][0];
#pragma unroll
            for (int n = 0; n < NTP; ++n) {
                const int ch = n * 8 + g;
                const uint32_t b0 = to_tf32(ch < D ? f0[ch] : 0.f), b1 = to_tf32(ch < D ? f1[ch] : 0.f);
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    mma_tf32(acc[m][n], ahi[m], b0, b1);
                    mma_tf32(acc[m][n], alo[m], b0, b1);
                }
            }
            __syncwarp();
            nc = 0;
        }
    };

    for (int s = 0; s < nstage; ++s) {
        const int buf = s % NST;
        mbar_wait(&sm.full[buf], (s / NST) & 1);
        if (!warp_done) {
            const int cnt = (int)min((uint32_t)SE, re - (rs + (uint32_t)s * SE));
#pragma unroll 1
            for (int half = 0; half < SE / 32; ++half) {
                const int j = half * 32 + (int)lane;
                bool hit = false;
                if (j < cnt) {
                    const float4 a = sm.rec[buf][j][0];   // u, v, ca, cb
                    const float4 b = sm.rec[buf][j][1];   // cc, o, q_cut, -
                    hit = ellipse_hits_rect(a.x, a.y, a.z, a.w, b.x, b.z, rx0, rx1, ry0, ry1);
                }
                uint32_t msk = __ballot_sync(0xffffffffu, hit);
                while (msk) {
                    const int k = half * 32 + __ffs(msk) - 1;
                    msk &= msk - 1u;
                    float wgt = 0.f;
                    if (!done) {
                        const float4 a = sm.rec[buf][k][0];
                        const float4 b = sm.rec[buf][k][1];
                        const float dx = __fsub_rn(a.x, pxf), dy = __fsub_rn(a.y, pyf);
                        const float t1 = __fmul_rn(__fmul_rn(a.z, dx), dx);
                        const float t2 = __fmul_rn(__fmul_rn(b.x, dy), dy);
                        const float t3 = __fmul_rn(__fmul_rn(a.w, dx), dy);
                        const float power = __fsub_rn(__fmul_rn(-0.5f, __fadd_rn(t1, t2)), t3);
                        if (!(power > 0.0f)) {          // oracle: skip iff power > 0
                            const float alpha = fminf(P.alpha_max, __fmul_rn(b.y, __expf(power)));
                            if (!(alpha < P.alpha_min)) {   // oracle: skip iff alpha < alpha_min
                                const float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                                if (Tn < P.t_min) {
                                    done = true;
                                } else {
                                    wgt = __fmul_rn(alpha, T);
                                    const float4 c = sm.rec[buf][k][2];   // r, g, b, z
                                    C0 = fmaf(wgt, c.x, C0);
                                    C1 = fmaf(wgt, c.y, C1);
                                    C2 = fmaf(wgt, c.z, C2);
                                    Dz = fmaf(wgt, c.w, Dz);
                                    T = Tn;
                                }
                            }
                        }
                    }
                    if constexpr (D > 0) {
                        sm.wbuf[warp][nc][lane] = wgt;
                        if (lane == 0) sm.ent[warp][nc] = k;
                        if (++nc == 8) {
                            __syncwarp();
                            mma_flush(buf);
                        }
                    }
                }
                warp_done = __all_sync(0xffffffffu, done);
                if (warp_done) break;
            }
            if (D > 0 && nc > 0) {
                __syncwarp();
                mma_flush(buf);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[buf]);
    }

    // ---------------------------------------------------------------- outputs
    const int64_t HW = (int64_t)W * H;
    if (inside) {
        const int64_t loc = (int64_t)py * W + px;
        out_rgb[3 * V.pix_offset + loc] = C0;
        out_rgb[3 * V.pix_offset + HW + loc] = C1;
        out_rgb[3 * V.pix_offset + 2 * HW + loc] = C2;
        out_depth[V.pix_offset + loc] = Dz;
        out_alpha[V.pix_offset + loc] = 1.0f - T;
    }
    if (D > 0) {
        // accumulator (m, n, i): pixel p = 16 m + g + 8 (i >> 1) -> (sx + g, sy + 2 m + (i >> 1)),
        // channel n*8 + 2 t4 + (i & 1)
        float* fo = out_feat + (int64_t)D * V.pix_offset;
        const int fx = sx + g;
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int fy = sy + 2 * m + (i >> 1);
                if (fx < W && fy < H) {
                    const int64_t loc = (int64_t)fy * W + fx;
#pragma unroll
                    for (int n = 0; n < NTP; ++n) {
                        const int ch = n * 8 + 2 * t4 + (i & 1);
                        if (ch < D) fo[(int64_t)ch * HW + loc] = acc[m][n][i];
                    }
                }
            }
    }
}

template <int D>
gs_status launch(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins, const gs_view* views_dev,
                 int n_views, int64_t T, const gs_params* P, gs_images* out, cudaStream_t s) {
    const int smem = (int)sizeof(RasterSmem<D>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(rasterize_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    rasterize_kernel<D><<<(unsigned)T, RT_THREADS, smem, s>>>(views_dev, n_views, proj->rec, bins->sorted_rec,
                                                              bins->ranges, scene->feat, *P, out->rgb, out->depth,
                                                              out->alpha, out->feat, proj->status);
    return check_launch("rasterize_kernel");
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" gs_status gs_rasterize(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins,
                                  const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                                  const gs_params* params, gs_images* out, void* stream) {
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
    switch (scene->feat_dim) {
#define GS_CASE(d) \
    case d: return launch<d>(scene, proj, bins, views_dev, n_views, T, params, out, s);
        GS_CASE(0) GS_CASE(4) GS_CASE(8) GS_CASE(12) GS_CASE(16) GS_CASE(20) GS_CASE(24) GS_CASE(28) GS_CASE(32)
        GS_CASE(36) GS_CASE(40) GS_CASE(44) GS_CASE(48) GS_CASE(52) GS_CASE(56) GS_CASE(60) GS_CASE(64)
#undef GS_CASE
        default:
            gs::set_error("feat_dim = %d unsupported", scene->feat_dim);
            return GS_UNSUPPORTED;
    }
}
