// gs_rasterize.cu -- O12: per pixel front-to-back alpha
// compositing of colour, depth (sum w z), opacity (1 - T) and an optional
// D-channel feature.  P:136 "Color attributes c are rasterized ... using alpha
// blending, while feature attributes f are rendered ... through identical
// rasterization"; "render dense feature and depth maps"; S:157;
// readings Q4, Q11, Q14-Q18.
//
// Design (B200, SIMT -- not a dense contraction, no tensor cores):
//   * one 256-thread CTA per 16x16 tile; each warp owns an 8x4 sub-tile;
//   * the tile's sorted list is staged through shared memory in chunks of 64
//     records (+ their feature rows) with cp.async (LDGSTS) bulk copies;
//   * warp-level culling: the 32 lanes test 32 list entries at once against
//     the warp's 8x4 sub-tile using the bounding box of each Gaussian's
//     alpha >= 1/255 ellipse (conservative, so it never drops a Gaussian the
//     oracle would blend -- Q11); a ballot gives the entries the warp walks;
//   * warp-ballot early termination: a warp stops when all 32 pixels have
//     hit T < t_min; the CTA stops when all warps have.
// The per-pixel arithmetic that decides a skip / stop (power, alpha, Tn) is
// written with explicit _rn intrinsics in the oracle's operation order.
#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int RT_THREADS = 256;
constexpr int CH = 64;  // list entries staged per chunk

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int D>
struct SmemT {
    float4 rec[CH][4];               // full 64-byte records
    float feat[D > 0 ? CH : 1][D > 0 ? D : 1];
    int view;
};

template <int D>
__global__ void __launch_bounds__(RT_THREADS)
rasterize_kernel(const gs_view* __restrict__ views, int n_views, const gs_record* __restrict__ rec,
                 const uint32_t* __restrict__ sorted_rec, const uint32_t* __restrict__ ranges,
                 const float* __restrict__ feat, gs_params P, float* __restrict__ out_rgb,
                 float* __restrict__ out_depth, float* __restrict__ out_alpha, float* __restrict__ out_feat,
                 const uint32_t* __restrict__ status) {
    if (*status) return;
    __shared__ __align__(16) SmemT<D> sm;
    const uint32_t tile = blockIdx.x;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) sm.view = find_view_by_tile(views, n_views, tile);
    __syncthreads();
    const gs_view& V = views[sm.view];
    const int W = V.width, H = V.height;
    const int TX = (W + GS_TILE - 1) / GS_TILE;
    const uint32_t lt = tile - V.tile_offset;
    const int tx = (int)(lt % (uint32_t)TX), ty = (int)(lt / (uint32_t)TX);
    const int sx = tx * 16 + (int)(warp & 1u) * 8, sy = ty * 16 + (int)(warp >> 1) * 4;
    const int px = sx + (int)(lane & 7u), py = sy + (int)(lane >> 3);
    const bool inside = px < W && py < H;
    const float pxf = (float)px, pyf = (float)py;
    const float sx0 = (float)sx, sx1 = (float)(sx + 7), sy0 = (float)sy, sy1 = (float)(sy + 3);

    const uint32_t rs = ranges[2 * tile], re = ranges[2 * tile + 1];
    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Dz = 0.f;
    float F[D > 0 ? D : 1];
#pragma unroll
    for (int c = 0; c < (D > 0 ? D : 1); ++c) F[c] = 0.f;
    bool done = !inside;

    for (uint32_t c0 = rs; c0 < re; c0 += CH) {
        const int cnt = (int)min((uint32_t)CH, re - c0);
        // ---- stage records (and feature rows) of this chunk ----
        {
            const int j = threadIdx.x >> 2, piece = threadIdx.x & 3;
            if (j < cnt) {
                const uint32_t slot = __ldg(&sorted_rec[c0 + j]);
                cp_async16(&sm.rec[j][piece], reinterpret_cast<const float4*>(rec + slot) + piece);
                if (D > 0) {
                    const uint32_t gid = __ldg(&rec[slot].gid);
                    const float4* src = reinterpret_cast<const float4*>(feat + (int64_t)gid * D);
                    for (int q = piece; q < D / 4; q += 4) cp_async16(&sm.feat[j][q * 4], src + q);
                }
            }
            cp_async_wait_all();
            __syncthreads();
        }
        // ---- walk the chunk (warp-uniform) ----
        if (!__all_sync(0xffffffffu, done)) {
            for (int base = 0; base < cnt; base += 32) {
                const int j = base + (int)lane;
                bool hit = false;
                if (j < cnt) {
                    const float4 a = sm.rec[j][0], b = sm.rec[j][1];
                    hit = a.x + b.z >= sx0 && a.x - b.z <= sx1 && a.y + b.w >= sy0 && a.y - b.w <= sy1;
                }
                uint32_t m = __ballot_sync(0xffffffffu, hit);
                while (m) {
                    const int k = base + __ffs(m) - 1;
                    m &= m - 1u;
                    if (done) continue;
                    const float4 a = sm.rec[k][0];   // u, v, ca, cb
                    const float4 b = sm.rec[k][1];   // cc, o, ex, ey
                    const float dx = __fsub_rn(a.x, pxf), dy = __fsub_rn(a.y, pyf);
                    const float t1 = __fmul_rn(__fmul_rn(a.z, dx), dx);
                    const float t2 = __fmul_rn(__fmul_rn(b.x, dy), dy);
                    const float t3 = __fmul_rn(__fmul_rn(a.w, dx), dy);
                    const float power = __fsub_rn(__fmul_rn(-0.5f, __fadd_rn(t1, t2)), t3);
                    if (power > 0.0f) continue;
                    const float alpha = fminf(P.alpha_max, __fmul_rn(b.y, __expf(power)));
                    if (alpha < P.alpha_min) continue;
                    const float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                    if (Tn < P.t_min) { done = true; continue; }
                    const float w = __fmul_rn(alpha, T);
                    const float4 c = sm.rec[k][2];   // r, g, b, z
                    C0 += w * c.x; C1 += w * c.y; C2 += w * c.z; Dz += w * c.w;
                    if (D > 0) {
#pragma unroll
                        for (int q = 0; q < D; q += 4) {
                            const float4 f = *reinterpret_cast<const float4*>(&sm.feat[k][q]);
                            F[q] += w * f.x; F[q + 1] += w * f.y; F[q + 2] += w * f.z; F[q + 3] += w * f.w;
                        }
                    }
                    T = Tn;
                }
                if (__all_sync(0xffffffffu, done)) break;
            }
        }
        const int active = __syncthreads_count(!done);
        if (active == 0) break;
    }
    if (inside) {
        const int64_t HW = (int64_t)W * H;
        const int64_t pix = V.pix_offset + (int64_t)py * W + px;
        const int64_t loc = (int64_t)py * W + px;
        out_rgb[3 * V.pix_offset + loc] = C0;
        out_rgb[3 * V.pix_offset + HW + loc] = C1;
        out_rgb[3 * V.pix_offset + 2 * HW + loc] = C2;
        out_depth[pix] = Dz;
        out_alpha[pix] = 1.0f - T;
        if (D > 0) {
#pragma unroll
            for (int c = 0; c < D; ++c) out_feat[(int64_t)D * V.pix_offset + (int64_t)c * HW + loc] = F[c];
        }
    }
}

template <int D>
gs_status launch(const gs_scene* scene, const gs_projected* proj, const gs_bins* bins, const gs_view* views_dev,
                 int n_views, int64_t T, const gs_params* P, gs_images* out, cudaStream_t s) {
    rasterize_kernel<D><<<(unsigned)T, RT_THREADS, 0, s>>>(views_dev, n_views, proj->rec, bins->sorted_rec,
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
