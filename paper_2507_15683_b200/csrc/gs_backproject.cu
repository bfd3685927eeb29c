// gs_backproject.cu -- O13: rendered depth -> world points.
// P:278 "we fully leverage the depth information from Gaussian rendering for
// 3D constraints ... 2D-3D PnP algorithm with RANSAC"; S:492 back-project each
// matched rendered pixel via rendered depth; "matches with accum_alpha
// < 0.5 at that pixel are discarded"; readings Q16, Q24.
//
// A streaming HBM-bound pass: per pixel read depth + alpha (8 B), write xyz
// (12 B) + valid (1 B).  One thread per 4 consecutive pixels of a row-major
// view (float4 loads / stores when aligned), views on grid.y.
#include <cuda_fp16.h>

#include "gs_common.cuh"

namespace gs {
namespace {

__global__ void __launch_bounds__(256)
backproject_kernel(const gs_view* __restrict__ views, const float* __restrict__ depth,
                   const float* __restrict__ alpha, float a_min, float* __restrict__ xyz,
                   uint8_t* __restrict__ valid) {
    const gs_view V = views[blockIdx.y];
    const int64_t HW = (int64_t)V.width * V.height;
    const int64_t base = V.pix_offset;
    const float* dz = depth + base;
    const float* al = alpha + base;
    float* ox = xyz + 3 * base;
    uint8_t* ov = valid + base;
    const bool vec = ((base & 3) == 0) && ((HW & 3) == 0);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 4 < HW; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p0 = q * 4;
        if (vec) {
            const float4 d4 = __ldcs(reinterpret_cast<const float4*>(dz + p0));
            const float4 a4 = __ldcs(reinterpret_cast<const float4*>(al + p0));
            float X[4], Y[4], Z[4];
            uint8_t ok[4];
            const float dd[4] = {d4.x, d4.y, d4.z, d4.w}, aa[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t p = p0 + k;
                bp_pixel(V, dd[k], aa[k], a_min, (int)(p % V.width), (int)(p / V.width), X[k], Y[k], Z[k], ok[k]);
            }
            __stcs(reinterpret_cast<float4*>(ox + p0), make_float4(X[0], X[1], X[2], X[3]));
            __stcs(reinterpret_cast<float4*>(ox + HW + p0), make_float4(Y[0], Y[1], Y[2], Y[3]));
            __stcs(reinterpret_cast<float4*>(ox + 2 * HW + p0), make_float4(Z[0], Z[1], Z[2], Z[3]));
            const uint32_t packed = (uint32_t)ok[0] | ((uint32_t)ok[1] << 8) | ((uint32_t)ok[2] << 16) |
                                    ((uint32_t)ok[3] << 24);
            *reinterpret_cast<uint32_t*>(ov + p0) = packed;
        } else {
            for (int k = 0; k < 4 && p0 + k < HW; ++k) {
                const int64_t p = p0 + k;
                float X, Y, Z;
                uint8_t ok;
                bp_pixel(V, dz[p], al[p], a_min, (int)(p % V.width), (int)(p / V.width), X, Y, Z, ok);
                ox[p] = X; ox[HW + p] = Y; ox[2 * HW + p] = Z;
                ov[p] = ok;
            }
        }
    }
}

// gs_pack_images (GS_PACK_COMPACT): per view, at byte 12 * pix_offset, fp16 R, G, B and
// A planes (hw halves each) then the fp32 sum-w-z plane (hw floats).  Two pixels per
// thread (half2 stores) when the view's planes are even-sized and aligned.
__global__ void __launch_bounds__(256)
pack_compact_kernel(const gs_view* __restrict__ views, const float* __restrict__ rgb, const float* __restrict__ depth,
                    const float* __restrict__ alpha, unsigned char* __restrict__ out) {
    const gs_view V = views[blockIdx.y];
    const int64_t HW = (int64_t)V.width * V.height;
    const int64_t po = V.pix_offset;
    const float* r = rgb + 3 * po;
    const float* al = alpha + po;
    const float* dz = depth + po;
    __half* oh = reinterpret_cast<__half*>(out + 12 * po);   // 4 half planes
    float* od = reinterpret_cast<float*>(out + 12 * po + 8 * HW);
    const bool vec = ((po & 1) == 0) && ((HW & 1) == 0);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 2 < HW; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = 2 * q;
        if (vec) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float2 v = __ldcs(reinterpret_cast<const float2*>(r + c * HW + p));
                __stcs(reinterpret_cast<__half2*>(oh + c * HW + p), __floats2half2_rn(v.x, v.y));
            }
            const float2 a = __ldcs(reinterpret_cast<const float2*>(al + p));
            __stcs(reinterpret_cast<__half2*>(oh + 3 * HW + p), __floats2half2_rn(a.x, a.y));
            __stcs(reinterpret_cast<float2*>(od + p), __ldcs(reinterpret_cast<const float2*>(dz + p)));
        } else {
            for (int64_t k = p; k < p + 2 && k < HW; ++k) {
                for (int c = 0; c < 3; ++c) oh[c * HW + k] = __float2half_rn(r[c * HW + k]);
                oh[3 * HW + k] = __float2half_rn(al[k]);
                od[k] = dz[k];
            }
        }
    }
}

// GS_PACK_DENSE11 (reading Q39): batch-planar R, G, B (fp16), A (unorm16, round(65535 A)),
// then sum(w z) as the upper 24 bits of its fp32 pattern (rounded; 3 bytes, little-endian).
__device__ __forceinline__ uint32_t depth24(float z) { return (__float_as_uint(z) + 0x80u) >> 8; }
__device__ __forceinline__ uint16_t unorm16(float a) { return (uint16_t)__float2uint_rn(fminf(fmaxf(a, 0.f), 1.f) * 65535.f); }

__global__ void __launch_bounds__(256)
pack_dense11_kernel(const gs_view* __restrict__ views, int64_t total_pixels, const float* __restrict__ rgb,
                    const float* __restrict__ depth, const float* __restrict__ alpha, unsigned char* __restrict__ out) {
    const gs_view V = views[blockIdx.y];
    const int64_t HW = (int64_t)V.width * V.height;
    const int64_t po = V.pix_offset, TP = total_pixels;
    const float* r = rgb + 3 * po;
    __half* oh = reinterpret_cast<__half*>(out);                  // R, G, B planes of TP halves
    uint16_t* oa = reinterpret_cast<uint16_t*>(out + 6 * TP);     // A plane
    unsigned char* od = out + 8 * TP;                             // depth, 3 bytes per pixel
    const bool vec = ((po & 3) == 0) && ((HW & 3) == 0) && ((TP & 3) == 0);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q * 4 < HW; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = 4 * q;
        if (vec) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(r + c * HW + p));
                __half2 h[2] = {__floats2half2_rn(v.x, v.y), __floats2half2_rn(v.z, v.w)};
                __stcs(reinterpret_cast<uint2*>(oh + c * TP + po + p), *reinterpret_cast<const uint2*>(h));
            }
            const float4 a = __ldcs(reinterpret_cast<const float4*>(alpha + po + p));
            const uint2 av = make_uint2((uint32_t)unorm16(a.x) | ((uint32_t)unorm16(a.y) << 16),
                                        (uint32_t)unorm16(a.z) | ((uint32_t)unorm16(a.w) << 16));
            __stcs(reinterpret_cast<uint2*>(oa + po + p), av);
            const float4 z = __ldcs(reinterpret_cast<const float4*>(depth + po + p));
            const uint32_t d0 = depth24(z.x), d1 = depth24(z.y), d2 = depth24(z.z), d3 = depth24(z.w);
            // 4 x 24 bits -> 3 little-endian words
            const uint3 w = make_uint3(d0 | (d1 << 24), (d1 >> 8) | (d2 << 16), (d2 >> 16) | (d3 << 8));
            uint32_t* o32 = reinterpret_cast<uint32_t*>(od + 3 * (po + p));
            __stcs(o32, w.x); __stcs(o32 + 1, w.y); __stcs(o32 + 2, w.z);
        } else {
            for (int64_t k = p; k < p + 4 && k < HW; ++k) {
                for (int c = 0; c < 3; ++c) oh[c * TP + po + k] = __float2half_rn(r[c * HW + k]);
                oa[po + k] = unorm16(alpha[po + k]);
                const uint32_t d = depth24(depth[po + k]);
                unsigned char* b = od + 3 * (po + k);
                b[0] = (unsigned char)d; b[1] = (unsigned char)(d >> 8); b[2] = (unsigned char)(d >> 16);
            }
        }
    }
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" size_t gs_pack_bytes(int64_t total_pixels, int32_t format) {
    if (total_pixels <= 0) return 0;
    return format == GS_PACK_COMPACT ? (size_t)(12 * total_pixels)
         : format == GS_PACK_DENSE11 ? (size_t)(11 * total_pixels) : 0;
}

extern "C" gs_status gs_pack_images(const gs_images* in, const gs_view* views_host, const gs_view* views_dev,
                                    int32_t n_views, int32_t format, void* out, void* stream) {
    int64_t total_pixels = 0, T = 0;
    gs_status st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(format == GS_PACK_COMPACT || format == GS_PACK_DENSE11, GS_UNSUPPORTED,
               "gs_pack_images: unknown format %d", format);
    GS_REQUIRE(in && in->rgb && in->depth && in->alpha && out, GS_INVALID_ARG, "gs_pack_images: NULL pointer");
    GS_REQUIRE(((uintptr_t)out & 15) == 0 && ((uintptr_t)in->rgb & 7) == 0 && ((uintptr_t)in->depth & 7) == 0 &&
                   ((uintptr_t)in->alpha & 7) == 0,
               GS_INVALID_ARG, "gs_pack_images: out must be 16-byte and the planes 8-byte aligned");
    int64_t maxhw = 0;
    for (int i = 0; i < n_views; ++i) maxhw = std::max<int64_t>(maxhw, (int64_t)views_host[i].width * views_host[i].height);
    const int64_t pairs = (maxhw + 1) / 2;
    const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((pairs + 255) / 256, (int64_t)num_sms() * 8 / n_views + 1));
    if (format == GS_PACK_DENSE11) {
        GS_REQUIRE(((uintptr_t)in->rgb & 15) == 0 && ((uintptr_t)in->depth & 15) == 0 && ((uintptr_t)in->alpha & 15) == 0,
                   GS_INVALID_ARG, "gs_pack_images: GS_PACK_DENSE11 needs 16-byte aligned planes");
        pack_dense11_kernel<<<dim3((unsigned)gx, (unsigned)n_views), 256, 0, (cudaStream_t)stream>>>(
            views_dev, total_pixels, in->rgb, in->depth, in->alpha, static_cast<unsigned char*>(out));
        return check_launch("pack_dense11_kernel");
    }
    pack_compact_kernel<<<dim3((unsigned)gx, (unsigned)n_views), 256, 0, (cudaStream_t)stream>>>(
        views_dev, in->rgb, in->depth, in->alpha, static_cast<unsigned char*>(out));
    return check_launch("pack_compact_kernel");
}

extern "C" gs_status gs_backproject(const gs_images* in, const gs_view* views_host, const gs_view* views_dev,
                                    int32_t n_views, float a_min, float* xyz, uint8_t* valid, void* stream) {
    int64_t total_pixels = 0, T = 0;
    gs_status st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(in && in->depth && in->alpha, GS_INVALID_ARG, "images depth/alpha is NULL");
    GS_REQUIRE(xyz && valid, GS_INVALID_ARG, "xyz/valid is NULL");
    GS_REQUIRE(a_min == a_min, GS_INVALID_ARG, "a_min is NaN");
    GS_REQUIRE(((uintptr_t)xyz & 15) == 0 && ((uintptr_t)in->depth & 15) == 0 && ((uintptr_t)in->alpha & 15) == 0 &&
                   ((uintptr_t)valid & 3) == 0,
               GS_INVALID_ARG, "xyz/depth/alpha must be 16-byte and valid 4-byte aligned");
    int64_t maxhw = 0;
    for (int i = 0; i < n_views; ++i) maxhw = std::max<int64_t>(maxhw, (int64_t)views_host[i].width * views_host[i].height);
    const int64_t quads = (maxhw + 3) / 4;
    int64_t gx = (quads + 255) / 256;
    const int64_t target = std::max<int64_t>(1, (int64_t)num_sms() * 8 / n_views);
    gx = std::min(gx, std::max<int64_t>(target, 1));
    dim3 grid((unsigned)std::max<int64_t>(gx, 1), (unsigned)n_views);
    backproject_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(views_dev, in->depth, in->alpha, a_min, xyz, valid);
    return check_launch("backproject_kernel");
}
