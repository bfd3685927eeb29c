// gs_common.cuh -- internal helpers of libgs (CUDA side only; not shared with
// the oracle).  Error reporting for the C ABI and small device utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdarg>

#include "../../include/gs.h"

namespace gs {

// Device-side bounds checks (substitute for compute-sanitizer, which the GPU pool
// disables): built with -DGS_CHECKS they trap with the failing condition; compiled out
// otherwise.  tools/build_checks.sh builds the checked library.
#ifdef GS_CHECKS
#define GS_DCHECK(c)                                                                       \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("GS_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,  \
                   (int)blockIdx.x, (int)threadIdx.x, #c);                                 \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define GS_DCHECK(c) \
    do {             \
    } while (0)
#endif

// thread-local last-error message (gs_api.cu)
void set_error(const char* fmt, ...);

#define GS_REQUIRE(cond, code, ...)          \
    do {                                     \
        if (!(cond)) {                       \
            ::gs::set_error(__VA_ARGS__);    \
            return (code);                   \
        }                                    \
    } while (0)

inline gs_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return GS_CUDA_ERROR;
    }
    return GS_OK;
}

inline int tiles_x(const gs_view& v) { return (v.width + GS_TILE - 1) / GS_TILE; }
inline int tiles_y(const gs_view& v) { return (v.height + GS_TILE - 1) / GS_TILE; }

// host-side validation of a view batch (offsets must be the contiguous layout)
gs_status validate_views(const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                         int64_t* total_pixels, int64_t* total_tiles);
gs_status validate_scene(const gs_scene* s, bool need_geometry);

// Per-device caches (a process may drive several GPUs; kernel attributes and
// occupancy are per device): index = the current device, atomic so concurrent
// host threads never race.
constexpr int GS_MAX_DEVICES = 64;
inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
inline int num_sms() {
    static std::atomic<int> cache[GS_MAX_DEVICES];
    const int dev = current_device();
    int v = (dev >= 0 && dev < GS_MAX_DEVICES) ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (v <= 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        if (dev >= 0 && dev < GS_MAX_DEVICES) cache[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// ---------------------------------------------------------------- device side
// Reading Q30 (N3 tight binning): does the alpha >= alpha_min ellipse p(d) >=
// e_cut reach the pixel centres [16tx, 16tx+15] x [16ty, 16ty+15]?  p is
// concave: with the mean outside the rectangle its maximum lies on a facing
// edge at the clamped 1-D stationary point.  IEEE fp32 in the oracle's exact
// order (explicit _rn intrinsics: no contraction), so key lists are bit-exact.
__device__ __forceinline__ float p_at(float ea, float eb, float ec, float dx, float dy) {
    return __fadd_rn(__fadd_rn(__fmul_rn(__fmul_rn(ea, dx), dx), __fmul_rn(__fmul_rn(eb, dx), dy)),
                     __fmul_rn(__fmul_rn(ec, dy), dy));
}
struct TightRec {
    float u, v, ea, eb, ec, ecut, sx, sy;
};
__device__ __forceinline__ TightRec tight_make(float u, float v, float ea, float eb, float ec, float ecut) {
    // stationary-point slopes, one rounded division each (the oracle's sx, sy)
    const float sy = __fdiv_rn(-eb, __fmul_rn(2.0f, ec)), sx = __fdiv_rn(-eb, __fmul_rn(2.0f, ea));
    return TightRec{u, v, ea, eb, ec, ecut, sx, sy};
}
__device__ __forceinline__ TightRec tight_of(const gs_record* r) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(r));       // u, v, ea, eb
    const float4 b = __ldg(reinterpret_cast<const float4*>(r) + 1);   // ec, o, e_cut, tile_mask
    return tight_make(a.x, a.y, a.z, a.w, b.x, b.z);
}
// record.tile_mask: bit p = (ty - y0) nx + (tx - x0) set iff tile (tx, ty) of the
// rectangle passes tile_hit, for rectangles of <= 31 tiles; GS_TILE_MASK_FULL
// (bit 31) = larger rectangle, test per tile when binning
constexpr uint32_t GS_TILE_MASK_FULL = 0x80000000u;
__device__ __forceinline__ bool tile_hit(const TightRec& g, uint32_t tx, uint32_t ty) {
    const float X0 = (float)(tx * 16u), X1 = (float)(tx * 16u + 15u);
    const float Y0 = (float)(ty * 16u), Y1 = (float)(ty * 16u + 15u);
    const bool inx = X0 <= g.u && g.u <= X1, iny = Y0 <= g.v && g.v <= Y1;
    if (inx && iny) return true;
    float pmax = -INFINITY;
    if (!inx) {
        const float dx = __fsub_rn(g.u < X0 ? X0 : X1, g.u);
        const float dy = fminf(fmaxf(__fmul_rn(g.sy, dx), __fsub_rn(Y0, g.v)), __fsub_rn(Y1, g.v));
        pmax = fmaxf(pmax, p_at(g.ea, g.eb, g.ec, dx, dy));
    }
    if (!iny) {
        const float dy = __fsub_rn(g.v < Y0 ? Y0 : Y1, g.v);
        const float dx = fminf(fmaxf(__fmul_rn(g.sx, dy), __fsub_rn(X0, g.u)), __fsub_rn(X1, g.u));
        pmax = fmaxf(pmax, p_at(g.ea, g.eb, g.ec, dx, dy));
    }
    return pmax >= g.ecut;
}

__device__ __forceinline__ int view_tiles_x(const gs_view& v) { return (v.width + GS_TILE - 1) / GS_TILE; }

// index of the view owning batch tile `t` (views sorted by tile_offset)
__device__ __forceinline__ int find_view_by_tile(const gs_view* __restrict__ views, int n_views, uint32_t t) {
    int lo = 0, hi = n_views - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(&views[mid].tile_offset) <= t) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// O13 for one pixel (gs_backproject and the fused epilogue of gs_rasterize_backproject):
// valid iff A >= a_min and Dz/A > 0 (fp32); X = R^T(((px - cx)/fx zb, (py - cy)/fy zb, zb) - t)
__device__ __forceinline__ void bp_pixel(const gs_view& V, float Dz, float A, float a_min, int px, int py, float& X,
                                         float& Y, float& Z, uint8_t& ok) {
    // validity decided in fp32 on the fp32 A (same precision as the oracle)
    const bool valid = A >= a_min && (Dz / A) > 0.0f;
    if (!valid) { X = Y = Z = 0.f; ok = 0; return; }
    const float zb = Dz / A;
    const float c0 = ((float)px - V.cx) / V.fx * zb - V.t[0];
    const float c1 = ((float)py - V.cy) / V.fy * zb - V.t[1];
    const float c2 = zb - V.t[2];
    X = V.R[0] * c0 + V.R[3] * c1 + V.R[6] * c2;
    Y = V.R[1] * c0 + V.R[4] * c1 + V.R[7] * c2;
    Z = V.R[2] * c0 + V.R[5] * c1 + V.R[8] * c2;
    ok = 1;
}

}  // namespace gs
