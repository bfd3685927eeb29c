// gs_common.cuh -- internal helpers of libgs (CUDA side only; not shared with
// the oracle).  Error reporting for the C ABI and small device utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdarg>

#include "../../include/gs.h"

namespace gs {

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

inline int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// ---------------------------------------------------------------- device side
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

}  // namespace gs
