// gs_api.cu -- host-side helpers of the C ABI (include/gs.h): version, error
// string, default parameters, batch layout, argument validation.
#include <cmath>
#include <cstring>

#include "gs_common.cuh"

namespace gs {

static thread_local char g_err[512] = "no error";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

gs_status validate_views(const gs_view* vh, const gs_view* vd, int32_t n_views, int64_t* total_pixels,
                         int64_t* total_tiles) {
    GS_REQUIRE(vh != nullptr, GS_INVALID_ARG, "views_host is NULL");
    GS_REQUIRE(vd != nullptr, GS_INVALID_ARG, "views_dev is NULL");
    GS_REQUIRE(n_views >= 1, GS_INVALID_ARG, "n_views = %d < 1", n_views);
    GS_REQUIRE(n_views <= GS_MAX_VIEWS, GS_UNSUPPORTED, "n_views = %d > %d", n_views, GS_MAX_VIEWS);
    int64_t pix = 0, tiles = 0;
    for (int32_t i = 0; i < n_views; ++i) {
        const gs_view& v = vh[i];
        GS_REQUIRE(v.width >= 1 && v.height >= 1 && v.width <= 65535 * 16 && v.height <= 65535 * 16,
                   GS_INVALID_ARG, "views[%d]: bad image size %dx%d", i, v.width, v.height);
        GS_REQUIRE(std::isfinite(v.fx) && std::isfinite(v.fy) && v.fx > 0.f && v.fy > 0.f &&
                       std::isfinite(v.cx) && std::isfinite(v.cy),
                   GS_INVALID_ARG, "views[%d]: bad intrinsics", i);
        for (int k = 0; k < 9; ++k)
            GS_REQUIRE(std::isfinite(v.R[k]), GS_INVALID_ARG, "views[%d].R[%d] not finite", i, k);
        for (int k = 0; k < 3; ++k)
            GS_REQUIRE(std::isfinite(v.t[k]), GS_INVALID_ARG, "views[%d].t[%d] not finite", i, k);
        GS_REQUIRE(v.pix_offset == pix, GS_INVALID_ARG,
                   "views[%d].pix_offset = %lld, expected %lld (use gs_views_layout)", i,
                   (long long)v.pix_offset, (long long)pix);
        GS_REQUIRE((int64_t)v.tile_offset == tiles, GS_INVALID_ARG,
                   "views[%d].tile_offset = %u, expected %lld (use gs_views_layout)", i, v.tile_offset,
                   (long long)tiles);
        pix += (int64_t)v.width * v.height;
        tiles += (int64_t)tiles_x(v) * tiles_y(v);
    }
    GS_REQUIRE(tiles < (int64_t(1) << 31), GS_UNSUPPORTED, "total tiles %lld >= 2^31", (long long)tiles);
    if (total_pixels) *total_pixels = pix;
    if (total_tiles) *total_tiles = tiles;
    return GS_OK;
}

gs_status validate_scene(const gs_scene* s, bool need_geometry) {
    GS_REQUIRE(s != nullptr, GS_INVALID_ARG, "scene is NULL");
    GS_REQUIRE(s->n >= 0 && s->n < (int64_t(1) << 32), GS_INVALID_ARG, "scene->n = %lld out of range",
               (long long)s->n);
    GS_REQUIRE(s->sh_degree >= 0 && s->sh_degree <= 3, GS_UNSUPPORTED, "sh_degree = %d not in 0..3",
               s->sh_degree);
    GS_REQUIRE(s->feat_dim >= 0 && s->feat_dim <= GS_MAX_FEAT_DIM && s->feat_dim % 4 == 0, GS_UNSUPPORTED,
               "feat_dim = %d (need 0..64, multiple of 4)", s->feat_dim);
    GS_REQUIRE(s->feat_dim == 0 || s->feat != nullptr || s->n == 0, GS_INVALID_ARG,
               "feat_dim = %d but feat is NULL", s->feat_dim);
    if (need_geometry && s->n > 0) {
        GS_REQUIRE(s->pos && s->quat && s->scale && s->opacity && s->sh, GS_INVALID_ARG,
                   "scene geometry pointer is NULL");
    }
    GS_REQUIRE(s->n_blocks >= 0, GS_INVALID_ARG, "n_blocks = %d < 0", s->n_blocks);
    if (s->n_blocks > 0 && need_geometry) {
        GS_REQUIRE(s->block_offsets && s->block_bounds, GS_INVALID_ARG,
                   "n_blocks = %d but block_offsets/block_bounds is NULL", s->n_blocks);
    }
    return GS_OK;
}

}  // namespace gs

extern "C" {

int32_t gs_abi_version(void) { return GS_ABI_VERSION; }

const char* gs_last_error(void) { return gs::g_err; }

gs_params gs_default_params(void) {
    gs_params p;
    p.z_near = 0.2f;
    p.dilation = 0.3f;
    p.clamp_margin = 0.15f;
    p.alpha_min = 1.0f / 255.0f;
    p.alpha_max = 0.99f;
    p.t_min = 1e-4f;
    return p;
}

gs_status gs_views_layout(gs_view* views_host, int32_t n_views, int64_t* total_pixels, int64_t* total_tiles) {
    GS_REQUIRE(views_host != nullptr, GS_INVALID_ARG, "views_host is NULL");
    GS_REQUIRE(n_views >= 1, GS_INVALID_ARG, "n_views = %d < 1", n_views);
    GS_REQUIRE(n_views <= GS_MAX_VIEWS, GS_UNSUPPORTED, "n_views = %d > %d", n_views, GS_MAX_VIEWS);
    int64_t pix = 0, tiles = 0;
    for (int32_t i = 0; i < n_views; ++i) {
        gs_view& v = views_host[i];
        GS_REQUIRE(v.width >= 1 && v.height >= 1 && v.width <= 65535 * 16 && v.height <= 65535 * 16,
                   GS_INVALID_ARG, "views[%d]: bad image size %dx%d", i, v.width, v.height);
        GS_REQUIRE(tiles < (int64_t(1) << 31), GS_UNSUPPORTED, "total tiles >= 2^31");
        v.pix_offset = pix;
        v.tile_offset = (uint32_t)tiles;
        v.reserved = 0;
        pix += (int64_t)v.width * v.height;
        tiles += (int64_t)gs::tiles_x(v) * gs::tiles_y(v);
    }
    GS_REQUIRE(tiles < (int64_t(1) << 31), GS_UNSUPPORTED, "total tiles %lld >= 2^31", (long long)tiles);
    if (total_pixels) *total_pixels = pix;
    if (total_tiles) *total_tiles = tiles;
    return GS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// gs_validate_scene (debug): per Gaussian invariant checks, first offender by
// a 64-bit atomicMin on (index << 8 | reason).
// ---------------------------------------------------------------------------
namespace gs {
namespace {
__device__ __forceinline__ bool finite_f(float x) { return isfinite(x); }

__global__ void validate_scene_kernel(gs_scene S, int32_t unit_quat, unsigned long long* key) {
    const int64_t n = S.n;
    const int nk = (S.sh_degree + 1) * (S.sh_degree + 1) * 3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t r = GS_BAD_NONE;
        const float px = S.pos[i], py = S.pos[n + i], pz = S.pos[2 * n + i];
        const float qw = S.quat[i], qx = S.quat[n + i], qy = S.quat[2 * n + i], qz = S.quat[3 * n + i];
        const float sx = S.scale[i], sy = S.scale[n + i], sz = S.scale[2 * n + i];
        const float o = S.opacity[i];
        const double qn = sqrt((double)qw * qw + (double)qx * qx + (double)qy * qy + (double)qz * qz);
        if (!(finite_f(px) && finite_f(py) && finite_f(pz))) r = GS_BAD_POSITION;
        else if (!(finite_f(qw) && finite_f(qx) && finite_f(qy) && finite_f(qz)) || !(qn > 0.0)) r = GS_BAD_QUAT;
        else if (unit_quat && fabs(qn - 1.0) > 1e-6) r = GS_BAD_QUAT_NORM;
        else if (!(finite_f(sx) && finite_f(sy) && finite_f(sz) && sx > 0.f && sy > 0.f && sz > 0.f))
            r = GS_BAD_SCALE;
        else if (!(o >= 0.f && o <= 1.f)) r = GS_BAD_OPACITY;
        else {
            for (int k = 0; k < nk && r == GS_BAD_NONE; ++k)
                if (!finite_f(S.sh[(int64_t)k * n + i])) r = GS_BAD_SH;
            for (int c = 0; c < S.feat_dim && r == GS_BAD_NONE; ++c)
                if (!finite_f(S.feat[i * S.feat_dim + c])) r = GS_BAD_FEATURE;
        }
        if (r != GS_BAD_NONE) atomicMin(key, ((unsigned long long)i << 8) | r);
    }
}

// gs_sanitize_scene: project the parameters back onto the set gs_project renders
// (opacity in [opacity_min, 1], finite scales >= scale_min, a non-zero finite
// quaternion); counts the Gaussians it changed.
__global__ void sanitize_scene_kernel(gs_scene S, float opacity_min, float scale_min, unsigned long long* changed) {
    const int64_t n = S.n;
    unsigned long long local = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        bool ch = false;
        float* op = const_cast<float*>(S.opacity) + i;
        const float o = *op;
        const float oc = (o == o) ? fminf(fmaxf(o, opacity_min), 1.0f) : opacity_min;
        if (oc != o) { *op = oc; ch = true; }
        for (int k = 0; k < 3; ++k) {
            float* sp = const_cast<float*>(S.scale) + (int64_t)k * n + i;
            const float sv = *sp;
            const float sc = (sv == sv) ? fminf(fmaxf(sv, scale_min), 3.0e38f) : scale_min;   // NaN -> scale_min
            if (sc != sv) { *sp = sc; ch = true; }
        }
        float* q = const_cast<float*>(S.quat);
        const float qw = q[i], qx = q[n + i], qy = q[2 * n + i], qz = q[3 * n + i];
        const float qq = qw * qw + qx * qx + qy * qy + qz * qz;
        if (!(isfinite(qq) && qq > 1e-30f)) {
            q[i] = 1.f; q[n + i] = 0.f; q[2 * n + i] = 0.f; q[3 * n + i] = 0.f;
            ch = true;
        }
        local += ch;
    }
    if (local) atomicAdd(changed, local);
}

__global__ void validate_finish_kernel(unsigned long long* key, int32_t* reason) {
    const unsigned long long k = *key;
    const bool valid = k == ~0ull;
    *reason = valid ? GS_BAD_NONE : (int32_t)(k & 0xffull);
    *reinterpret_cast<int64_t*>(key) = valid ? -1 : (int64_t)(k >> 8);
}
}  // namespace
}  // namespace gs

extern "C" gs_status gs_validate_scene(const gs_scene* scene, int32_t unit_quat, int64_t* first_bad, int32_t* reason,
                                       void* stream) {
    gs_status st = gs::validate_scene(scene, true);
    if (st != GS_OK) return st;
    GS_REQUIRE(first_bad != nullptr && reason != nullptr, GS_INVALID_ARG, "first_bad / reason is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* key = reinterpret_cast<unsigned long long*>(first_bad);
    cudaMemsetAsync(key, 0xff, sizeof(*key), s);
    if (scene->n > 0) {
        const int64_t blocks = std::min<int64_t>((scene->n + 255) / 256, (int64_t)gs::num_sms() * 8);
        gs::validate_scene_kernel<<<(unsigned)blocks, 256, 0, s>>>(*scene, unit_quat, key);
        if ((st = gs::check_launch("validate_scene_kernel")) != GS_OK) return st;
    }
    gs::validate_finish_kernel<<<1, 1, 0, s>>>(key, reason);
    return gs::check_launch("validate_finish_kernel");
}

extern "C" gs_status gs_sanitize_scene(const gs_scene* scene, float opacity_min, float scale_min, uint64_t* changed,
                                       void* stream) {
    gs_status st = gs::validate_scene(scene, true);
    if (st != GS_OK) return st;
    GS_REQUIRE(opacity_min >= 0.f && opacity_min <= 1.f && scale_min > 0.f && changed != nullptr, GS_INVALID_ARG,
               "gs_sanitize_scene: need 0 <= opacity_min <= 1, scale_min > 0, changed != NULL");
    if (scene->n == 0) return GS_OK;
    const int64_t blocks = std::min<int64_t>((scene->n + 255) / 256, (int64_t)gs::num_sms() * 8);
    gs::sanitize_scene_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        *scene, opacity_min, scale_min, reinterpret_cast<unsigned long long*>(changed));
    return gs::check_launch("sanitize_scene_kernel");
}
