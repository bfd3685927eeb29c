// gs_visibility.cu -- N1: Alg. 1 render
// visibility with projection filtering and significance scoring
// Eq. 4-6 over the records of a batch.
//
// One thread per record slot (views on grid.y).  M^r = contrib > eps, the
// forward criterion SPEC S:180 substitutes for the render-gradient test
// "||grad (X,Y,Z)[j]|| > 0" (Alg. 1 l.5); M^i = 0 <= U < W and 0 <= V < H
// (Alg. 1 l.17).  Visible records add 1 to count[gid] (Eq. 6's M) and, with
// target maps, cos(f_gid, F^t(U', V')) (Eq. 4) to score_sum[gid] (Eq. 5) as
// 2^-32 fixed point -- integer atomics, so the sums do not depend on order.
#include "gs_common.cuh"

namespace gs {
namespace {

// planar [D][Hf][Wf] -> channels-last [Hf][Wf][D] for every view (one 128-B row per
// cell at D = 32), so each visible record samples one contiguous feature row
__global__ void __launch_bounds__(256)
to_channels_last_kernel(const float* __restrict__ src, float* __restrict__ dst, const gs_view* __restrict__ views,
                        int n_views, int D, int stride) {
    const int v = blockIdx.y;
    int64_t off = 0;
    for (int u = 0; u < v; ++u)
        off += (int64_t)D * ((views[u].height + stride - 1) / stride) * ((views[u].width + stride - 1) / stride);
    const int64_t cells = (int64_t)((views[v].height + stride - 1) / stride) * ((views[v].width + stride - 1) / stride);
    const int64_t n = cells * D;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cell = i / D, c = i % D;                 // coalesced writes
        dst[off + i] = __ldg(&src[off + c * cells + cell]);
    }
}

template <bool CL>
__global__ void __launch_bounds__(256)
visibility_kernel(const gs_record* __restrict__ rec, int64_t cap, const uint32_t* __restrict__ n_rec,
                  const unsigned long long* __restrict__ contrib, const gs_view* __restrict__ views, int n_views,
                  unsigned long long eps_fixed, const float* __restrict__ feat, int D, const float* __restrict__ fmaps,
                  int stride, uint8_t* __restrict__ visible, uint32_t* __restrict__ n_visible,
                  unsigned long long* __restrict__ score_sum, uint32_t* __restrict__ count,
                  const uint32_t* __restrict__ status) {
    if (*status) return;
    const int v = blockIdx.y;
    const gs_view V = views[v];
    const uint32_t nv = min((uint64_t)n_rec[v], (uint64_t)cap);
    const int Wf = (V.width + stride - 1) / stride, Hf = (V.height + stride - 1) / stride;
    // offset of this view's target map: maps of all views are concatenated in view order
    int64_t moff = 0;
    if (fmaps)
        for (int u = 0; u < v; ++u)
            moff += (int64_t)D * ((views[u].height + stride - 1) / stride) * ((views[u].width + stride - 1) / stride);
    uint32_t nvis = 0;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < (uint32_t)cap; k += gridDim.x * blockDim.x) {
        const int64_t slot = (int64_t)v * cap + k;
        if (k >= nv) { visible[slot] = 0; continue; }
        const float4 q0 = __ldg(reinterpret_cast<const float4*>(rec + slot));            // u, v, ...
        const uint32_t gid = __ldg(&rec[slot].gid);
        const bool mi = q0.x >= 0.0f && q0.x < (float)V.width && q0.y >= 0.0f && q0.y < (float)V.height;
        const bool mr = contrib[slot] > eps_fixed;
        const bool vis = mi && mr;
        visible[slot] = vis ? 1 : 0;
        if (!vis) continue;
        ++nvis;
        atomicAdd(&count[gid], 1u);
        if (fmaps && D > 0) {
            const int cx = min(max((int)floorf((q0.x + 0.5f) / (float)stride), 0), Wf - 1);
            const int cy = min(max((int)floorf((q0.y + 0.5f) / (float)stride), 0), Hf - 1);
            const float* f = feat + (int64_t)gid * D;
            float dot = 0.f, nf = 0.f, nt = 0.f;
            if (CL) {                                   // channels-last: one contiguous row
                const float4* t4 = reinterpret_cast<const float4*>(fmaps + moff + ((int64_t)cy * Wf + cx) * D);
                const float4* f4 = reinterpret_cast<const float4*>(f);
                for (int c = 0; c < D / 4; ++c) {
                    const float4 a = __ldg(&f4[c]), b = __ldg(&t4[c]);
                    dot = fmaf(a.x, b.x, fmaf(a.y, b.y, fmaf(a.z, b.z, fmaf(a.w, b.w, dot))));
                    nf = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, nf))));
                    nt = fmaf(b.x, b.x, fmaf(b.y, b.y, fmaf(b.z, b.z, fmaf(b.w, b.w, nt))));
                }
            } else {
                const float* t = fmaps + moff + (int64_t)cy * Wf + cx;
                const int64_t plane = (int64_t)Hf * Wf;
                for (int c = 0; c < D; ++c) {
                    const float a = __ldg(&f[c]), b = __ldg(&t[c * plane]);
                    dot = fmaf(a, b, dot);
                    nf = fmaf(a, a, nf);
                    nt = fmaf(b, b, nt);
                }
            }
            const float cs = (nf > 0.f && nt > 0.f) ? dot * rsqrtf(nf) * rsqrtf(nt) : 0.f;
            atomicAdd(&score_sum[gid], (unsigned long long)__float2ll_rn(cs * 4294967296.0f));
        }
    }
    nvis = __reduce_add_sync(0xffffffffu, nvis);
    if ((threadIdx.x & 31) == 0 && nvis) atomicAdd(&n_visible[v], nvis);
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" size_t gs_visibility_workspace_bytes(const gs_view* views_host, int32_t n_views, int32_t feat_dim,
                                                int32_t stride) {
    if (!views_host || n_views < 1 || stride < 1 || feat_dim < 0) return 0;
    size_t n = 0;
    for (int i = 0; i < n_views; ++i)
        n += (size_t)feat_dim * ((views_host[i].height + stride - 1) / stride) * ((views_host[i].width + stride - 1) / stride);
    return n * sizeof(float);
}

extern "C" gs_status gs_visibility_score(const gs_projected* proj, const gs_view* views_host, const gs_view* views_dev,
                                         int32_t n_views, float eps, const float* feat, int32_t feat_dim,
                                         const float* fmaps, int32_t stride, void* ws, size_t ws_bytes,
                                         uint8_t* visible, uint32_t* n_visible, unsigned long long* score_sum,
                                         uint32_t* count, void* stream) {
    int64_t total_pixels = 0, T = 0;
    gs_status st = validate_views(views_host, views_dev, n_views, &total_pixels, &T);
    if (st != GS_OK) return st;
    GS_REQUIRE(proj && proj->rec && proj->n_rec && proj->status, GS_INVALID_ARG, "proj has a NULL pointer");
    GS_REQUIRE(proj->contrib != nullptr, GS_INVALID_ARG, "proj->contrib is NULL (render with contributions first)");
    GS_REQUIRE(visible && n_visible && count, GS_INVALID_ARG, "visible / n_visible / count is NULL");
    GS_REQUIRE(eps >= 0.f && eps == eps, GS_INVALID_ARG, "eps = %g must be >= 0", (double)eps);
    GS_REQUIRE(fmaps == nullptr || (feat != nullptr && score_sum != nullptr && feat_dim > 0), GS_INVALID_ARG,
               "target maps need feat, feat_dim > 0 and score_sum");
    GS_REQUIRE(stride >= 1, GS_INVALID_ARG, "stride = %d < 1", stride);
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(n_visible, 0, sizeof(uint32_t) * n_views, s);
    const unsigned long long eps_fixed = (unsigned long long)((double)eps * 4294967296.0);
    const int64_t cap = proj->rec_capacity;
    const int64_t per_view = std::max<int64_t>(1, std::min<int64_t>((cap + 255) / 256, 4 * num_sms() / n_views + 1));
    dim3 grid((unsigned)per_view, (unsigned)n_views);
    const bool cl = fmaps != nullptr && feat_dim % 4 == 0 && ws != nullptr &&
                    ws_bytes >= gs_visibility_workspace_bytes(views_host, n_views, feat_dim, stride);
    if (cl) {
        dim3 tg((unsigned)std::max<int64_t>(1, 2 * num_sms() / n_views + 1), (unsigned)n_views);
        to_channels_last_kernel<<<tg, 256, 0, s>>>(fmaps, static_cast<float*>(ws), views_dev, n_views, feat_dim, stride);
        if ((st = check_launch("to_channels_last_kernel")) != GS_OK) return st;
        visibility_kernel<true><<<grid, 256, 0, s>>>(proj->rec, cap, proj->n_rec, proj->contrib, views_dev, n_views,
                                                     eps_fixed, feat, feat_dim, static_cast<const float*>(ws), stride,
                                                     visible, n_visible, score_sum, count, proj->status);
    } else {
        visibility_kernel<false><<<grid, 256, 0, s>>>(proj->rec, cap, proj->n_rec, proj->contrib, views_dev, n_views,
                                                      eps_fixed, feat, feat_dim, fmaps, stride, visible, n_visible,
                                                      score_sum, count, proj->status);
    }
    return check_launch("visibility_kernel");
}
