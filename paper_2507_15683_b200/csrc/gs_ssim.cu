// gs_ssim.cu -- N4: Eq. 3's D-SSIM term and its gradient w.r.t. the rendered
// image (reading Q37: 1 - SSIM, 11 x 11 Gaussian window sigma 1.5,
// zero padding, C1 = 0.01^2, C2 = 0.03^2).
//
// Two HBM-bound tiled passes over n_planes contiguous H x W planes.  Each CTA
// owns a 32 x 16 output tile: it stages the (16 + 10) x (32 + 10) halo of its
// input planes in shared memory (zero outside the plane = the zero padding),
// runs the separable window horizontally into a (16 + 10) x 32 buffer and then
// vertically, one output column per lane.
//   pass 1 (ssim_moments_kernel): the five window moments of (x, y) -> the SSIM
//     map S, *loss += scale sum (1 - S), and the three partials
//     dS/dmu_x, dS/dE_xx, dS/dE_xy written to the workspace (12 B/px);
//   pass 2 (ssim_grad_kernel): the window correlation of the three partials
//     (its own transpose: the window is symmetric, the padding zero) combined
//     with x, y into grad += -scale (w*dmu + 2 x w*dxx + y w*dxy).
// Algorithmic bytes: pass 1 reads x, y (8 B/px) and writes 12 B/px; pass 2
// reads the partials, x, y (20 B/px) and read-modify-writes grad (8 B/px):
// 48 B per pixel per plane in all.  fp32 arithmetic, fp64 loss accumulation.
#include "gs_common.cuh"

#include <cmath>

namespace gs {
namespace {

constexpr int SS_TW = 32, SS_TH = 16, SS_R = 5, SS_K = 2 * SS_R + 1;
constexpr int SS_HW = SS_TW + 2 * SS_R, SS_HH = SS_TH + 2 * SS_R;
constexpr int SS_THREADS = 256;
constexpr float SS_C1 = 0.01f * 0.01f, SS_C2 = 0.03f * 0.03f;

struct Win {
    float w[SS_K];
};  // the window, passed by value (kernel-parameter constant bank)

template <int NIN>
__device__ __forceinline__ void load_halo(float (*s)[SS_HH][SS_HW], const float* const (&src)[NIN], int H, int W,
                                          int x0, int y0) {
    for (int i = threadIdx.x; i < SS_HH * SS_HW; i += SS_THREADS) {
        const int r = i / SS_HW, c = i - r * SS_HW;
        const int gy = y0 - SS_R + r, gx = x0 - SS_R + c;
        const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
        const int64_t o = (int64_t)gy * W + gx;
#pragma unroll
        for (int k = 0; k < NIN; ++k) s[k][r][c] = in ? __ldg(src[k] + o) : 0.f;
    }
}

__global__ void __launch_bounds__(SS_THREADS) ssim_moments_kernel(const float* __restrict__ X,
                                                                  const float* __restrict__ Y, int H, int W,
                                                                  float scale, float* __restrict__ dmu,
                                                                  float* __restrict__ dxx, float* __restrict__ dxy,
                                                                  int64_t ws_plane_stride, double* __restrict__ loss,
                                                                  const Win win) {
    __shared__ float s_in[2][SS_HH][SS_HW];
    __shared__ float s_h[5][SS_HH][SS_TW];
    const int64_t off = (int64_t)blockIdx.z * H * W;
    const int x0 = blockIdx.x * SS_TW, y0 = blockIdx.y * SS_TH;
    const float* const src[2] = {X + off, Y + off};
    load_halo<2>(s_in, src, H, W, x0, y0);
    __syncthreads();
    for (int i = threadIdx.x; i < SS_HH * SS_TW; i += SS_THREADS) {
        const int r = i / SS_TW, c = i - r * SS_TW;
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
        for (int k = 0; k < SS_K; ++k) {
            const float a = s_in[0][r][c + k], b = s_in[1][r][c + k], w = win.w[k];
            m0 = fmaf(w, a, m0);
            m1 = fmaf(w, b, m1);
            m2 = fmaf(w, a * a, m2);
            m3 = fmaf(w, b * b, m3);
            m4 = fmaf(w, a * b, m4);
        }
        s_h[0][r][c] = m0;
        s_h[1][r][c] = m1;
        s_h[2][r][c] = m2;
        s_h[3][r][c] = m3;
        s_h[4][r][c] = m4;
    }
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double part = 0.0;
    for (int rr = ty; rr < SS_TH; rr += SS_THREADS / 32) {
        const int gy = y0 + rr, gx = x0 + tx;
        float mx = 0.f, my = 0.f, exx = 0.f, eyy = 0.f, exy = 0.f;
#pragma unroll
        for (int k = 0; k < SS_K; ++k) {
            const float w = win.w[k];
            mx = fmaf(w, s_h[0][rr + k][tx], mx);
            my = fmaf(w, s_h[1][rr + k][tx], my);
            exx = fmaf(w, s_h[2][rr + k][tx], exx);
            eyy = fmaf(w, s_h[3][rr + k][tx], eyy);
            exy = fmaf(w, s_h[4][rr + k][tx], exy);
        }
        if (gy < H && gx < W) {
            const float sxx = exx - mx * mx, syy = eyy - my * my, sxy = exy - mx * my;
            const float A1 = 2.f * mx * my + SS_C1, A2 = 2.f * sxy + SS_C2;
            const float B1 = mx * mx + my * my + SS_C1, B2 = sxx + syy + SS_C2;
            const float iA1 = 1.f / A1, iA2 = 1.f / A2, iB1 = 1.f / B1, iB2 = 1.f / B2;
            const float S = (A1 * A2) * (iB1 * iB2);
            const int64_t o = (int64_t)blockIdx.z * ws_plane_stride + (int64_t)gy * W + gx;
            dmu[o] = 2.f * S * (my * iA1 - my * iA2 - mx * iB1 + mx * iB2);
            dxx[o] = -S * iB2;
            dxy[o] = 2.f * S * iA2;
            part += (double)(1.f - S);
        }
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (tx == 0 && part != 0.0) atomicAdd(loss, part * (double)scale);
}

__global__ void __launch_bounds__(SS_THREADS) ssim_grad_kernel(const float* __restrict__ X,
                                                               const float* __restrict__ Y, int H, int W,
                                                               float scale, const float* __restrict__ dmu,
                                                               const float* __restrict__ dxx,
                                                               const float* __restrict__ dxy, int64_t ws_plane_stride,
                                                               float* __restrict__ G, const Win win) {
    __shared__ float s_in[3][SS_HH][SS_HW];
    __shared__ float s_h[3][SS_HH][SS_TW];
    const int64_t off = (int64_t)blockIdx.z * H * W, woff = (int64_t)blockIdx.z * ws_plane_stride;
    const int x0 = blockIdx.x * SS_TW, y0 = blockIdx.y * SS_TH;
    const float* const src[3] = {dmu + woff, dxx + woff, dxy + woff};
    load_halo<3>(s_in, src, H, W, x0, y0);
    __syncthreads();
    for (int i = threadIdx.x; i < SS_HH * SS_TW; i += SS_THREADS) {
        const int r = i / SS_TW, c = i - r * SS_TW;
        float m0 = 0.f, m1 = 0.f, m2 = 0.f;
#pragma unroll
        for (int k = 0; k < SS_K; ++k) {
            const float w = win.w[k];
            m0 = fmaf(w, s_in[0][r][c + k], m0);
            m1 = fmaf(w, s_in[1][r][c + k], m1);
            m2 = fmaf(w, s_in[2][r][c + k], m2);
        }
        s_h[0][r][c] = m0;
        s_h[1][r][c] = m1;
        s_h[2][r][c] = m2;
    }
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int rr = ty; rr < SS_TH; rr += SS_THREADS / 32) {
        const int gy = y0 + rr, gx = x0 + tx;
        float b0 = 0.f, b1 = 0.f, b2 = 0.f;
#pragma unroll
        for (int k = 0; k < SS_K; ++k) {
            const float w = win.w[k];
            b0 = fmaf(w, s_h[0][rr + k][tx], b0);
            b1 = fmaf(w, s_h[1][rr + k][tx], b1);
            b2 = fmaf(w, s_h[2][rr + k][tx], b2);
        }
        if (gy < H && gx < W) {
            const int64_t o = off + (int64_t)gy * W + gx;
            const float x = __ldg(X + o), y = __ldg(Y + o);
            G[o] -= scale * (b0 + 2.f * x * b1 + y * b2);
        }
    }
}

Win make_window() {
    double g[SS_K], sum = 0.0;
    for (int k = 0; k < SS_K; ++k) {
        const double d = k - SS_R;
        g[k] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += g[k];
    }
    Win w;
    for (int k = 0; k < SS_K; ++k) w.w[k] = (float)(g[k] / sum);
    return w;
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" size_t gs_dssim_workspace_bytes(int32_t n_planes, int32_t height, int32_t width) {
    if (n_planes <= 0 || height <= 0 || width <= 0) return 0;
    return (size_t)3 * n_planes * (size_t)height * (size_t)width * sizeof(float);
}

extern "C" gs_status gs_dssim_grad(const float* rendered, const float* target, int32_t n_planes, int32_t height,
                                   int32_t width, float scale, float* grad_image, float* workspace,
                                   size_t workspace_bytes, double* loss, void* stream) {
    GS_REQUIRE(n_planes >= 0 && height >= 0 && width >= 0, GS_INVALID_ARG, "gs_dssim_grad: negative size");
    GS_REQUIRE(n_planes <= 65535, GS_INVALID_ARG, "gs_dssim_grad: n_planes %d > 65535", n_planes);
    if (n_planes == 0 || height == 0 || width == 0) return GS_OK;
    GS_REQUIRE(rendered && target && grad_image && workspace && loss, GS_INVALID_ARG, "gs_dssim_grad: NULL pointer");
    GS_REQUIRE(workspace_bytes >= gs_dssim_workspace_bytes(n_planes, height, width), GS_INVALID_ARG,
               "gs_dssim_grad: workspace %zu < %zu bytes", workspace_bytes,
               gs_dssim_workspace_bytes(n_planes, height, width));
    cudaStream_t s = (cudaStream_t)stream;
    const Win win = make_window();
    const int64_t plane = (int64_t)height * width, ws_stride = plane;
    float* dmu = workspace;
    float* dxx = dmu + (int64_t)n_planes * plane;
    float* dxy = dxx + (int64_t)n_planes * plane;
    const dim3 grid((width + SS_TW - 1) / SS_TW, (height + SS_TH - 1) / SS_TH, n_planes);
    ssim_moments_kernel<<<grid, SS_THREADS, 0, s>>>(rendered, target, height, width, scale, dmu, dxx, dxy, ws_stride,
                                                    loss, win);
    gs_status st = check_launch("ssim_moments_kernel");
    if (st != GS_OK) return st;
    ssim_grad_kernel<<<grid, SS_THREADS, 0, s>>>(rendered, target, height, width, scale, dmu, dxx, dxy, ws_stride,
                                                 grad_image, win);
    return check_launch("ssim_grad_kernel");
}
