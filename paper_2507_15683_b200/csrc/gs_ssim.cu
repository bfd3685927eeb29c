// gs_ssim.cu -- N4: Eq. 3's D-SSIM term and its gradient w.r.t. the rendered
// image (reading Q37: 1 - SSIM, 11 x 11 Gaussian window sigma 1.5,
// zero padding, C1 = 0.01^2, C2 = 0.03^2).
//
// Two tiled passes over n_planes contiguous H x W planes (measured: bound by
// instruction issue, 81-87 %, at 0.43 of the HBM roofline).  Each CTA
// owns a 32 x 32 output tile: it stages the (32 + 10) x (32 + 10) halo of its
// input planes in shared memory (zero outside the plane = the zero padding),
// runs the separable window horizontally into a (32 + 10) x 32 buffer (four
// adjacent columns per lane from a 14-value register window) and then
// vertically (four adjacent rows per lane, one column per lane).
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

#ifndef GS_SSIM_TH
#define GS_SSIM_TH 32
#endif
#ifndef GS_SSIM_HJ_MOM
#define GS_SSIM_HJ_MOM 4
#endif
#ifndef GS_SSIM_PRELOAD
#define GS_SSIM_PRELOAD 1
#endif
#ifndef GS_SSIM_HJ_GRAD
#define GS_SSIM_HJ_GRAD 4
#endif
constexpr int SS_TW = 32, SS_TH = GS_SSIM_TH, SS_R = 5, SS_K = 2 * SS_R + 1;
constexpr int SS_HW = SS_TW + 2 * SS_R, SS_HH = SS_TH + 2 * SS_R;
// halo row stride: 45 = 13 (mod 32) puts the four rows a warp's horizontal pass
// reads (8 lanes x 4 columns each) in distinct bank classes mod 4 -> conflict-free
constexpr int SS_RS = 45;
constexpr int SS_THREADS = 256, SS_WARPS = SS_THREADS / 32, SS_VR = SS_TH / SS_WARPS;  // 4 rows per lane
// columns per lane in the horizontal pass (measured optimum: 4 for both passes)
constexpr int SS_HJ_MOM = GS_SSIM_HJ_MOM, SS_HJ_GRAD = GS_SSIM_HJ_GRAD;
constexpr float SS_C1 = 0.01f * 0.01f, SS_C2 = 0.03f * 0.03f;

struct Win {
    float w[SS_K];
};  // the window, passed by value (kernel-parameter constant bank)

// All of a thread's halo loads are issued before the first shared-memory store
// (SS_LD = 7 iterations x NIN loads in flight per thread).
constexpr int SS_LD = (SS_HH * SS_HW + SS_THREADS - 1) / SS_THREADS;

template <int NIN>
__device__ __forceinline__ void load_halo(float (*s)[SS_HH][SS_RS], const float* const (&src)[NIN], int H, int W,
                                          int x0, int y0) {
    float v[SS_LD][NIN];
#pragma unroll
    for (int t = 0; t < SS_LD; ++t) {
        const int i = threadIdx.x + t * SS_THREADS;
        const int r = i / SS_HW, c = i - r * SS_HW;
        const int gy = y0 - SS_R + r, gx = x0 - SS_R + c;
        const bool in = i < SS_HH * SS_HW && gy >= 0 && gy < H && gx >= 0 && gx < W;
        const int64_t o = (int64_t)gy * W + gx;
#pragma unroll
        for (int k = 0; k < NIN; ++k) v[t][k] = in ? __ldg(src[k] + o) : 0.f;
    }
#pragma unroll
    for (int t = 0; t < SS_LD; ++t) {
        const int i = threadIdx.x + t * SS_THREADS;
        const int r = i / SS_HW, c = i - r * SS_HW;
        if (i < SS_HH * SS_HW) {
#pragma unroll
            for (int k = 0; k < NIN; ++k) s[k][r][c] = v[t][k];
        }
    }
}

// Horizontal window pass: NOUT row sums over SS_HH x SS_TW positions, each lane
// SS_HJ adjacent columns from a register window of SS_HJ + 10 halo values per
// input (MOM: the five moments x, y, xx, yy, xy of two inputs; else identity).
template <int NIN, int NOUT, bool MOM, int SS_HJ>
__device__ __forceinline__ void horizontal(const float (*s_in)[SS_HH][SS_RS], float (*s_h)[SS_HH][SS_TW],
                                           const Win& win) {
    constexpr int G = SS_TW / SS_HJ;
    for (int it = threadIdx.x; it < SS_HH * G; it += SS_THREADS) {
        const int r = it / G, c0 = (it - r * G) * SS_HJ;
        float v[MOM ? 5 : NIN][SS_HJ + SS_K - 1];
#pragma unroll
        for (int q = 0; q < NIN; ++q)
#pragma unroll
            for (int k = 0; k < SS_HJ + SS_K - 1; ++k) v[q][k] = s_in[q][r][c0 + k];
        if constexpr (MOM) {   // the products once per halo value, not once per tap
#pragma unroll
            for (int k = 0; k < SS_HJ + SS_K - 1; ++k) {
                v[2][k] = v[0][k] * v[0][k];
                v[3][k] = v[1][k] * v[1][k];
                v[4][k] = v[0][k] * v[1][k];
            }
        }
        float acc[NOUT][SS_HJ];
#pragma unroll
        for (int m = 0; m < NOUT; ++m)
#pragma unroll
            for (int j = 0; j < SS_HJ; ++j) acc[m][j] = 0.f;
#pragma unroll
        for (int k = 0; k < SS_K; ++k) {
            const float w = win.w[k];
#pragma unroll
            for (int j = 0; j < SS_HJ; ++j)
#pragma unroll
                for (int m = 0; m < NOUT; ++m) acc[m][j] = fmaf(w, v[m][j + k], acc[m][j]);
        }
#pragma unroll
        for (int m = 0; m < NOUT; ++m) {
            if constexpr (SS_HJ == 4)
                *reinterpret_cast<float4*>(&s_h[m][r][c0]) = make_float4(acc[m][0], acc[m][1], acc[m][2], acc[m][3]);
            else if constexpr (SS_HJ == 2)
                *reinterpret_cast<float2*>(&s_h[m][r][c0]) = make_float2(acc[m][0], acc[m][1]);
            else
#pragma unroll
                for (int j = 0; j < SS_HJ; ++j) s_h[m][r][c0 + j] = acc[m][j];
        }
    }
}

// Vertical window pass for lane column tx and output rows r0 .. r0 + SS_VR - 1.
template <int NOUT>
__device__ __forceinline__ void vertical(const float (*s_h)[SS_HH][SS_TW], int r0, int tx, const Win& win,
                                         float (&out)[NOUT][SS_VR]) {
#pragma unroll
    for (int m = 0; m < NOUT; ++m) {
        float v[SS_VR + SS_K - 1];
#pragma unroll
        for (int k = 0; k < SS_VR + SS_K - 1; ++k) v[k] = s_h[m][r0 + k][tx];
#pragma unroll
        for (int j = 0; j < SS_VR; ++j) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < SS_K; ++k) acc = fmaf(win.w[k], v[j + k], acc);
            out[m][j] = acc;
        }
    }
}

__global__ void __launch_bounds__(SS_THREADS) ssim_moments_kernel(const float* __restrict__ X,
                                                                  const float* __restrict__ Y, int H, int W,
                                                                  float scale, float* __restrict__ dmu,
                                                                  float* __restrict__ dxx, float* __restrict__ dxy,
                                                                  int64_t ws_plane_stride, double* __restrict__ loss,
                                                                  const Win win) {
    __shared__ __align__(16) float s_in[2][SS_HH][SS_RS];
    __shared__ __align__(16) float s_h[5][SS_HH][SS_TW];
    const int64_t off = (int64_t)blockIdx.z * H * W;
    const int x0 = blockIdx.x * SS_TW, y0 = blockIdx.y * SS_TH;
    const float* const src[2] = {X + off, Y + off};
    load_halo<2>(s_in, src, H, W, x0, y0);
    __syncthreads();
    horizontal<2, 5, true, SS_HJ_MOM>(s_in, s_h, win);
    __syncthreads();
    const int tx = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * SS_VR;
    float mom[5][SS_VR];
    vertical<5>(s_h, r0, tx, win, mom);
    double part = 0.0;
    const int gx = x0 + tx;
#pragma unroll
    for (int j = 0; j < SS_VR; ++j) {
        const int gy = y0 + r0 + j;
        if (gy < H && gx < W) {
            const float mx = mom[0][j], my = mom[1][j];
            const float sxx = mom[2][j] - mx * mx, syy = mom[3][j] - my * my, sxy = mom[4][j] - mx * my;
            const float A1 = 2.f * mx * my + SS_C1, A2 = 2.f * sxy + SS_C2;
            const float B1 = mx * mx + my * my + SS_C1, B2 = sxx + syy + SS_C2;
            // one division: with iQ = 1 / (B1 B2), S = A1 A2 iQ, S/A1 = A2 iQ,
            // S/A2 = A1 iQ, S/B1 = S B2 iQ, S/B2 = S B1 iQ
            const float iQ = 1.f / (B1 * B2);
            const float S = (A1 * A2) * iQ;
            const int64_t o = (int64_t)blockIdx.z * ws_plane_stride + (int64_t)gy * W + gx;
            dmu[o] = 2.f * iQ * (my * (A2 - A1) + mx * S * (B1 - B2));
            dxx[o] = -S * B1 * iQ;
            dxy[o] = 2.f * A1 * iQ;
            part += (double)(1.f - S);
        }
    }
    // one same-address fp64 atomic per CTA (per warp they serialise: ~1.2 M per 64 C4 views)
    __shared__ double s_part[SS_WARPS];
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (tx == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < SS_WARPS; ++w) sum += s_part[w];
        if (sum != 0.0) atomicAdd(loss, sum * (double)scale);
    }
}

__global__ void __launch_bounds__(SS_THREADS) ssim_grad_kernel(const float* __restrict__ X,
                                                               const float* __restrict__ Y, int H, int W,
                                                               float scale, const float* __restrict__ dmu,
                                                               const float* __restrict__ dxx,
                                                               const float* __restrict__ dxy, int64_t ws_plane_stride,
                                                               float* __restrict__ G, const Win win) {
    __shared__ __align__(16) float s_in[3][SS_HH][SS_RS];
    __shared__ __align__(16) float s_h[3][SS_HH][SS_TW];
    const int64_t off = (int64_t)blockIdx.z * H * W, woff = (int64_t)blockIdx.z * ws_plane_stride;
    const int x0 = blockIdx.x * SS_TW, y0 = blockIdx.y * SS_TH;
    const float* const src[3] = {dmu + woff, dxx + woff, dxy + woff};
    const int tx = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * SS_VR;
    const int gx = x0 + tx;
#if GS_SSIM_PRELOAD
    // the epilogue's x, y and gradient loads issued first, in flight during the window passes
    float px[SS_VR], py[SS_VR], pg[SS_VR];
#pragma unroll
    for (int j = 0; j < SS_VR; ++j) {
        const int gy = y0 + r0 + j;
        const bool in = gy < H && gx < W;
        const int64_t o = off + (int64_t)gy * W + gx;
        px[j] = in ? __ldg(X + o) : 0.f;
        py[j] = in ? __ldg(Y + o) : 0.f;
        pg[j] = in ? G[o] : 0.f;
    }
#endif
    load_halo<3>(s_in, src, H, W, x0, y0);
    __syncthreads();
    horizontal<3, 3, false, SS_HJ_GRAD>(s_in, s_h, win);
    __syncthreads();
    float b[3][SS_VR];
    vertical<3>(s_h, r0, tx, win, b);
#pragma unroll
    for (int j = 0; j < SS_VR; ++j) {
        const int gy = y0 + r0 + j;
        if (gy < H && gx < W) {
            const int64_t o = off + (int64_t)gy * W + gx;
#if GS_SSIM_PRELOAD
            G[o] = pg[j] - scale * (b[0][j] + 2.f * px[j] * b[1][j] + py[j] * b[2][j]);
#else
            const float x = __ldg(X + o), y = __ldg(Y + o);
            G[o] -= scale * (b[0][j] + 2.f * x * b[1][j] + y * b[2][j]);
#endif
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
    GS_REQUIRE(workspace_bytes >= gs_dssim_workspace_bytes(n_planes, height, width), GS_WORKSPACE_TOO_SMALL,
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
