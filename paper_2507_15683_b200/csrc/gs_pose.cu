// gs_pose.cu -- N2 pose stage: Eq. 10's
// robust PnP on the dense 2D-3D correspondences gs_match produces, and
// Algorithm 2's consistency verification (
// reading Q35).
//
// gs_pnp: one CTA per problem (query).  1. ordered compaction of the query
// pixels whose match carries a valid 3D point (block scans; with n > cap valid
// pixels, every k-th in pixel order, k = ceil(n / cap));
// 2. RANSAC: n_hyp hypotheses, each the exact fit of a 3-correspondence sample
// (counter-based hash, identical to the oracle's) by Gauss-Newton from the
// render pose, fp64, one thread each; 3. each hypothesis scored by its inlier
// count (e <= tau, z > 0) over all correspondences; best = most inliers, ties
// to the lowest index, the start pose kept unless beaten; 4. damped
// Gauss-Newton on the truncated quadratic min(e^2, tau^2): inliers re-selected
// every step, normal equations reduced over the CTA (warp shuffles, fp64),
// solved by one thread (6x6 Cholesky).  The refined pose is written into a
// gs_view (intrinsics and batch offsets copied), so the next gs_project of the
// refinement loop reads it directly -- no host round trip, graph-capturable.
#include <cmath>

#include "gs_common.cuh"

namespace gs {
namespace {

constexpr int PNP_THREADS = 256;
constexpr int NEWTON_ITERS = 8;
constexpr int REFINE_ITERS = 10;
constexpr double DAMPING = 1e-6;
constexpr int MAX_HYP = PNP_THREADS;

struct Pose {
    double R[9], t[3];
};

__device__ __forceinline__ uint32_t sample_hash(uint32_t seed, uint32_t h, uint32_t k) {
    uint32_t x = seed * 0x9E3779B1u + h * 0x85EBCA77u + k * 0xC2B2AE3Du;
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}

__device__ void so3_exp(const double w[3], double E[9]) {
    const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    const double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    double a, b;
    if (th < 1e-12) {
        a = 1.0;
        b = 0.0;
    } else {
        a = sin(th) / th;
        b = (1.0 - cos(th)) / (th * th);
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double kk = 0;
            for (int m = 0; m < 3; ++m) kk += K[i * 3 + m] * K[m * 3 + j];
            E[i * 3 + j] = (i == j ? 1.0 : 0.0) + a * K[i * 3 + j] + b * kk;
        }
}

// T <- Exp(xi) T, xi = (v, w)
__device__ void apply(Pose& P, const double xi[6]) {
    double E[9];
    so3_exp(xi + 3, E);
    double R[9], t[3];
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) R[i * 3 + j] = E[i * 3] * P.R[j] + E[i * 3 + 1] * P.R[3 + j] + E[i * 3 + 2] * P.R[6 + j];
        t[i] = E[i * 3] * P.t[0] + E[i * 3 + 1] * P.t[1] + E[i * 3 + 2] * P.t[2] + xi[i];
    }
    for (int i = 0; i < 9; ++i) P.R[i] = R[i];
    for (int i = 0; i < 3; ++i) P.t[i] = t[i];
}

struct Obs {
    double r[2];      // residual (pixel - observation)
    double J[2][6];   // d residual / d xi
    double z;
};

__device__ __forceinline__ void observe(const Pose& P, const float4& K, float u, float v, float X, float Y, float Z,
                                        Obs& o, bool want_j) {
    const double x = P.R[0] * X + P.R[1] * Y + P.R[2] * Z + P.t[0];
    const double y = P.R[3] * X + P.R[4] * Y + P.R[5] * Z + P.t[1];
    const double z = P.R[6] * X + P.R[7] * Y + P.R[8] * Z + P.t[2];
    o.z = z;
    const double zs = fabs(z) > 1e-12 ? z : 1e-12;
    o.r[0] = K.x * x / zs + K.z - u;
    o.r[1] = K.y * y / zs + K.w - v;
    if (!want_j) return;
    const double a = K.x / zs, c = -K.x * x / (zs * zs), d = K.y / zs, e = -K.y * y / (zs * zs);
    // d(pixel)/d(Pc) . [I | -[Pc]x]
    o.J[0][0] = a; o.J[0][1] = 0; o.J[0][2] = c;
    o.J[0][3] = c * y; o.J[0][4] = a * z - c * x; o.J[0][5] = -a * y;
    o.J[1][0] = 0; o.J[1][1] = d; o.J[1][2] = e;
    o.J[1][3] = -d * z + e * y; o.J[1][4] = -e * x; o.J[1][5] = d * x;
}

// 6x6 SPD solve A x = b by Cholesky (in place); false if not positive definite
__device__ bool chol_solve(double A[36], const double b[6], double x[6]) {
    for (int j = 0; j < 6; ++j) {
        double s = A[j * 6 + j];
        for (int k = 0; k < j; ++k) s -= A[j * 6 + k] * A[j * 6 + k];
        if (!(s > 0.0)) return false;
        const double l = sqrt(s);
        A[j * 6 + j] = l;
        for (int i = j + 1; i < 6; ++i) {
            double q = A[i * 6 + j];
            for (int k = 0; k < j; ++k) q -= A[i * 6 + k] * A[j * 6 + k];
            A[i * 6 + j] = q / l;
        }
    }
    double y[6];
    for (int i = 0; i < 6; ++i) {
        double q = b[i];
        for (int k = 0; k < i; ++k) q -= A[i * 6 + k] * y[k];
        y[i] = q / A[i * 6 + i];
    }
    for (int i = 5; i >= 0; --i) {
        double q = y[i];
        for (int k = i + 1; k < 6; ++k) q -= A[k * 6 + i] * x[k];
        x[i] = q / A[i * 6 + i];
    }
    for (int i = 0; i < 6; ++i)
        if (!isfinite(x[i])) return false;
    return true;
}

__device__ __forceinline__ bool is_inlier(const Obs& o, double tau) {
    return o.z > 0.0 && sqrt(o.r[0] * o.r[0] + o.r[1] * o.r[1]) <= tau;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__global__ void __launch_bounds__(PNP_THREADS)
pnp_kernel(const uint8_t* __restrict__ valid, const float* __restrict__ xyz, int H, int W,
           const gs_view* __restrict__ views_in, float tau_f, int n_hyp, uint32_t seed, int cap,
           float4* __restrict__ list_x, float2* __restrict__ list_uv, gs_view* __restrict__ views_out,
           gs_pnp_stats* __restrict__ stats) {
    __shared__ int s_n;
    __shared__ int wsum[PNP_THREADS / 32];
    __shared__ Pose s_pose;
    __shared__ Pose s_hyp[MAX_HYP + 1];
    __shared__ int s_cnt[MAX_HYP + 1];
    __shared__ double red[PNP_THREADS / 32][28];
    __shared__ int s_stop;
    __shared__ int s_stride;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t HW = (int64_t)H * W;
    const gs_view V = views_in[b];
    const float4 K = make_float4(V.fx, V.fy, V.cx, V.cy);
    const double tau = tau_f;
    float4* LX = list_x + (int64_t)b * cap;
    float2* LU = list_uv + (int64_t)b * cap;
    // ---------------------------------------------------------- 1. compaction
    if (tid == 0) {
        s_n = 0;
        for (int i = 0; i < 9; ++i) s_pose.R[i] = V.R[i];
        for (int i = 0; i < 3; ++i) s_pose.t[i] = V.t[i];
    }
    __syncthreads();
    const uint8_t* vb = valid + (int64_t)b * HW;
    const float* X = xyz + (int64_t)b * 3 * HW;
    // pass 1: number of valid correspondences; keep every k-th (k = ceil(n / cap)) so a
    // capped list still spans the whole image
    {
        int cnt = 0;
        for (int64_t p = 4 * tid; p < HW; p += 4 * PNP_THREADS)
#pragma unroll
            for (int k = 0; k < 4; ++k) cnt += (p + k < HW && vb[p + k]) ? 1 : 0;
        cnt = (int)warp_sum((double)cnt);
        if (lane == 0) wsum[warp] = cnt;
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < PNP_THREADS / 32; ++w) tot += wsum[w];
            s_stride = (tot + cap - 1) / cap;
            if (s_stride < 1) s_stride = 1;
        }
        __syncthreads();
    }
    const int stride = s_stride;
    const bool vec = ((uintptr_t)vb & 15) == 0;
    for (int64_t p0 = 0; p0 < HW; p0 += 16 * PNP_THREADS) {
        const int64_t p = p0 + 16 * tid;
        uint32_t f[16];
        if (vec && p + 16 <= HW) {
            const uint4 q = *reinterpret_cast<const uint4*>(vb + p);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) f[k] = ((w[k >> 2] >> (8 * (k & 3))) & 0xffu) ? 1u : 0u;
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) f[k] = (p + k < HW && vb[p + k]) ? 1u : 0u;
        }
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) c += f[k];
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[warp] = (int)inc;
        __syncthreads();
        const int base = s_n;
        int off = 0;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        int pos = base + off + (int)(inc - c);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (f[k]) {
                if (pos % stride == 0 && pos / stride < cap) {
                    const int64_t q = p + k;
                    LX[pos / stride] = make_float4(X[q], X[HW + q], X[2 * HW + q], 0.f);
                    LU[pos / stride] = make_float2((float)(q % W), (float)(q / W));
                }
                ++pos;
            }
        }
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < PNP_THREADS / 32; ++w) tot += wsum[w];
            s_n = base + tot;
        }
        __syncthreads();
    }
    const int n = min((s_n + stride - 1) / stride, cap);
    // ---------------------------------------------------------- 2./3. hypotheses
    if (tid < n_hyp) {
        Pose P = s_pose;
        bool ok = n >= 3;
        int idx[3] = {0, 0, 0};
        if (ok) {
            int got = 0;
            for (uint32_t k = 0; k < 32 && got < 3; ++k) {
                const int i = (int)(sample_hash(seed, (uint32_t)tid, k) % (uint32_t)n);
                bool dup = false;
                for (int q = 0; q < got; ++q) dup |= idx[q] == i;
                if (!dup) idx[got++] = i;
            }
            ok = got == 3;
        }
        for (int it = 0; ok && it < NEWTON_ITERS; ++it) {
            double A[36] = {0}, g[6] = {0};
            for (int q = 0; q < 3; ++q) {
                Obs o;
                const float4 x = LX[idx[q]];
                const float2 uv = LU[idx[q]];
                observe(P, K, uv.x, uv.y, x.x, x.y, x.z, o, true);
                if (!(o.z > 0.0)) ok = false;
                for (int r = 0; r < 2; ++r)
                    for (int i = 0; i < 6; ++i) {
                        g[i] += o.J[r][i] * o.r[r];
                        for (int j = 0; j < 6; ++j) A[i * 6 + j] += o.J[r][i] * o.J[r][j];
                    }
            }
            if (!ok) break;
            const double tr = (A[0] + A[7] + A[14] + A[21] + A[28] + A[35]) / 6.0;
            for (int i = 0; i < 6; ++i) A[i * 7] += 1e-12 * tr;
            double xi[6];
            const double nb[6] = {-g[0], -g[1], -g[2], -g[3], -g[4], -g[5]};
            if (!chol_solve(A, nb, xi)) { ok = false; break; }
            apply(P, xi);
        }
        s_hyp[tid] = P;
        s_cnt[tid] = ok ? 0 : -1;
    }
    if (tid == 0) s_hyp[n_hyp] = s_pose;   // the start pose is scored alongside
    __syncthreads();
    // 3. inlier counts, one warp per hypothesis at a time, lanes over the points; fp32
    //    without division: e^2 <= tau^2 <=> (fx x + (cx - u) z)^2 + (fy y + (cy - v) z)^2 <= tau^2 z^2
    for (int h = warp; h <= n_hyp; h += PNP_THREADS / 32) {
        if (h < n_hyp && s_cnt[h] < 0) continue;
        const Pose& Q = s_hyp[h];
        float R[9], t[3];
        for (int k = 0; k < 9; ++k) R[k] = (float)Q.R[k];
        for (int k = 0; k < 3; ++k) t[k] = (float)Q.t[k];
        const float tau2 = tau_f * tau_f;
        int c = 0;
        for (int i = lane; i < n; i += 32) {
            const float4 x = LX[i];
            const float2 uv = LU[i];
            const float px = fmaf(R[0], x.x, fmaf(R[1], x.y, fmaf(R[2], x.z, t[0])));
            const float py = fmaf(R[3], x.x, fmaf(R[4], x.y, fmaf(R[5], x.z, t[1])));
            const float pz = fmaf(R[6], x.x, fmaf(R[7], x.y, fmaf(R[8], x.z, t[2])));
            const float ex = fmaf(K.x, px, (K.z - uv.x) * pz), ey = fmaf(K.y, py, (K.w - uv.y) * pz);
            c += (pz > 0.f && ex * ex + ey * ey <= tau2 * pz * pz) ? 1 : 0;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) s_cnt[h] = c;
    }
    __syncthreads();
    if (tid == 0) {
        // the start pose unless a hypothesis has strictly more inliers (lowest index on ties)
        int best_cnt = s_cnt[n_hyp];
        int best = -1;
        for (int h = 0; h < n_hyp; ++h)
            if (s_cnt[h] > best_cnt) { best_cnt = s_cnt[h]; best = h; }
        if (best >= 0) s_pose = s_hyp[best];
        stats[b].best_hypothesis = best;
        s_stop = n < 3;
    }
    __syncthreads();
    // ---------------------------------------------------------- 4. refinement
    for (int it = 0; it < REFINE_ITERS && !s_stop; ++it) {
        double acc[28];
#pragma unroll
        for (int k = 0; k < 28; ++k) acc[k] = 0.0;
        const Pose P = s_pose;
        for (int i = tid; i < n; i += PNP_THREADS) {
            Obs o;
            observe(P, K, LU[i].x, LU[i].y, LX[i].x, LX[i].y, LX[i].z, o, true);
            if (!is_inlier(o, tau)) continue;
            int k = 0;
            for (int a = 0; a < 6; ++a)
                for (int c = a; c < 6; ++c) acc[k++] += o.J[0][a] * o.J[0][c] + o.J[1][a] * o.J[1][c];
            for (int a = 0; a < 6; ++a) acc[21 + a] += o.J[0][a] * o.r[0] + o.J[1][a] * o.r[1];
            acc[27] += 1.0;
        }
#pragma unroll
        for (int k = 0; k < 28; ++k) acc[k] = warp_sum(acc[k]);
        if (lane == 0)
            for (int k = 0; k < 28; ++k) red[warp][k] = acc[k];
        __syncthreads();
        if (tid == 0) {
            double t[28];
            for (int k = 0; k < 28; ++k) {
                t[k] = 0.0;
                for (int w = 0; w < PNP_THREADS / 32; ++w) t[k] += red[w][k];
            }
            if (t[27] < 3.0) {
                s_stop = 1;
            } else {
                double A[36];
                int k = 0;
                for (int a = 0; a < 6; ++a)
                    for (int c = a; c < 6; ++c) { A[a * 6 + c] = t[k]; A[c * 6 + a] = t[k]; ++k; }
                const double tr = (A[0] + A[7] + A[14] + A[21] + A[28] + A[35]) / 6.0;
                for (int i = 0; i < 6; ++i) A[i * 7] += DAMPING * tr;
                const double nb[6] = {-t[21], -t[22], -t[23], -t[24], -t[25], -t[26]};
                double xi[6];
                if (chol_solve(A, nb, xi)) apply(s_pose, xi);
                else s_stop = 1;
            }
        }
        __syncthreads();
    }
    // ---------------------------------------------------------- 5. outputs
    int ni = 0;
    double es = 0.0;
    const Pose P = s_pose;
    for (int i = tid; i < n; i += PNP_THREADS) {
        Obs o;
        observe(P, K, LU[i].x, LU[i].y, LX[i].x, LX[i].y, LX[i].z, o, false);
        if (is_inlier(o, tau)) {
            ++ni;
            es += sqrt(o.r[0] * o.r[0] + o.r[1] * o.r[1]);
        }
    }
    const double nid = warp_sum((double)ni), esd = warp_sum(es);
    if (lane == 0) { red[warp][0] = nid; red[warp][1] = esd; }
    __syncthreads();
    if (tid == 0) {
        double tn = 0, te = 0;
        for (int w = 0; w < PNP_THREADS / 32; ++w) { tn += red[w][0]; te += red[w][1]; }
        gs_view out = V;
        for (int i = 0; i < 9; ++i) out.R[i] = (float)P.R[i];
        for (int i = 0; i < 3; ++i) out.t[i] = (float)P.t[i];
        views_out[b] = out;
        stats[b].n_corr = n;
        stats[b].n_inliers = (int)tn;
        stats[b].mean_err = tn > 0 ? (float)(te / tn) : 0.f;
    }
}

// Algorithm 2: per problem, angle / translation between consecutive poses of the trace
__global__ void consistency_kernel(const gs_view* __restrict__ trace, int n_iters, int n_problems, float tau_deg,
                                   float* __restrict__ angle_deg, float* __restrict__ dtrans,
                                   int32_t* __restrict__ verdict) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n_problems) return;
    int v = n_iters < 2 ? -2 : -1;
    for (int i = 0; i + 1 < n_iters; ++i) {
        const gs_view& A = trace[(int64_t)i * n_problems + b];
        const gs_view& B = trace[(int64_t)(i + 1) * n_problems + b];
        double tr = 0.0;   // trace(R_A R_B^T) = sum_ij A_ij B_ij
        for (int k = 0; k < 9; ++k) tr += (double)A.R[k] * (double)B.R[k];
        tr = fmin(3.0, fmax(tr, -1.0));
        const double th = acos((tr - 1.0) / 2.0) * (180.0 / 3.14159265358979323846);
        const double dx = A.t[0] - B.t[0], dy = A.t[1] - B.t[1], dz = A.t[2] - B.t[2];
        angle_deg[(int64_t)b * (n_iters - 1) + i] = (float)th;
        dtrans[(int64_t)b * (n_iters - 1) + i] = (float)sqrt(dx * dx + dy * dy + dz * dz);
        if (v == -1 && th > tau_deg) v = i;
    }
    verdict[b] = v;
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" size_t gs_pnp_workspace_bytes(int32_t n_problems, int32_t cap) {
    if (n_problems < 1 || cap < 1) return 0;
    return (size_t)n_problems * cap * (sizeof(float4) + sizeof(float2)) + 256;
}

extern "C" gs_status gs_pnp(const uint8_t* valid, const float* xyz, int32_t n_problems, int32_t H, int32_t W,
                            const gs_view* views_in_dev, float tau_px, int32_t n_hyp, uint32_t seed, int32_t cap,
                            void* ws, size_t ws_bytes, gs_view* views_out_dev, gs_pnp_stats* stats_dev,
                            void* stream) {
    GS_REQUIRE(valid && xyz && views_in_dev && views_out_dev && stats_dev, GS_INVALID_ARG, "gs_pnp: NULL pointer");
    GS_REQUIRE(n_problems >= 1 && H >= 1 && W >= 1, GS_INVALID_ARG, "gs_pnp: bad sizes");
    GS_REQUIRE(n_hyp >= 0 && n_hyp <= MAX_HYP, GS_UNSUPPORTED, "gs_pnp: n_hyp = %d (0..%d)", n_hyp, MAX_HYP);
    GS_REQUIRE(cap >= 3, GS_INVALID_ARG, "gs_pnp: cap = %d < 3", cap);
    GS_REQUIRE(tau_px > 0.f && std::isfinite(tau_px), GS_INVALID_ARG, "gs_pnp: tau = %g", (double)tau_px);
    GS_REQUIRE(views_in_dev != views_out_dev, GS_INVALID_ARG, "gs_pnp: views_in and views_out must not alias");
    const size_t need = gs_pnp_workspace_bytes(n_problems, cap);
    GS_REQUIRE(ws != nullptr && ws_bytes >= need && ((uintptr_t)ws & 15) == 0, GS_WORKSPACE_TOO_SMALL,
               "gs_pnp workspace %zu < %zu (or misaligned)", ws_bytes, need);
    float4* lx = static_cast<float4*>(ws);
    float2* lu = reinterpret_cast<float2*>(lx + (size_t)n_problems * cap);
    pnp_kernel<<<n_problems, PNP_THREADS, 0, (cudaStream_t)stream>>>(valid, xyz, H, W, views_in_dev, tau_px, n_hyp,
                                                                      seed, cap, lx, lu, views_out_dev, stats_dev);
    return check_launch("pnp_kernel");
}

extern "C" gs_status gs_verify_consistency(const gs_view* trace_dev, int32_t n_iters, int32_t n_problems,
                                           float tau_deg, float* angle_deg, float* dtrans, int32_t* verdict,
                                           void* stream) {
    GS_REQUIRE(trace_dev && verdict && (n_iters < 2 || (angle_deg && dtrans)), GS_INVALID_ARG,
               "gs_verify_consistency: NULL pointer");
    GS_REQUIRE(n_iters >= 1 && n_problems >= 1, GS_INVALID_ARG, "gs_verify_consistency: bad sizes");
    consistency_kernel<<<(n_problems + 127) / 128, 128, 0, (cudaStream_t)stream>>>(trace_dev, n_iters, n_problems,
                                                                                  tau_deg, angle_deg, dtrans, verdict);
    return check_launch("consistency_kernel");
}
