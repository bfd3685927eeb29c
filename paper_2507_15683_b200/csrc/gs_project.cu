// gs_project.cu -- O1-O10: per (view, Gaussian) camera
// transform, cull, EWA 2D covariance, conic, radius, tile rectangle, depth
// key and SH colour.  PAPER.md Alg. 1 l.9-12.
//
// THIS TRANSLATION UNIT IS COMPILED WITH -fmad=false (no FMA contraction),
// IEEE division and square root, no flush-to-zero: every fp32 expression in
// the "pinned" sections below is evaluated exactly in the written order, so
// u, v, z, conic, radius and the tile rectangle are bit-identical to the
// oracle's (and hence so are the duplicated keys).
//
// Design (B200): one thread per Gaussian reads its 44 B of geometry ONCE per
// batch (coalesced SoA loads), builds the view-independent 3D covariance once,
// then loops over the views of the batch that can see its block (a
// conservative per-(view, block) frustum test fills a bitmask first).  The
// view loop is warp-uniform, so record slots are reserved with one atomic per
// warp per view.  SH coefficients are read only for visible records.
#include "gs_common.cuh"

namespace gs {
namespace {

// reading Q29: k = -log2(e)/2 as the nearest fp32 (same literal as the oracle's)
constexpr float K_EXP2 = -0.72134752044448170368f;

struct ViewConst {        // per-view constants (pinned fp32, computed once per batch)
    float lox, hix, loy, hiy;   // Jacobian clamp bounds on x/z, y/z (Q6)
    float ccx, ccy, ccz;        // camera centre in world, -R^T t (SH direction)
    float kbound;               // fx^2 (1 + tx^2) + fy^2 (1 + ty^2): ||J||_F^2 z^2 bound
    float wpix, hpix;           // 16*TX, 16*TY (grid extent in pixels)
    float txf, tyf;             // TX, TY as float
    int32_t tx, ty;
    int32_t pad0, pad1;
};

__global__ void view_const_kernel(const gs_view* __restrict__ views, int n_views, gs_params P,
                                  ViewConst* __restrict__ vc) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_views) return;
    const gs_view V = views[i];
    ViewConst c;
    const float W = (float)V.width, H = (float)V.height;
    const float m = P.clamp_margin;
    // pinned (same expressions as the oracle)
    c.lox = (-(m * W) - V.cx) / V.fx;
    c.hix = ((1.0f + m) * W - V.cx) / V.fx;
    c.loy = (-(m * H) - V.cy) / V.fy;
    c.hiy = ((1.0f + m) * H - V.cy) / V.fy;
    // not pinned (tolerance / conservative bound only)
    c.ccx = -(V.R[0] * V.t[0] + V.R[3] * V.t[1] + V.R[6] * V.t[2]);
    c.ccy = -(V.R[1] * V.t[0] + V.R[4] * V.t[1] + V.R[7] * V.t[2]);
    c.ccz = -(V.R[2] * V.t[0] + V.R[5] * V.t[1] + V.R[8] * V.t[2]);
    const float txm = fmaxf(fabsf(c.lox), fabsf(c.hix)), tym = fmaxf(fabsf(c.loy), fabsf(c.hiy));
    c.kbound = V.fx * V.fx * (1.0f + txm * txm) + V.fy * V.fy * (1.0f + tym * tym);
    c.tx = (V.width + GS_TILE - 1) / GS_TILE;
    c.ty = (V.height + GS_TILE - 1) / GS_TILE;
    c.txf = (float)c.tx;
    c.tyf = (float)c.ty;
    c.wpix = 16.0f * c.txf;
    c.hpix = 16.0f * c.tyf;
    c.pad0 = c.pad1 = 0;
    vc[i] = c;
}

// Conservative radius bound (px) for a Gaussian with max scale smax at depth z:
// lambda_max(Sigma') <= smax^2 ||J||_F^2 + dilation, ||J||_F^2 <= kbound / z^2
// (DESIGN.md §4.1).  Inflated to absorb fp32 rounding.
__device__ __forceinline__ float radius_bound(float smax, float kbound, float z, float dil) {
    const float lam = smax * smax * kbound / (z * z) + dil;
    return 3.0f * sqrtf(lam) * 1.01f + 2.0f;
}

// The same bound with MUFU reciprocal / reciprocal square root instead of the IEEE
// division and square root of this -prec-div / -prec-sqrt translation unit: a few ulp
// on a bound that is already inflated by 1 % + 2 px (the cheap per-(view, Gaussian)
// test runs ~10^9 times per C5 batch).
__device__ __forceinline__ float radius_bound_fast(float smax, float kbound, float z, float dil) {
    const float lam = __fdividef(smax * smax * kbound, z * z) + dil;
    return 3.0f * (lam * rsqrtf(lam)) * 1.01f + 2.0f;
}

// One thread per (block, 32-view word): bit set unless the whole block is
// provably culled (all centres behind z_near, or every Gaussian's rectangle
// provably off the tile grid).  Conservative: never clears a needed bit.
__global__ void block_cull_kernel(const gs_view* __restrict__ views, const ViewConst* __restrict__ vcs,
                                  int n_views, int n_blocks, const float* __restrict__ bounds, gs_params P,
                                  uint32_t* __restrict__ mask) {
    const int nw = (n_views + 31) >> 5;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n_blocks * nw) return;
    const int b = (int)(idx / nw), w = (int)(idx % nw);
    const float* bb = bounds + (int64_t)b * 8;
    const float lo[3] = {bb[0], bb[1], bb[2]}, hi[3] = {bb[3], bb[4], bb[5]};
    const float smax = bb[6];
    uint32_t word = 0;
    const bool empty = !(lo[0] <= hi[0]);   // empty block: bounds are +inf/-inf
    for (int j = 0; j < 32; ++j) {
        const int v = w * 32 + j;
        if (v >= n_views || empty) break;
        const gs_view& V = views[v];
        const ViewConst& c = vcs[v];
        float zmin = 3.4e38f, zmax = -3.4e38f, umin = 3.4e38f, umax = -3.4e38f, vmin = 3.4e38f, vmax = -3.4e38f;
        float slack = 0.f;
        bool all_front = true;
        for (int k = 0; k < 8; ++k) {
            const float x = (k & 1) ? hi[0] : lo[0], y = (k & 2) ? hi[1] : lo[1], z = (k & 4) ? hi[2] : lo[2];
            const float pz = V.R[6] * x + V.R[7] * y + V.R[8] * z + V.t[2];
            const float mag = fabsf(V.R[6] * x) + fabsf(V.R[7] * y) + fabsf(V.R[8] * z) + fabsf(V.t[2]);
            slack = fmaxf(slack, 1e-5f * mag + 1e-6f);
            zmin = fminf(zmin, pz);
            zmax = fmaxf(zmax, pz);
            if (!(pz > P.z_near + 2.0f * slack)) { all_front = false; continue; }
            const float px = V.R[0] * x + V.R[1] * y + V.R[2] * z + V.t[0];
            const float py = V.R[3] * x + V.R[4] * y + V.R[5] * z + V.t[1];
            const float u = V.fx * (px / pz) + V.cx, vv = V.fy * (py / pz) + V.cy;
            umin = fminf(umin, u); umax = fmaxf(umax, u);
            vmin = fminf(vmin, vv); vmax = fmaxf(vmax, vv);
        }
        bool visible = true;
        if (zmax < P.z_near - 2.0f * slack) {
            visible = false;                                   // every centre is near-culled
        } else if (all_front) {
            // projection of the box = hull of corner projections (z > 0 everywhere)
            const float rb = radius_bound(smax, c.kbound, zmin, P.dilation);
            const float mu = 1e-4f * (fabsf(umin) + fabsf(umax) + fabsf(vmin) + fabsf(vmax)) + 1.0f;
            if (umax + rb < -mu || umin - rb >= c.wpix + mu || vmax + rb < -mu || vmin - rb >= c.hpix + mu)
                visible = false;
        }
        if (visible) word |= 1u << j;
    }
    mask[idx] = word;
}

__global__ void block_bounds_kernel(const float* __restrict__ pos, const float* __restrict__ scale, int64_t n,
                                    const int64_t* __restrict__ offs, int n_blocks, float* __restrict__ out) {
    const int b = blockIdx.x;
    if (b >= n_blocks) return;
    const int64_t s = offs[b], e = offs[b + 1];
    float lo[3] = {3.4e38f, 3.4e38f, 3.4e38f}, hi[3] = {-3.4e38f, -3.4e38f, -3.4e38f}, sm = 0.f;
    for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) {
        for (int k = 0; k < 3; ++k) {
            const float p = pos[k * n + i];
            lo[k] = fminf(lo[k], p);
            hi[k] = fmaxf(hi[k], p);
            sm = fmaxf(sm, scale[k * n + i]);
        }
    }
    __shared__ float red[7][32];
    float vals[7] = {lo[0], lo[1], lo[2], -hi[0], -hi[1], -hi[2], -sm};
    for (int k = 0; k < 7; ++k) {
        float x = vals[k];
        for (int o = 16; o; o >>= 1) x = fminf(x, __shfl_xor_sync(0xffffffffu, x, o));
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        float x = 3.4e38f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x = fminf(x, red[threadIdx.x][w]);
        out[(int64_t)b * 8 + threadIdx.x] = threadIdx.x < 3 ? x : -x;
    }
    if (threadIdx.x == 7) out[(int64_t)b * 8 + 7] = 0.f;
}

__device__ __forceinline__ bool finite3(float a, float b, float c) {
    return isfinite(a) && isfinite(b) && isfinite(c);
}

// SH colour (O10, fp32, tolerance-checked): [3DGS] real SH basis up to degree 3.
// Coefficient k of channel c is coef[(k * 3 + c) * stride] (global SoA plane: stride
// n; the warp's shared-memory copy: stride 32).
__device__ __forceinline__ void sh_color(int deg, const float* __restrict__ coef, int64_t stride, float dx,
                                         float dy, float dz, float* rgb) {
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    float b[16];
    b[0] = C0;
    int nk = 1;
    if (deg >= 1) {
        b[1] = -C1 * dy; b[2] = C1 * dz; b[3] = -C1 * dx;
        nk = 4;
    }
    if (deg >= 2) {
        const float xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yz = dy * dz, xz = dx * dz;
        b[4] = 1.0925484305920792f * xy;
        b[5] = -1.0925484305920792f * yz;
        b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
        b[7] = -1.0925484305920792f * xz;
        b[8] = 0.5462742152960396f * (xx - yy);
        nk = 9;
        if (deg >= 3) {
            b[9] = -0.5900435899266435f * dy * (3.0f * xx - yy);
            b[10] = 2.890611442640554f * xy * dz;
            b[11] = -0.4570457994644658f * dy * (4.0f * zz - xx - yy);
            b[12] = 0.3731763325901154f * dz * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            b[13] = -0.4570457994644658f * dx * (4.0f * zz - xx - yy);
            b[14] = 1.445305721320277f * dz * (xx - yy);
            b[15] = -0.5900435899266435f * dx * (xx - 3.0f * yy);
            nk = 16;
        }
    }
    float r = 0.5f, g = 0.5f, bl = 0.5f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        if (k < nk) {
            // fused (the file is built with -fmad=false for the pinned geometry; the colour
            // decides nothing and is tolerance-checked, so it may use FMAs)
            r = __fmaf_rn(b[k], coef[(int64_t)(k * 3 + 0) * stride], r);
            g = __fmaf_rn(b[k], coef[(int64_t)(k * 3 + 1) * stride], g);
            bl = __fmaf_rn(b[k], coef[(int64_t)(k * 3 + 2) * stride], bl);
        }
    }
    rgb[0] = fmaxf(r, 0.f);
    rgb[1] = fmaxf(g, 0.f);
    rgb[2] = fmaxf(bl, 0.f);
}

constexpr int PROJ_THREADS = 256;

// a queued Gaussian's view-independent state (per-warp table, one row per lane)
struct GTab {
    float mx, my, mz, op;
    float sg[6];
    float smax, ecut;
    uint32_t gid, pad;
};

// r2: each warp copies its 32 Gaussians' SH coefficients into shared memory once
// (coalesced rows) instead of every queued (view, Gaussian) pair re-reading 48
// scattered coefficients from L2 -- the per-pair SH reads were a third of the stage
#ifndef GS_PROJ_SH_SMEM
#define GS_PROJ_SH_SMEM 1
#endif
#ifndef GS_PROJ_MIN_BLOCKS
#define GS_PROJ_MIN_BLOCKS (GS_PROJ_SH_SMEM ? 3 : 4)
#endif
__global__ void __launch_bounds__(PROJ_THREADS, GS_PROJ_MIN_BLOCKS)
project_kernel(gs_scene S, const gs_view* __restrict__ views, const ViewConst* __restrict__ vcs, int n_views,
               gs_params P, const uint32_t* __restrict__ mask, gs_record* __restrict__ rec, int64_t cap,
               uint32_t* __restrict__ n_rec, uint64_t* __restrict__ diag, uint32_t* __restrict__ status) {
    __shared__ GTab s_tab[PROJ_THREADS / 32][32];
    __shared__ uint32_t s_queue[PROJ_THREADS / 32][64];
    const int64_t n = S.n;
    const int64_t i = (int64_t)blockIdx.x * PROJ_THREADS + threadIdx.x;
    const bool in = i < n;
    const uint32_t lane = threadIdx.x & 31u;
    const int nw = (n_views + 31) >> 5;

    // ---- view-independent part (once per Gaussian per batch) ----
    float mx = 0.f, my = 0.f, mz = 0.f, op = 0.f, s0 = 1.f, s1 = 1.f, s2 = 1.f;
    float qw = 1.f, qx = 0.f, qy = 0.f, qz = 0.f;
    if (in) {
        mx = __ldg(&S.pos[i]); my = __ldg(&S.pos[n + i]); mz = __ldg(&S.pos[2 * n + i]);
        op = __ldg(&S.opacity[i]);
        s0 = __ldg(&S.scale[i]); s1 = __ldg(&S.scale[n + i]); s2 = __ldg(&S.scale[2 * n + i]);
        qw = __ldg(&S.quat[i]); qx = __ldg(&S.quat[n + i]); qy = __ldg(&S.quat[2 * n + i]);
        qz = __ldg(&S.quat[3 * n + i]);
    }
    const bool transparent = !(op >= P.alpha_min);
    bool degenerate = !(s0 > 0.0f) || !(s1 > 0.0f) || !(s2 > 0.0f) || !finite3(s0, s1, s2) ||
                      !finite3(qw, qx, qy) || !isfinite(qz);
    // O4 (pinned): Sigma = M M^T, M = R(q) diag(s), q normalised
    float Sg[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // S00 S01 S02 S11 S12 S22
    {
        const float qn2 = ((qw * qw + qx * qx) + qy * qy) + qz * qz;
        bool qbad = !(qn2 > 0.0f);
        if (!degenerate && !qbad) {
            const float qn = sqrtf(qn2);
            const float w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
            const float xx = x * x, yy = y * y, zz = z * z;
            const float xy = x * y, xz = x * z, yz = y * z;
            const float wx = w * x, wy = w * y, wz = w * z;
            const float M0 = (1.0f - 2.0f * (yy + zz)) * s0, M1 = (2.0f * (xy - wz)) * s1, M2 = (2.0f * (xz + wy)) * s2;
            const float M3 = (2.0f * (xy + wz)) * s0, M4 = (1.0f - 2.0f * (xx + zz)) * s1, M5 = (2.0f * (yz - wx)) * s2;
            const float M6 = (2.0f * (xz - wy)) * s0, M7 = (2.0f * (yz + wx)) * s1, M8 = (1.0f - 2.0f * (xx + yy)) * s2;
            Sg[0] = (M0 * M0 + M1 * M1) + M2 * M2;
            Sg[1] = (M0 * M3 + M1 * M4) + M2 * M5;
            Sg[2] = (M0 * M6 + M1 * M7) + M2 * M8;
            Sg[3] = (M3 * M3 + M4 * M4) + M5 * M5;
            Sg[4] = (M3 * M6 + M4 * M7) + M5 * M8;
            Sg[5] = (M6 * M6 + M7 * M7) + M8 * M8;
        }
        // a zero/non-finite quaternion is degenerate, but only after the near /
        // transparent tests (oracle order)
        if (qbad) degenerate = true;
    }
    const float smax = fmaxf(fmaxf(s0, s1), s2);
    // block of this Gaussian: one binary search per CTA (its first Gaussian), then a short
    // forward scan per thread (a CTA's 256 consecutive Gaussians span one or two blocks)
    int blk = -1;
    if (S.n_blocks > 0) {
        __shared__ int s_blk0;
        if (threadIdx.x == 0) {
            const int64_t i0 = min((int64_t)blockIdx.x * PROJ_THREADS, n - 1);
            int lo = 0, hi = S.n_blocks - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (__ldg(&S.block_offsets[mid]) <= i0) lo = mid; else hi = mid - 1;
            }
            s_blk0 = lo;
        }
        __syncthreads();
        if (in) {
            int lo = s_blk0;
            while (lo + 1 < S.n_blocks && __ldg(&S.block_offsets[lo + 1]) <= i) ++lo;
            blk = lo;
        }
    }
    uint32_t c_near = 0, c_transp = 0, c_degen = 0, c_off = 0;
    // reading Q30: alpha >= alpha_min cut in log2 units from exactly-rounded operations
    // (identical to the oracle's e_cut_of): x = o / alpha_min = m 2^k, m in [1, 2);
    // log2(x) <= k + (m - 0.9135) (tangent of the concave log2 at 1/ln 2), inflated
    // by 5% + 0.0075 so the cull and the tight binning stay conservative
    float e_cut = 0.f;
    if (in && !transparent) {
        const float x = op / P.alpha_min;
        const uint32_t xb = __float_as_uint(x);
        const int k = (int)((xb >> 23) & 0xffu) - 127;
        const float m = __uint_as_float((xb & 0x7fffffu) | 0x3f800000u);
        const float lub = (float)k + (m - 0.9135f);
        e_cut = -(lub * 1.05f + 0.0075f);
    }

    // Per-warp candidate queue: the cheap per-view tests run in the warp-uniform view
    // loop; surviving (Gaussian, view) pairs are queued and the heavy EWA + SH path runs
    // 32 of them at a time with every lane busy (a view typically keeps a few percent
    // of a warp's Gaussians, so running it in place idles most lanes).
    const int wid = threadIdx.x >> 5;
#if GS_PROJ_SH_SMEM
    extern __shared__ float s_sh[];   // [warp][(deg+1)^2 * 3][32]
    const int nk3 = (S.sh_degree + 1) * (S.sh_degree + 1) * 3;
    float* my_sh = s_sh + (int64_t)wid * nk3 * 32;
    bool sh_staged = false;           // warp-uniform
#endif
    GTab& me = s_tab[wid][lane];
    me.mx = mx; me.my = my; me.mz = mz; me.op = op;
    for (int k = 0; k < 6; ++k) me.sg[k] = Sg[k];
    me.smax = smax; me.ecut = e_cut; me.gid = (uint32_t)i;
    uint32_t* queue = s_queue[wid];
    uint32_t qn = 0;   // warp-uniform
    __syncwarp();

    // heavy path for queue items [0, cnt): lane k takes item k
    auto process = [&](uint32_t cnt) {
#if GS_PROJ_SH_SMEM
        if (!sh_staged) {   // first visible pair of this warp: stage its Gaussians' SH rows
            for (int q = 0; q < nk3; ++q) my_sh[q * 32 + lane] = in ? __ldg(&S.sh[(int64_t)q * n + i]) : 0.f;
            __syncwarp();
            sh_staged = true;
        }
#endif
        const bool act = lane < cnt;
        const uint32_t item = act ? queue[lane] : 0u;
        const int vi = (int)(item >> 5);
        const GTab& g = s_tab[wid][item & 31u];
        bool visible = false;
        gs_record r;
        if (act) {
            const gs_view& V = views[vi];
            const ViewConst& c = vcs[vi];
            // O1 (pinned), recomputed
            const float px = ((V.R[0] * g.mx + V.R[1] * g.my) + V.R[2] * g.mz) + V.t[0];
            const float py = ((V.R[3] * g.mx + V.R[4] * g.my) + V.R[5] * g.mz) + V.t[1];
            const float pz = ((V.R[6] * g.mx + V.R[7] * g.my) + V.R[8] * g.mz) + V.t[2];
            // O3 (pinned): divide by depth first, then apply K (Alg. 1 l.12-14)
            const float xn = px / pz, yn = py / pz;
            const float u = V.fx * xn + V.cx;
            const float v = V.fy * yn + V.cy;
            // O5 (pinned): EWA with the clamped Jacobian
            const float xc = fminf(fmaxf(xn, c.lox), c.hix) * pz;
            const float yc = fminf(fmaxf(yn, c.loy), c.hiy) * pz;
            const float z2 = pz * pz;
            const float j00 = V.fx / pz, j02 = -((V.fx * xc) / z2);
            const float j11 = V.fy / pz, j12 = -((V.fy * yc) / z2);
            float T0[3], T1[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                T0[k] = j00 * V.R[0 * 3 + k] + j02 * V.R[2 * 3 + k];
                T1[k] = j11 * V.R[1 * 3 + k] + j12 * V.R[2 * 3 + k];
            }
            const float S00 = g.sg[0], S01 = g.sg[1], S02 = g.sg[2], S11 = g.sg[3], S12 = g.sg[4], S22 = g.sg[5];
            const float V00 = (T0[0] * S00 + T0[1] * S01) + T0[2] * S02;
            const float V01 = (T0[0] * S01 + T0[1] * S11) + T0[2] * S12;
            const float V02 = (T0[0] * S02 + T0[1] * S12) + T0[2] * S22;
            const float V10 = (T1[0] * S00 + T1[1] * S01) + T1[2] * S02;
            const float V11 = (T1[0] * S01 + T1[1] * S11) + T1[2] * S12;
            const float V12 = (T1[0] * S02 + T1[1] * S12) + T1[2] * S22;
            const float s00 = (V00 * T0[0] + V01 * T0[1]) + V02 * T0[2];
            const float s01 = (V00 * T1[0] + V01 * T1[1]) + V02 * T1[2];
            const float s11 = (V10 * T1[0] + V11 * T1[1]) + V12 * T1[2];
            const float a = s00 + P.dilation, b = s01, cc = s11 + P.dilation;
            // O6 (pinned)
            const float det = a * cc - b * b;
            if (!(det > 0.0f)) { ++c_degen; goto done; }
            {
                const float ca = cc / det, cb = -(b / det), ccn = a / det;
                // O7 (pinned)
                const float mid = 0.5f * (a + cc);
                const float lam = mid + sqrtf(fmaxf(mid * mid - det, 0.0f));
                const float rad = ceilf(3.0f * sqrtf(lam));
                // O8 (pinned)
                if (!isfinite(u) || !isfinite(v) || !isfinite(rad)) { ++c_degen; goto done; }
                const float fx0 = floorf((u - rad) * 0.0625f), fx1 = floorf((u + rad) * 0.0625f);
                const float fy0 = floorf((v - rad) * 0.0625f), fy1 = floorf((v + rad) * 0.0625f);
                if (fx1 < 0.0f || fx0 >= c.txf || fy1 < 0.0f || fy0 >= c.tyf) { ++c_off; goto done; }
                r.x0 = (uint16_t)fmaxf(fx0, 0.0f);
                r.x1 = (uint16_t)fminf(fx1, c.txf - 1.0f);
                r.y0 = (uint16_t)fmaxf(fy0, 0.0f);
                r.y1 = (uint16_t)fminf(fy1, c.tyf - 1.0f);
                r.u = u; r.v = v; r.z = pz;
                // exponent coefficients in log2 units (reading Q29): k = fp32(-log2(e)/2),
                // ea = k ca, eb = 2k cb, ec = k cc
                r.ea = K_EXP2 * ca; r.eb = (2.0f * K_EXP2) * cb; r.ec = K_EXP2 * ccn;
                r.opacity = g.op;
                // alpha >= alpha_min needs p(d) >= -log2(o / alpha_min) >= e_cut
                r.e_cut = g.ecut;
                r.tile_mask = GS_TILE_MASK_FULL;   // decided by gs_bin_sort (tight mode)
                r.gid = g.gid;
                r.view_radius = (uint32_t)vi | ((uint32_t)fminf(rad, 65535.0f) << 16);
                // O10: SH colour at d = (mu - c_cam)/|mu - c_cam|
                const float dx = g.mx - c.ccx, dy = g.my - c.ccy, dz = g.mz - c.ccz;
                const float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
#if GS_PROJ_SH_SMEM
                sh_color(S.sh_degree, my_sh + (item & 31u), 32, dx * inv, dy * inv, dz * inv, r.rgb);
#else
                sh_color(S.sh_degree, S.sh + g.gid, n, dx * inv, dy * inv, dz * inv, r.rgb);
#endif
                visible = true;
            }
        done:;
        }
        // slot reservation: one atomic per distinct view among the visible lanes
        const uint32_t vm = __ballot_sync(0xffffffffu, visible);
        if (visible) {
            const uint32_t grp = __match_any_sync(vm, vi);
            const uint32_t leader = __ffs(grp) - 1;
            uint32_t base = 0;
            if (lane == leader) base = atomicAdd(&n_rec[vi], (uint32_t)__popc(grp));
            base = __shfl_sync(grp, base, leader);
            const uint32_t slot = base + __popc(grp & ((1u << lane) - 1u));
            if ((int64_t)slot < cap) {
                float4* dst = reinterpret_cast<float4*>(rec + (int64_t)vi * cap + slot);
                const float4* src = reinterpret_cast<const float4*>(&r);
                dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2]; dst[3] = src[3];
            } else {
                atomicOr(status, GS_STATUS_RECORD_OVERFLOW);
            }
        }
        __syncwarp();
    };

    for (int w = 0; w < nw; ++w) {
        uint32_t my_mask = 0;
        if (in) {
            if (S.n_blocks > 0) my_mask = __ldg(&mask[(int64_t)blk * nw + w]);
            else my_mask = (w == nw - 1 && (n_views & 31)) ? ((1u << (n_views & 31)) - 1u) : 0xffffffffu;
        }
        uint32_t any = __reduce_or_sync(0xffffffffu, my_mask);
        while (any) {
            const int j = __ffs(any) - 1;
            any &= any - 1u;
            const int vi = w * 32 + j;
            bool cand = false;
            if ((my_mask >> j) & 1u) {
                const gs_view& V = views[vi];
                const ViewConst& c = vcs[vi];
                // O1 (pinned)
                const float px = ((V.R[0] * mx + V.R[1] * my) + V.R[2] * mz) + V.t[0];
                const float py = ((V.R[3] * mx + V.R[4] * my) + V.R[5] * mz) + V.t[1];
                const float pz = ((V.R[6] * mx + V.R[7] * my) + V.R[8] * mz) + V.t[2];
                if (!(pz > P.z_near)) { ++c_near; goto cheap_done; }
                if (transparent) { ++c_transp; goto cheap_done; }
                if (degenerate || !finite3(px, py, pz)) { ++c_degen; goto cheap_done; }
                {
                    // conservative early off-screen test (never culls a Gaussian the exact test
                    // keeps): an approximate u, v (MUFU reciprocal, relative error ~2^-22 of
                    // |u - cx|) is covered by the margin mu; the exact O3 runs in process()
                    const float iz = __fdividef(1.0f, pz);
                    const float u = V.fx * (px * iz) + V.cx;
                    const float v = V.fy * (py * iz) + V.cy;
                    if (isfinite(u) && isfinite(v) && P.dilation > 0.f) {
                        const float rb = radius_bound_fast(smax, c.kbound, pz, P.dilation);
                        const float mu = 1e-5f * (fabsf(u) + fabsf(v)) + 1.0f;
                        if (u + rb < -mu || u - rb >= c.wpix + mu || v + rb < -mu || v - rb >= c.hpix + mu) {
                            ++c_off;
                            goto cheap_done;
                        }
                    }
                    cand = true;
                }
            cheap_done:;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, cand);
            if (cand) queue[qn + __popc(bal & ((1u << lane) - 1u))] = lane | ((uint32_t)vi << 5);
            qn += __popc(bal);
            __syncwarp();
            if (qn >= 32) {
                process(32);
                if (lane < qn - 32) queue[lane] = queue[32 + lane];
                __syncwarp();
                qn -= 32;
            }
        }
    }
    if (qn > 0) process(qn);
    // diagnostics: warp-reduce then one atomic per counter per warp
    uint32_t cnt[4] = {c_near, c_transp, c_degen, c_off};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t s = __reduce_add_sync(0xffffffffu, cnt[k]);
        if (lane == 0 && s) atomicAdd((unsigned long long*)&diag[k], (unsigned long long)s);
    }
}

// ---------------------------------------------------------------- N4: projection backward
// dL/dmu for every record from its 2D gradients (gs_radiance_backward's grad_rec:
// u, v, ea, eb, ec, ..., z) through O1-O7: p = R mu + t; u, v
// pinhole; J(p) with the Q6 clamp; Sigma' = (J R) Sigma (J R)^T + dilation I;
// conic = (c, -b, a)/det; e = k conic.  fp64 (per-record work is small);
// accumulated into grad_pos [3][n] (the layout of gs_scene.pos) with atomics.
__global__ void mean_backward_kernel(gs_scene S, const gs_view* __restrict__ views, gs_params P,
                                     const gs_record* __restrict__ rec, int64_t cap,
                                     const uint32_t* __restrict__ n_rec, int n_views,
                                     const float* __restrict__ grad_rec, float* __restrict__ grad_pos) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= cap * n_views) return;
    const int vi = (int)(slot / cap);
    if ((uint32_t)(slot - (int64_t)vi * cap) >= min((uint64_t)n_rec[vi], (uint64_t)cap)) return;
    const float* gr = grad_rec + slot * 10;
    const double gu = gr[0], gv = gr[1], gea = gr[2], geb = gr[3], gec = gr[4], gz = gr[9];
    const gs_record& rc = rec[slot];
    // colour gradient through the SH view direction (zero for degree 0 or a clamped channel)
    double grgb[3];
    for (int c = 0; c < 3; ++c) grgb[c] = (S.sh_degree >= 1 && rc.rgb[c] > 0.0f) ? (double)gr[6 + c] : 0.0;
    if (gu == 0.0 && gv == 0.0 && gea == 0.0 && geb == 0.0 && gec == 0.0 && gz == 0.0 && grgb[0] == 0.0 &&
        grgb[1] == 0.0 && grgb[2] == 0.0)
        return;
    const int64_t n = S.n;
    const uint32_t g = rc.gid;
    const gs_view& V = views[vi];
    double R[9], t[3];
    for (int k = 0; k < 9; ++k) R[k] = V.R[k];
    for (int k = 0; k < 3; ++k) t[k] = V.t[k];
    const double mx = S.pos[g], my = S.pos[n + g], mz = S.pos[2 * n + g];
    const double px = R[0] * mx + R[1] * my + R[2] * mz + t[0];
    const double py = R[3] * mx + R[4] * my + R[5] * mz + t[1];
    const double pz = R[6] * mx + R[7] * my + R[8] * mz + t[2];
    // Sigma = M M^T, M = R(q) diag(s)
    double qw = S.quat[g], qx = S.quat[n + g], qy = S.quat[2 * n + g], qz = S.quat[3 * n + g];
    const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    qw /= qn; qx /= qn; qy /= qn; qz /= qn;
    const double s0 = S.scale[g], s1 = S.scale[n + g], s2 = S.scale[2 * n + g];
    const double Rq[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy),
                          2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx),
                          2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)};
    double M[9];
    for (int r = 0; r < 3; ++r) { M[r * 3] = Rq[r * 3] * s0; M[r * 3 + 1] = Rq[r * 3 + 1] * s1; M[r * 3 + 2] = Rq[r * 3 + 2] * s2; }
    double Sg[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) Sg[r * 3 + c] = M[r * 3] * M[c * 3] + M[r * 3 + 1] * M[c * 3 + 1] + M[r * 3 + 2] * M[c * 3 + 2];
    const double fx = V.fx, fy = V.fy, cx = V.cx, cy = V.cy, W = V.width, H = V.height, m = P.clamp_margin;
    const double lox = (-(m * W) - cx) / fx, hix = ((1.0 + m) * W - cx) / fx;
    const double loy = (-(m * H) - cy) / fy, hiy = ((1.0 + m) * H - cy) / fy;
    const double xn = px / pz, yn = py / pz;
    const double xcl = fmin(fmax(xn, lox), hix), ycl = fmin(fmax(yn, loy), hiy);
    const double j00 = fx / pz, j11 = fy / pz, j02 = -fx * xcl / pz, j12 = -fy * ycl / pz;
    double T0[3], T1[3], ST0[3], ST1[3];
    for (int k = 0; k < 3; ++k) { T0[k] = j00 * R[k] + j02 * R[6 + k]; T1[k] = j11 * R[3 + k] + j12 * R[6 + k]; }
    for (int r = 0; r < 3; ++r) {
        ST0[r] = Sg[r * 3] * T0[0] + Sg[r * 3 + 1] * T0[1] + Sg[r * 3 + 2] * T0[2];
        ST1[r] = Sg[r * 3] * T1[0] + Sg[r * 3 + 1] * T1[1] + Sg[r * 3 + 2] * T1[2];
    }
    const double a = T0[0] * ST0[0] + T0[1] * ST0[1] + T0[2] * ST0[2] + P.dilation;
    const double b = T0[0] * ST1[0] + T0[1] * ST1[1] + T0[2] * ST1[2];
    const double c = T1[0] * ST1[0] + T1[1] * ST1[1] + T1[2] * ST1[2] + P.dilation;
    const double det = a * c - b * b, d2 = det * det;
    const double K = (double)K_EXP2;
    const double gca = K * gea, gcb = 2.0 * K * geb, gcc = K * gec;
    const double ga = gca * (-c * c / d2) + gcb * (b * c / d2) + gcc * (1.0 / det - a * c / d2);
    const double gb = gca * (2.0 * b * c / d2) + gcb * (-1.0 / det - 2.0 * b * b / d2) + gcc * (2.0 * a * b / d2);
    const double gc = gca * (1.0 / det - c * a / d2) + gcb * (b * a / d2) + gcc * (-a * a / d2);
    double dT0[3], dT1[3];
    for (int k = 0; k < 3; ++k) {
        dT0[k] = 2.0 * ga * ST0[k] + gb * ST1[k];
        dT1[k] = gb * ST0[k] + 2.0 * gc * ST1[k];
    }
    const double gj00 = dT0[0] * R[0] + dT0[1] * R[1] + dT0[2] * R[2];
    const double gj02 = dT0[0] * R[6] + dT0[1] * R[7] + dT0[2] * R[8];
    const double gj11 = dT1[0] * R[3] + dT1[1] * R[4] + dT1[2] * R[5];
    const double gj12 = dT1[0] * R[6] + dT1[1] * R[7] + dT1[2] * R[8];
    const double z2 = pz * pz;
    double gp0 = gu * fx / pz, gp1 = gv * fy / pz;
    double gp2 = -gu * fx * px / z2 - gv * fy * py / z2 + gz - gj00 * fx / z2 - gj11 * fy / z2;
    if (lox < xn && xn < hix) { gp0 += -gj02 * fx / z2; gp2 += gj02 * 2.0 * fx * px / (z2 * pz); }
    else gp2 += gj02 * fx * xcl / z2;
    if (loy < yn && yn < hiy) { gp1 += -gj12 * fy / z2; gp2 += gj12 * 2.0 * fy * py / (z2 * pz); }
    else gp2 += gj12 * fy * ycl / z2;
    // dL/dmu = R^T dL/dp + (I - d d^T)/|mu - c| dL/dd  (O10's direction d = (mu - c)/|mu - c|)
    double gm[3];
    for (int k = 0; k < 3; ++k) gm[k] = R[k] * gp0 + R[3 + k] * gp1 + R[6 + k] * gp2;
    if (grgb[0] != 0.0 || grgb[1] != 0.0 || grgb[2] != 0.0) {
        double dv[3];
        for (int k = 0; k < 3; ++k) dv[k] = (k == 0 ? mx : k == 1 ? my : mz) + (R[k] * t[0] + R[3 + k] * t[1] + R[6 + k] * t[2]);
        const double dn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
        const double x = dv[0] / dn, y = dv[1] / dn, z = dv[2] / dn;
        // w_k = sum_c f_kc dL/drgb_c, then dL/dd = sum_k w_k grad b_k(d)
        const int nk = (S.sh_degree + 1) * (S.sh_degree + 1);
        double w[16];
        for (int k = 0; k < nk; ++k)
            w[k] = (double)S.sh[(int64_t)(k * 3) * n + g] * grgb[0] + (double)S.sh[(int64_t)(k * 3 + 1) * n + g] * grgb[1] +
                   (double)S.sh[(int64_t)(k * 3 + 2) * n + g] * grgb[2];
        const double C1 = 0.4886025119029199;
        double gx = -C1 * w[3], gy = -C1 * w[1], gz_ = C1 * w[2];
        if (nk >= 9) {
            const double a0 = 1.0925484305920792, a1 = -1.0925484305920792, a2 = 0.31539156525252005,
                         a3 = -1.0925484305920792, a4 = 0.5462742152960396;
            gx += a0 * y * w[4] - 2 * a2 * x * w[6] + a3 * z * w[7] + 2 * a4 * x * w[8];
            gy += a0 * x * w[4] + a1 * z * w[5] - 2 * a2 * y * w[6] - 2 * a4 * y * w[8];
            gz_ += a1 * y * w[5] + 4 * a2 * z * w[6] + a3 * x * w[7];
        }
        if (nk >= 16) {
            const double b0 = -0.5900435899266435, b1 = 2.890611442640554, b2 = -0.4570457994644658,
                         b3 = 0.3731763325901154, b4 = -0.4570457994644658, b5 = 1.445305721320277,
                         b6 = -0.5900435899266435;
            const double xx = x * x, yy = y * y, zz = z * z;
            gx += 6 * b0 * x * y * w[9] + b1 * y * z * w[10] - 2 * b2 * x * y * w[11] - 6 * b3 * x * z * w[12] +
                  b4 * (4 * zz - 3 * xx - yy) * w[13] + 2 * b5 * x * z * w[14] + b6 * (3 * xx - 3 * yy) * w[15];
            gy += b0 * (3 * xx - 3 * yy) * w[9] + b1 * x * z * w[10] + b2 * (4 * zz - xx - 3 * yy) * w[11] -
                  6 * b3 * y * z * w[12] - 2 * b4 * x * y * w[13] - 2 * b5 * y * z * w[14] - 6 * b6 * x * y * w[15];
            gz_ += b1 * x * y * w[10] + 8 * b2 * y * z * w[11] + b3 * (6 * zz - 3 * xx - 3 * yy) * w[12] +
                   8 * b4 * x * z * w[13] + b5 * (xx - yy) * w[14];
        }
        const double dd = x * gx + y * gy + z * gz_;
        gm[0] += (gx - x * dd) / dn;
        gm[1] += (gy - y * dd) / dn;
        gm[2] += (gz_ - z * dd) / dn;
    }
    for (int k = 0; k < 3; ++k) atomicAdd(&grad_pos[(int64_t)k * n + g], (float)gm[k]);
}

// dL/d{scale, quat, opacity, SH} of one record (gs_param_backward): the chain of
// mean_backward_kernel up to G = dL/dSigma', then dL/dSigma = T^T G T, Sigma = M M^T,
// M = R(q) diag(s), the normalised quaternion, and O10's basis for the SH rows
__global__ void param_backward_kernel(gs_scene S, const gs_view* __restrict__ views, gs_params P,
                                      const gs_record* __restrict__ rec, int64_t cap,
                                      const uint32_t* __restrict__ n_rec, int n_views,
                                      const float* __restrict__ grad_rec, float* __restrict__ g_scale,
                                      float* __restrict__ g_quat, float* __restrict__ g_opacity,
                                      float* __restrict__ g_sh) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= cap * n_views) return;
    const int vi = (int)(slot / cap);
    if ((uint32_t)(slot - (int64_t)vi * cap) >= min((uint64_t)n_rec[vi], (uint64_t)cap)) return;
    const float* gr = grad_rec + slot * 10;
    const gs_record& rc = rec[slot];
    const int64_t n = S.n;
    const uint32_t g = rc.gid;
    if (g_opacity && gr[5] != 0.0f) atomicAdd(&g_opacity[g], gr[5]);
    const gs_view& V = views[vi];
    double R[9], t[3];
    for (int k = 0; k < 9; ++k) R[k] = V.R[k];
    for (int k = 0; k < 3; ++k) t[k] = V.t[k];
    const double mx = S.pos[g], my = S.pos[n + g], mz = S.pos[2 * n + g];
    if (g_sh) {
        double grgb[3];
        for (int c = 0; c < 3; ++c) grgb[c] = rc.rgb[c] > 0.0f ? (double)gr[6 + c] : 0.0;
        if (grgb[0] != 0.0 || grgb[1] != 0.0 || grgb[2] != 0.0) {
            double dv[3] = {mx, my, mz};
            for (int k = 0; k < 3; ++k) dv[k] += R[k] * t[0] + R[3 + k] * t[1] + R[6 + k] * t[2];
            const double dn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
            const double x = dv[0] / dn, y = dv[1] / dn, z = dv[2] / dn;
            double b[16];
            b[0] = 0.28209479177387814;
            const double C1 = 0.4886025119029199;
            b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
            const double xx = x * x, yy = y * y, zz = z * z;
            b[4] = 1.0925484305920792 * x * y; b[5] = -1.0925484305920792 * y * z;
            b[6] = 0.31539156525252005 * (2 * zz - xx - yy); b[7] = -1.0925484305920792 * x * z;
            b[8] = 0.5462742152960396 * (xx - yy);
            b[9] = -0.5900435899266435 * y * (3 * xx - yy); b[10] = 2.890611442640554 * x * y * z;
            b[11] = -0.4570457994644658 * y * (4 * zz - xx - yy);
            b[12] = 0.3731763325901154 * z * (2 * zz - 3 * xx - 3 * yy);
            b[13] = -0.4570457994644658 * x * (4 * zz - xx - yy); b[14] = 1.445305721320277 * z * (xx - yy);
            b[15] = -0.5900435899266435 * x * (xx - 3 * yy);
            const int nk = (S.sh_degree + 1) * (S.sh_degree + 1);
            for (int k = 0; k < nk; ++k)
                for (int c = 0; c < 3; ++c)
                    if (grgb[c] != 0.0) atomicAdd(&g_sh[(int64_t)(k * 3 + c) * n + g], (float)(b[k] * grgb[c]));
        }
    }
    const double gea = gr[2], geb = gr[3], gec = gr[4];
    if ((!g_scale && !g_quat) || (gea == 0.0 && geb == 0.0 && gec == 0.0)) return;
    const double px = R[0] * mx + R[1] * my + R[2] * mz + t[0];
    const double py = R[3] * mx + R[4] * my + R[5] * mz + t[1];
    const double pz = R[6] * mx + R[7] * my + R[8] * mz + t[2];
    const double q0 = S.quat[g], q1 = S.quat[n + g], q2 = S.quat[2 * n + g], q3 = S.quat[3 * n + g];
    const double qn = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const double qw = q0 / qn, qx = q1 / qn, qy = q2 / qn, qz = q3 / qn;
    const double sc[3] = {S.scale[g], S.scale[n + g], S.scale[2 * n + g]};
    const double Rq[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy),
                          2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx),
                          2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)};
    double M[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) M[r * 3 + c] = Rq[r * 3 + c] * sc[c];
    double Sg[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) Sg[r * 3 + c] = M[r * 3] * M[c * 3] + M[r * 3 + 1] * M[c * 3 + 1] + M[r * 3 + 2] * M[c * 3 + 2];
    const double fx = V.fx, fy = V.fy, cx = V.cx, cy = V.cy, W = V.width, H = V.height, m = P.clamp_margin;
    const double lox = (-(m * W) - cx) / fx, hix = ((1.0 + m) * W - cx) / fx;
    const double loy = (-(m * H) - cy) / fy, hiy = ((1.0 + m) * H - cy) / fy;
    const double xcl = fmin(fmax(px / pz, lox), hix), ycl = fmin(fmax(py / pz, loy), hiy);
    const double j00 = fx / pz, j11 = fy / pz, j02 = -fx * xcl / pz, j12 = -fy * ycl / pz;
    double T0[3], T1[3], ST0[3], ST1[3];
    for (int k = 0; k < 3; ++k) { T0[k] = j00 * R[k] + j02 * R[6 + k]; T1[k] = j11 * R[3 + k] + j12 * R[6 + k]; }
    for (int r = 0; r < 3; ++r) {
        ST0[r] = Sg[r * 3] * T0[0] + Sg[r * 3 + 1] * T0[1] + Sg[r * 3 + 2] * T0[2];
        ST1[r] = Sg[r * 3] * T1[0] + Sg[r * 3 + 1] * T1[1] + Sg[r * 3 + 2] * T1[2];
    }
    const double a = T0[0] * ST0[0] + T0[1] * ST0[1] + T0[2] * ST0[2] + P.dilation;
    const double b = T0[0] * ST1[0] + T0[1] * ST1[1] + T0[2] * ST1[2];
    const double c = T1[0] * ST1[0] + T1[1] * ST1[1] + T1[2] * ST1[2] + P.dilation;
    const double det = a * c - b * b, d2 = det * det;
    const double K = (double)K_EXP2;
    const double gca = K * gea, gcb = 2.0 * K * geb, gcc = K * gec;
    const double ga = gca * (-c * c / d2) + gcb * (b * c / d2) + gcc * (1.0 / det - a * c / d2);
    const double gb = gca * (2.0 * b * c / d2) + gcb * (-1.0 / det - 2.0 * b * b / d2) + gcc * (2.0 * a * b / d2);
    const double gc = gca * (1.0 / det - c * a / d2) + gcb * (b * a / d2) + gcc * (-a * a / d2);
    // dL/dM = 2 GS M, GS = ga T0 T0^T + gb (T0 T1^T + T1 T0^T) / 2 + gc T1 T1^T
    double GS[9];
    for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc)
            GS[r * 3 + cc] = ga * T0[r] * T0[cc] + 0.5 * gb * (T0[r] * T1[cc] + T1[r] * T0[cc]) + gc * T1[r] * T1[cc];
    double dM[9];
    for (int r = 0; r < 3; ++r)
        for (int cc = 0; cc < 3; ++cc)
            dM[r * 3 + cc] = 2.0 * (GS[r * 3] * M[cc] + GS[r * 3 + 1] * M[3 + cc] + GS[r * 3 + 2] * M[6 + cc]);
    if (g_scale)
        for (int i = 0; i < 3; ++i)
            atomicAdd(&g_scale[(int64_t)i * n + g],
                      (float)(dM[i] * Rq[i] + dM[3 + i] * Rq[3 + i] + dM[6 + i] * Rq[6 + i]));
    if (g_quat) {
        double dR[9];
        for (int r = 0; r < 3; ++r)
            for (int cc = 0; cc < 3; ++cc) dR[r * 3 + cc] = dM[r * 3 + cc] * sc[cc];
        // dR/dw, dR/dx, dR/dy, dR/dz of O4's matrix (row-major)
        const double Gw[9] = {0, -2 * qz, 2 * qy, 2 * qz, 0, -2 * qx, -2 * qy, 2 * qx, 0};
        const double Gx[9] = {0, 2 * qy, 2 * qz, 2 * qy, -4 * qx, -2 * qw, 2 * qz, 2 * qw, -4 * qx};
        const double Gy[9] = {-4 * qy, 2 * qx, 2 * qw, 2 * qx, 0, 2 * qz, -2 * qw, 2 * qz, -4 * qy};
        const double Gz[9] = {-4 * qz, -2 * qw, 2 * qx, 2 * qw, -4 * qz, 2 * qy, 2 * qx, 2 * qy, 0};
        double dq[4] = {0, 0, 0, 0};
        for (int k = 0; k < 9; ++k) {
            dq[0] += dR[k] * Gw[k]; dq[1] += dR[k] * Gx[k]; dq[2] += dR[k] * Gy[k]; dq[3] += dR[k] * Gz[k];
        }
        const double qh[4] = {qw, qx, qy, qz};
        const double pr = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
        for (int i = 0; i < 4; ++i) atomicAdd(&g_quat[(int64_t)i * n + g], (float)((dq[i] - qh[i] * pr) / qn));
    }
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" {

gs_status gs_param_backward(const gs_scene* scene, const gs_projected* proj, const gs_view* views_host,
                            const gs_view* views_dev, int32_t n_views, const gs_params* params,
                            const float* grad_rec, float* grad_scale, float* grad_quat, float* grad_opacity,
                            float* grad_sh, void* stream) {
    gs_status st = validate_scene(scene, true);
    if (st != GS_OK) return st;
    st = validate_views(views_host, views_dev, n_views, nullptr, nullptr);
    if (st != GS_OK) return st;
    GS_REQUIRE(params && proj && proj->rec && proj->n_rec && grad_rec, GS_INVALID_ARG,
               "gs_param_backward: NULL pointer");
    const int64_t total = proj->rec_capacity * (int64_t)n_views;
    if (total == 0 || (!grad_scale && !grad_quat && !grad_opacity && !grad_sh)) return GS_OK;
    param_backward_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        *scene, views_dev, *params, proj->rec, proj->rec_capacity, proj->n_rec, n_views, grad_rec, grad_scale,
        grad_quat, grad_opacity, grad_sh);
    return check_launch("param_backward_kernel");
}

size_t gs_project_workspace_bytes(int32_t n_blocks, int32_t n_views) {
    if (n_views < 1) n_views = 1;
    const size_t nw = ((size_t)n_views + 31) / 32;
    size_t bytes = (size_t)n_views * sizeof(ViewConst);
    bytes = (bytes + 255) & ~size_t(255);
    bytes += (size_t)(n_blocks > 0 ? n_blocks : 0) * nw * sizeof(uint32_t);
    return (bytes + 255) & ~size_t(255);
}

gs_status gs_scene_block_bounds(const gs_scene* scene, float* block_bounds_out, void* stream) {
    gs_status st = validate_scene(scene, false);
    if (st != GS_OK) return st;
    GS_REQUIRE(scene->n_blocks > 0, GS_INVALID_ARG, "scene has no blocks");
    GS_REQUIRE(scene->block_offsets && scene->pos && scene->scale && block_bounds_out, GS_INVALID_ARG,
               "NULL pointer");
    block_bounds_kernel<<<scene->n_blocks, 256, 0, (cudaStream_t)stream>>>(
        scene->pos, scene->scale, scene->n, scene->block_offsets, scene->n_blocks, block_bounds_out);
    return check_launch("block_bounds_kernel");
}

gs_status gs_project(const gs_scene* scene, const gs_view* views_host, const gs_view* views_dev, int32_t n_views,
                     const gs_params* params, gs_projected* out, void* ws, size_t ws_bytes, void* stream) {
    gs_status st = validate_scene(scene, true);
    if (st != GS_OK) return st;
    st = validate_views(views_host, views_dev, n_views, nullptr, nullptr);
    if (st != GS_OK) return st;
    GS_REQUIRE(params != nullptr, GS_INVALID_ARG, "params is NULL");
    GS_REQUIRE(out && out->rec && out->n_rec && out->diag && out->status, GS_INVALID_ARG,
               "out (gs_projected) has a NULL pointer");
    GS_REQUIRE(out->rec_capacity >= 1 && out->rec_capacity * (int64_t)n_views < (int64_t(1) << 32),
               GS_INVALID_ARG, "rec_capacity = %lld invalid (n_views * cap must be < 2^32)",
               (long long)out->rec_capacity);
    const size_t need = gs_project_workspace_bytes(scene->n_blocks, n_views);
    GS_REQUIRE(ws != nullptr && ws_bytes >= need, GS_WORKSPACE_TOO_SMALL, "gs_project workspace %zu < %zu",
               ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    ViewConst* vc = reinterpret_cast<ViewConst*>(ws);
    size_t off = ((size_t)n_views * sizeof(ViewConst) + 255) & ~size_t(255);
    uint32_t* mask = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + off);

    cudaMemsetAsync(out->n_rec, 0, sizeof(uint32_t) * n_views, s);
    cudaMemsetAsync(out->diag, 0, sizeof(uint64_t) * 4, s);
    view_const_kernel<<<(n_views + 127) / 128, 128, 0, s>>>(views_dev, n_views, *params, vc);
    if ((st = check_launch("view_const_kernel")) != GS_OK) return st;
    if (scene->n == 0) return GS_OK;
    if (scene->n_blocks > 0) {
        const int64_t work = (int64_t)scene->n_blocks * ((n_views + 31) / 32);
        block_cull_kernel<<<(unsigned)((work + 127) / 128), 128, 0, s>>>(views_dev, vc, n_views, scene->n_blocks,
                                                                        scene->block_bounds, *params, mask);
        if ((st = check_launch("block_cull_kernel")) != GS_OK) return st;
    }
    const unsigned grid = (unsigned)((scene->n + PROJ_THREADS - 1) / PROJ_THREADS);
    int sh_smem = 0;
#if GS_PROJ_SH_SMEM
    sh_smem = (PROJ_THREADS / 32) * (scene->sh_degree + 1) * (scene->sh_degree + 1) * 3 * 32 * (int)sizeof(float);
    // kernel attributes are per device: set on every call (cheap)
    cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sh_smem);
#endif
    project_kernel<<<grid, PROJ_THREADS, sh_smem, s>>>(*scene, views_dev, vc, n_views, *params, mask, out->rec,
                                                 out->rec_capacity, out->n_rec, out->diag, out->status);
    return check_launch("project_kernel");
}

}  // extern "C"

extern "C" gs_status gs_mean_backward(const gs_scene* scene, const gs_projected* proj, const gs_view* views_host,
                                      const gs_view* views_dev, int32_t n_views, const gs_params* params,
                                      const float* grad_rec, float* grad_pos, void* stream) {
    gs_status st = validate_scene(scene, true);
    if (st != GS_OK) return st;
    st = validate_views(views_host, views_dev, n_views, nullptr, nullptr);
    if (st != GS_OK) return st;
    GS_REQUIRE(params && proj && proj->rec && proj->n_rec && grad_rec && grad_pos, GS_INVALID_ARG,
               "gs_mean_backward: NULL pointer");
    const int64_t total = proj->rec_capacity * (int64_t)n_views;
    if (total == 0) return GS_OK;
    mean_backward_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        *scene, views_dev, *params, proj->rec, proj->rec_capacity, proj->n_rec, n_views, grad_rec, grad_pos);
    return check_launch("mean_backward_kernel");
}
