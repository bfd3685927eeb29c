// gs_match.cu -- N2: coarse-to-fine
// probabilistic mutual matching between a query feature map and a rendered
// feature map (Eq. 11 at P:312-316; readings
// Q31-Q34).
//
//   1. pool_kernel: w x w (w = 8) average pooling of both maps (Q31), L2
//      normalisation (Q32), split into fp16 hi + lo; written twice: K-major
//      rows (A operand, staged to TMEM) and 128-cell MN-major canonical chunks
//      (B operand, one TMA bulk copy per chunk).
//   2. row_kernel<STATS>: per 128 query cells, stream all column chunks of
//      128 cells through a double-buffered shared ring (cp.async.bulk) and a
//      double-buffered TMEM accumulator; M = A B^T by tcgen05 kind::f16 MMAs
//      (hi.hi + hi.lo + lo.hi, ~2^-22 relative: fp32-grade cosines); the 16
//      epilogue warps read their lane quarter / 32-column part with tcgen05.ld and
//      keep an online log2-sum-exp2 of x = M log2(e)/tau per row:
//      c_i = log2 sum_j 2^(x_ij).
//   3. row_kernel<ARGMAX>: same GEMM; log2 P_ij = 2 x_ij - c_i - c'_j (Eq. 11
//      in log2 units), so the row argmax of P is the argmax of 2 x_ij - c'_j --
//      no exponential per element; P is evaluated once at the maximum.
//      Both kernels run on both directions (query rows x rendered columns and
//      the transpose): the column statistics / column argmax of P are the row
//      statistics / row argmax of the transposed problem, so no kernel needs
//      a cross-CTA column reduction or atomics.
//   4. mnn_kernel: (i, j) iff argmax_row(i) = j, argmax_col(j) = i and
//      P_ij > p_min (ties to the lowest index, Q33).
//   5. fine_kernel: one CTA per coarse match -- Eq. 11 + MNN between the
//      64 pixels of the query cell and the 64 of the matched rendered cell
//      (Q34); the 64 x 64 x D cosine block on the tensor cores (mma.sync
//      m16n8k16, fp16 hi + lo operands, 3 products -- a window is too small to
//      amortise a TMEM allocation), the softmaxes / MNN in fp32, 3 x 3
//      soft-argmax around the peak, gather of the peak's back-projected point.
#include <cuda_fp16.h>

#include <cmath>

#include "gs_common.cuh"
#include "gs_tc.cuh"

namespace gs {
namespace {

constexpr int MW = 8;                    // window w = H_f / H_c
constexpr int CB = 128;                  // cells per row block (M) and per column chunk (N)
constexpr int NH = 4;                    // column parts per chunk
constexpr int CW = CB / NH;              // columns per epilogue warp per chunk
constexpr int EPI = 4 * NH;              // epilogue warps: 4 TMEM lane quarters x NH column parts
constexpr int ROW_THREADS = (EPI + 1) * 32;
constexpr uint32_t TMEM_COLS = 512;      // 2 x 128 accumulator columns + A (hi, lo)
constexpr float LOG2E = 1.4426950408889634f;

struct MatchWs {
    __half* a[2][2];      // [map][hi/lo] -> [n_pairs][Ncp][D] K-major rows
    __half* bimg[2];      // [map] -> [n_pairs][Ncp/128][2][128 D] canonical chunks (hi, lo)
    float* c2[2];         // [direction] -> [n_pairs][Ncp] row log2-sum-exp2
    int32_t* arg[2];      // [direction] -> [n_pairs][Ncp] row argmax of P
    float* pbest;         // [n_pairs][Ncp] P at the direction-0 argmax
};

inline int64_t pad_cells(int64_t nc) { return (nc + CB - 1) / CB * CB; }

MatchWs carve(void* ws, int64_t B, int64_t Ncp, int D, size_t* total) {
    MatchWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        char* p = static_cast<char*>(ws) + off;
        off += (bytes + 255) & ~size_t(255);
        return p;
    };
    const size_t plane = (size_t)B * Ncp * D * sizeof(__half);
    for (int m = 0; m < 2; ++m)
        for (int h = 0; h < 2; ++h) w.a[m][h] = reinterpret_cast<__half*>(take(plane));
    for (int m = 0; m < 2; ++m) w.bimg[m] = reinterpret_cast<__half*>(take(2 * plane));
    for (int d = 0; d < 2; ++d) w.c2[d] = reinterpret_cast<float*>(take((size_t)B * Ncp * 4));
    for (int d = 0; d < 2; ++d) w.arg[d] = reinterpret_cast<int32_t*>(take((size_t)B * Ncp * 4));
    w.pbest = reinterpret_cast<float*>(take((size_t)B * Ncp * 4));
    if (total) *total = off;
    return w;
}

// ---------------------------------------------------------------- 1. pooling
// one warp per (cell, map, pair); lane handles channels lane and lane + 32
__global__ void __launch_bounds__(256) pool_kernel(const float* __restrict__ Fq, const float* __restrict__ Fr, int D,
                                                   int H, int W, int Nc, int Ncp, MatchWs ws) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * 8 + warp, m = blockIdx.y, b = blockIdx.z;
    if (cell >= Ncp) return;
    const int Wc = W / MW;
    const float* F = (m == 0 ? Fq : Fr) + (int64_t)b * D * H * W;
    float v[2] = {0.f, 0.f};
    if (cell < Nc) {
        const int cy = cell / Wc, cx = cell % Wc;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int ch = lane + 32 * t;
            if (ch < D) {
                float s = 0.f;
                const float* p = F + (int64_t)ch * H * W + (int64_t)(cy * MW) * W + cx * MW;
                for (int y = 0; y < MW; ++y) {
                    const float4 a = __ldg(reinterpret_cast<const float4*>(p + (int64_t)y * W));
                    const float4 c = __ldg(reinterpret_cast<const float4*>(p + (int64_t)y * W) + 1);
                    s += ((a.x + a.y) + (a.z + a.w)) + ((c.x + c.y) + (c.z + c.w));
                }
                v[t] = s * (1.0f / (MW * MW));
            }
        }
    }
    float ss = v[0] * v[0] + v[1] * v[1];
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = ss > 0.f ? 1.0f / sqrtf(ss) : 0.f;   // zero vector stays zero (Q32)
    const int64_t rowbase = ((int64_t)b * Ncp + cell) * D;
    const int chunk = cell / CB, n = cell % CB;
    __half* bi = ws.bimg[m] + ((int64_t)b * (Ncp / CB) + chunk) * 2 * CB * D;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int k = lane + 32 * t;
        if (k < D) {
            const float x = v[t] * inv;
            const __half hi = __float2half_rn(x);
            const __half lo = __float2half_rn(x - __half2float(hi));
            ws.a[m][0][rowbase + k] = hi;
            ws.a[m][1][rowbase + k] = lo;
            // canonical MN-major (k, n): n/8 * 64 + (k%8) * 8 + (k/8) * (8 * CB) + n%8 halves
            const int64_t e = (n >> 3) * 64 + (k & 7) * 8 + (k >> 3) * (8 * CB) + (n & 7);
            bi[e] = hi;
            bi[CB * D + e] = lo;
        }
    }
}

// ---------------------------------------------------------------- 2./3. rows
template <int D>
struct RowSmem {
    alignas(128) __half b[3][2][CB * D];   // [stage][hi/lo] canonical chunk (3-stage ring)
    alignas(16) float cc[3][CB];            // [stage] column statistics c'_j of the chunk (argmax pass)
    float part_v[NH - 1][CB];               // column parts 1.. partials (m or best value)
    float part_w[NH - 1][CB];               // (l or best index)
    uint64_t full[3], empty[3], dfull[2], dfree[2];
    uint32_t tmem;
};

// Direction d: rows = map d (0 query, 1 rendered), columns = map 1 - d.
template <int D, bool ARGMAX>
__global__ void __launch_bounds__(ROW_THREADS, 1)
row_kernel(MatchWs ws, int Nc, int Ncp, float k2) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    RowSmem<D>& sm = *reinterpret_cast<RowSmem<D>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rb = blockIdx.x, d = blockIdx.y, b = blockIdx.z;
    const int nch = Ncp / CB;
    const int rows_map = d, cols_map = 1 - d;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 3; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.dfull[s], 1);
            mbar_init(&sm.dfree[s], EPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&sm.tmem, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem;
    const uint32_t tA = tmem + 2 * CB;           // A hi: D/2 columns, then A lo: D/2 columns
    // A (this block's 128 rows, hi and lo) -> TMEM, one lane per row
    if (warp < 4) {
        const int row = warp * 32 + lane;
        const int64_t base = ((int64_t)b * Ncp + rb * CB + row) * D;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint4* src = reinterpret_cast<const uint4*>(ws.a[rows_map][h] + base);
#pragma unroll
            for (int c8 = 0; c8 < D / 16; ++c8) {   // 16 halves = 8 TMEM columns per store
                const uint4 x = __ldg(src + 2 * c8), y = __ldg(src + 2 * c8 + 1);
                const uint32_t r[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
                tmem_st8(tA + ((uint32_t)(warp * 32) << 16) + h * (D / 2) + c8 * 8, r);
            }
        }
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    const __half* bsrc = ws.bimg[cols_map] + (int64_t)b * nch * 2 * CB * D;
    const float* csrc = ws.c2[1 - d] + (int64_t)b * Ncp;
    constexpr uint32_t CHUNK_BYTES = 2 * CB * D * sizeof(__half);
    if (warp == EPI) {
        // ------------------------------------------------ producer + MMA issuer
        if (lane == 0) {
            constexpr uint32_t IDESC = idesc_f16(CB, CB);
            auto load = [&](int c, int st) {
                mbar_expect_tx(&sm.full[st], CHUNK_BYTES + (ARGMAX ? CB * 4u : 0u));
                bulk_g2s(&sm.b[st][0][0], bsrc + (int64_t)c * 2 * CB * D, CHUNK_BYTES, &sm.full[st]);
                if (ARGMAX) bulk_g2s(&sm.cc[st][0], csrc + (int64_t)c * CB, CB * 4u, &sm.full[st]);
            };
            for (int c = 0; c < 2 && c < nch; ++c) load(c, c);
            for (int c = 0; c < nch; ++c) {
                const int st = c % 3, ds = c & 1;
                mbar_wait(&sm.full[st], (uint32_t)(c / 3) & 1u);
                if (c >= 2) mbar_wait(&sm.dfree[ds], (uint32_t)((c >> 1) - 1) & 1u);   // epilogue c-2 done
                tc_fence_after();
                const uint32_t dst = tmem + ds * CB;
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    // K-step ks = k-groups 2ks, 2ks+1: B start + ks * 2 * LBO, A columns + ks * 8
                    const uint64_t bh = smem_desc(&sm.b[st][0][0] + ks * 2 * 8 * CB, 16 * CB, 128);
                    const uint64_t bl = smem_desc(&sm.b[st][1][0] + ks * 2 * 8 * CB, 16 * CB, 128);
                    const uint32_t ah = tA + ks * 8, al = tA + D / 2 + ks * 8;
                    tc_mma_f16(dst, ah, bh, IDESC, ks > 0 ? 1u : 0u, 4);
                    tc_mma_f16(dst, ah, bl, IDESC, 1u, 4);
                    tc_mma_f16(dst, al, bh, IDESC, 1u, 4);
                }
                tc_commit(&sm.dfull[ds]);
                tc_commit(&sm.empty[st]);
                if (c + 2 < nch) {
                    // chunk c+2 goes to the stage of chunk c-1: its MMAs and (argmax: its c'
                    // values) its epilogue must be done -- the latter is what the accumulator
                    // double buffer needs before MMA c+1 anyway
                    const int sn = (c + 2) % 3;
                    if (c >= 1) {
                        mbar_wait(&sm.empty[sn], (uint32_t)((c - 1) / 3) & 1u);
                        if (ARGMAX) mbar_wait(&sm.dfree[(c - 1) & 1], (uint32_t)((c - 1) >> 1) & 1u);
                    }
                    load(c + 2, sn);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------ epilogue warps
        const int q = warp & 3, hh = warp >> 2;
        const int row = q * 32 + lane;
        const int64_t gi = (int64_t)b * Ncp + rb * CB + row;
        float run_m = -INFINITY, run_l = 0.f;      // STATS: online log2-sum-exp2
        float best = -INFINITY;                    // ARGMAX: max of 2x - c'_j
        int bj = -1;
        for (int c = 0; c < nch; ++c) {
            const int s = c & 1;
            const uint32_t ph = (c >> 1) & 1;
            mbar_wait(&sm.dfull[s], ph);
            tc_fence_after();
            float x[CW];
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + s * CB + hh * CW;
#pragma unroll
            for (int t = 0; t < CW; t += 32) tmem_ld32(ta + t, x + t);
            tmem_wait_ld();
            const int j0 = c * CB + hh * CW;
            const int nv = min(CW, Nc - j0);
            float cj[ARGMAX ? CW : 1];
            if constexpr (ARGMAX) {
                const float4* cs = reinterpret_cast<const float4*>(&sm.cc[c % 3][hh * CW]);
#pragma unroll
                for (int t = 0; t < CW / 4; ++t) {
                    const float4 v4 = cs[t];   // broadcast
                    cj[4 * t] = v4.x; cj[4 * t + 1] = v4.y; cj[4 * t + 2] = v4.z; cj[4 * t + 3] = v4.w;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.dfree[s]);
            if constexpr (!ARGMAX) {
                float mx = -INFINITY;
#pragma unroll
                for (int t = 0; t < CW; ++t) {
                    x[t] *= k2;
                    if (t < nv) mx = fmaxf(mx, x[t]);
                }
                if (nv > 0) {
                    const float mn = fmaxf(run_m, mx);
                    float acc = 0.f;
#pragma unroll
                    for (int t = 0; t < CW; ++t)
                        if (t < nv) acc += ex2_ftz(x[t] - mn);
                    run_l = run_l * ex2_ftz(run_m - mn) + acc;
                    run_m = mn;
                }
            } else {
                // argmax over the chunk of 2 x k2 - c'_j (one FFMA + compare / select per
                // element; the winner's column offset is an immediate), merged once
                const float k22 = 2.f * k2;
                float cb = -INFINITY;
                int ct = -1;
                if (nv == CW) {
#pragma unroll
                    for (int t = 0; t < CW; ++t) {
                        const float y = fmaf(x[t], k22, -cj[t]);
                        if (y > cb) { cb = y; ct = t; }
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < CW; ++t) {
                        const float y = fmaf(x[t], k22, -cj[t]);
                        if (t < nv && y > cb) { cb = y; ct = t; }
                    }
                }
                if (cb > best) { best = cb; bj = j0 + ct; }
            }
        }
        // combine the column parts of each row
        if (hh > 0) {
            sm.part_v[hh - 1][row] = ARGMAX ? best : run_m;
            sm.part_w[hh - 1][row] = ARGMAX ? __int_as_float(bj) : run_l;
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(EPI * 32) : "memory");
        if (hh == 0) {
            if constexpr (!ARGMAX) {
                float mt = run_m;
#pragma unroll
                for (int h = 0; h < NH - 1; ++h) mt = fmaxf(mt, sm.part_v[h][row]);
                float lt = run_l > 0.f ? run_l * ex2_ftz(run_m - mt) : 0.f;
#pragma unroll
                for (int h = 0; h < NH - 1; ++h) {
                    const float l1 = sm.part_w[h][row];
                    if (l1 > 0.f) lt += l1 * ex2_ftz(sm.part_v[h][row] - mt);
                }
                ws.c2[d][gi] = mt + log2f(lt);
            } else {
#pragma unroll
                for (int h = 0; h < NH - 1; ++h) {
                    const float b1 = sm.part_v[h][row];
                    const int j1 = __float_as_int(sm.part_w[h][row]);
                    if (b1 > best || (b1 == best && j1 >= 0 && (bj < 0 || j1 < bj))) { best = b1; bj = j1; }
                }
                ws.arg[d][gi] = (rb * CB + row < Nc) ? bj : -1;
                if (d == 0) ws.pbest[gi] = bj >= 0 ? ex2_ftz(best - ws.c2[0][gi]) : 0.f;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, TMEM_COLS);
    }
}

// ---------------------------------------------------------------- 4. MNN
__global__ void mnn_kernel(MatchWs ws, int Nc, int Ncp, float p_min, int32_t* __restrict__ coarse,
                           float* __restrict__ coarse_prob) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y;
    if (i >= Nc) return;
    const int64_t gi = (int64_t)b * Ncp + i;
    const int j = ws.arg[0][gi];
    const float p = ws.pbest[gi];
    const bool ok = j >= 0 && ws.arg[1][(int64_t)b * Ncp + j] == i && p > p_min;
    coarse[(int64_t)b * Nc + i] = ok ? j : -1;
    coarse_prob[(int64_t)b * Nc + i] = ok ? p : 0.f;
}

// ---------------------------------------------------------------- 5. fine windows
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int WP = MW * MW;   // 64 pixels per window

__global__ void __launch_bounds__(256) fine_kernel(const float* __restrict__ Fq, const float* __restrict__ Fr, int D,
                                                   int H, int W, int Nc, const int32_t* __restrict__ coarse,
                                                   float k2, float p_min, const float* __restrict__ xyz,
                                                   const uint8_t* __restrict__ valid, gs_matches out) {
    extern __shared__ float fsm[];
    // region 0 holds the fp32 pixel vectors until they are converted to fp16, then the
    // cosine block X (written only after the MMAs, which read the fp16 copies)
    const int R0 = max(2 * WP * (D + 1), WP * 65);
    float* qf = fsm;                      // [64][D + 1]
    float* rf = qf + WP * (D + 1);        // [64][D + 1]
    float* X = fsm;                       // [64][65]  x = cos * log2(e) / tau
    float* rc = fsm + R0;                 // [64] row log2-sum-exp2
    float* cc = rc + WP;                  // [64] column log2-sum-exp2
    int* carg = reinterpret_cast<int*>(cc + WP);   // [64] column argmax
    __half* qh = reinterpret_cast<__half*>(carg + WP);   // [64][D + 8] fp16 hi / lo operands
    __half* ql = qh + WP * (D + 8);
    __half* rh = ql + WP * (D + 8);
    __half* rl = rh + WP * (D + 8);
    const int ic = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    const int Wc = W / MW;
    const int64_t HW = (int64_t)H * W;
    const int jc = coarse[(int64_t)b * Nc + ic];
    const int qy0 = (ic / Wc) * MW, qx0 = (ic % Wc) * MW;
    if (jc < 0) {   // no coarse match: the window's query pixels stay unmatched
        if (tid < WP) {
            const int64_t pl = (int64_t)(qy0 + tid / MW) * W + qx0 + tid % MW;
            out.peak[(int64_t)b * HW + pl] = -1;
            out.prob[(int64_t)b * HW + pl] = 0.f;
            out.ref[(int64_t)b * 2 * HW + pl] = 0.f;
            out.ref[(int64_t)b * 2 * HW + HW + pl] = 0.f;
            if (out.xyz)
                for (int k = 0; k < 3; ++k) out.xyz[(int64_t)b * 3 * HW + k * HW + pl] = 0.f;
            if (out.valid) out.valid[(int64_t)b * HW + pl] = 0;
        }
        return;
    }
    const int ry0 = (jc / Wc) * MW, rx0 = (jc % Wc) * MW;
    const float* Q = Fq + (int64_t)b * D * HW;
    const float* R = Fr + (int64_t)b * D * HW;
    for (int e = tid; e < D * WP; e += blockDim.x) {
        const int ch = e / WP, a = e % WP;
        qf[a * (D + 1) + ch] = __ldg(&Q[ch * HW + (int64_t)(qy0 + a / MW) * W + qx0 + a % MW]);
        rf[a * (D + 1) + ch] = __ldg(&R[ch * HW + (int64_t)(ry0 + a / MW) * W + rx0 + a % MW]);
    }
    __syncthreads();
    if (tid < 2 * WP) {   // normalise the 128 pixel vectors (zero stays zero, Q32)
        float* v = (tid < WP ? qf : rf) + (tid % WP) * (D + 1);
        float ss = 0.f;
        for (int ch = 0; ch < D; ++ch) ss += v[ch] * v[ch];
        const float inv = ss > 0.f ? 1.0f / sqrtf(ss) : 0.f;
        for (int ch = 0; ch < D; ++ch) v[ch] *= inv;
    }
    __syncthreads();
    // the 64 x 64 x D cosine block on the tensor cores: fp16 hi + lo operands,
    // hi.hi + hi.lo + lo.hi (~2^-22 relative), fp32 accumulation
    const int HS = D + 8;                               // half row stride (conflict-free fragments)
    for (int e = tid; e < 2 * WP * D; e += blockDim.x) {
        const int m = e / (WP * D), rem = e % (WP * D), a = rem / D, ch = rem % D;
        const float x = (m == 0 ? qf : rf)[a * (D + 1) + ch];
        const __half hi = __float2half_rn(x);
        (m == 0 ? qh : rh)[a * HS + ch] = hi;
        (m == 0 ? ql : rl)[a * HS + ch] = __float2half_rn(x - __half2float(hi));
    }
    __syncthreads();
    {
        const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
        const int rb = warp & 3, chf = warp >> 2;        // rows 16 rb.., columns 32 chf..
        float acc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
        auto u32 = [](const __half* p) { return *reinterpret_cast<const uint32_t*>(p); };
        for (int ks = 0; ks < D / 16; ++ks) {
            const int r0 = (16 * rb + g) * HS + 16 * ks + 2 * t4, r1 = r0 + 8 * HS;
            const uint32_t ah[4] = {u32(qh + r0), u32(qh + r1), u32(qh + r0 + 8), u32(qh + r1 + 8)};
            const uint32_t al[4] = {u32(ql + r0), u32(ql + r1), u32(ql + r0 + 8), u32(ql + r1 + 8)};
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const int c0 = (32 * chf + 8 * nt + g) * HS + 16 * ks + 2 * t4;
                const uint32_t bh0 = u32(rh + c0), bh1 = u32(rh + c0 + 8);
                const uint32_t bl0 = u32(rl + c0), bl1 = u32(rl + c0 + 8);
                mma16816(acc[nt], ah, bh0, bh1);
                mma16816(acc[nt], ah, bl0, bl1);
                mma16816(acc[nt], al, bh0, bh1);
            }
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int col = 32 * chf + 8 * nt + 2 * t4, row = 16 * rb + g;
            X[row * 65 + col] = acc[nt][0] * k2;
            X[row * 65 + col + 1] = acc[nt][1] * k2;
            X[(row + 8) * 65 + col] = acc[nt][2] * k2;
            X[(row + 8) * 65 + col + 1] = acc[nt][3] * k2;
        }
    }
    __syncthreads();
    if (tid < 2 * WP) {   // row (tid < 64) / column log2-sum-exp2
        const int r = tid % WP;
        const bool rowwise = tid < WP;
        float mx = -INFINITY;
        for (int t = 0; t < WP; ++t) mx = fmaxf(mx, rowwise ? X[r * 65 + t] : X[t * 65 + r]);
        float l = 0.f;
        for (int t = 0; t < WP; ++t) l += ex2_ftz((rowwise ? X[r * 65 + t] : X[t * 65 + r]) - mx);
        (rowwise ? rc : cc)[r] = mx + log2f(l);
    }
    __syncthreads();
    if (tid >= WP && tid < 2 * WP) {   // column argmax of P: max over rows of 2x - c_a
        const int bb = tid - WP;
        float best = -INFINITY;
        int ba = -1;
        for (int a = 0; a < WP; ++a) {
            const float y = 2.f * X[a * 65 + bb] - rc[a];
            if (y > best) { best = y; ba = a; }
        }
        carg[bb] = ba;
    }
    __syncthreads();
    if (tid < WP) {
        const int a = tid;
        float best = -INFINITY;
        int bs = -1;
        for (int bb = 0; bb < WP; ++bb) {
            const float y = 2.f * X[a * 65 + bb] - cc[bb];
            if (y > best) { best = y; bs = bb; }
        }
        const float p = ex2_ftz(best - rc[a]);
        const bool ok = bs >= 0 && carg[bs] == a && p > p_min;
        const int64_t pl = (int64_t)(qy0 + a / MW) * W + qx0 + a % MW;   // query pixel in the view
        const int64_t pq = (int64_t)b * HW + pl;
        float rx = 0.f, ry = 0.f;
        int64_t peak = -1;
        if (ok) {
            const int by = bs / MW, bx = bs % MW;
            float num_x = 0.f, num_y = 0.f, den = 0.f;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int y = by + dy, x = bx + dx;
                    if (y < 0 || y >= MW || x < 0 || x >= MW) continue;
                    const float w = ex2_ftz(2.f * X[a * 65 + y * MW + x] - rc[a] - cc[y * MW + x]);
                    num_x += w * (float)x;
                    num_y += w * (float)y;
                    den += w;
                }
            rx = (float)rx0 + num_x / den;
            ry = (float)ry0 + num_y / den;
            peak = (int64_t)(ry0 + by) * W + rx0 + bx;
        }
        out.peak[pq] = (int32_t)peak;
        out.prob[pq] = ok ? p : 0.f;
        out.ref[(int64_t)b * 2 * HW + pl] = rx;
        out.ref[(int64_t)b * 2 * HW + HW + pl] = ry;
        if (out.xyz)
            for (int k = 0; k < 3; ++k)
                out.xyz[(int64_t)b * 3 * HW + k * HW + pl] =
                    ok && xyz ? __ldg(&xyz[(int64_t)b * 3 * HW + k * HW + peak]) : 0.f;
        if (out.valid) out.valid[pq] = ok && valid ? __ldg(&valid[(int64_t)b * HW + peak]) : 0;
    }
}

template <int D>
gs_status launch_rows(const MatchWs& w, int B, int Nc, int Ncp, float k2, cudaStream_t s) {
    // each CTA allocates all 512 TMEM columns: request enough shared memory that only
    // one CTA is resident per SM (a second would just wait in tcgen05.alloc)
    const int smem = std::max((int)sizeof(RowSmem<D>), 120 * 1024);
    cudaFuncSetAttribute(row_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(row_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const dim3 grid(Ncp / CB, 2, B);
    row_kernel<D, false><<<grid, ROW_THREADS, smem, s>>>(w, Nc, Ncp, k2);
    gs_status st = check_launch("row_kernel<stats>");
    if (st != GS_OK) return st;
    row_kernel<D, true><<<grid, ROW_THREADS, smem, s>>>(w, Nc, Ncp, k2);
    return check_launch("row_kernel<argmax>");
}

}  // namespace
}  // namespace gs

using namespace gs;

extern "C" size_t gs_match_workspace_bytes(int32_t n_pairs, int32_t D, int32_t H, int32_t W) {
    if (n_pairs < 1 || D < 1 || H < MW || W < MW) return 0;
    size_t total = 0;
    carve(nullptr, n_pairs, pad_cells((int64_t)(H / MW) * (W / MW)), D, &total);
    return total;
}

extern "C" gs_status gs_match(const float* query_feat, const float* rend_feat, int32_t n_pairs, int32_t D, int32_t H,
                              int32_t W, float tau, float p_min, const float* rend_xyz, const uint8_t* rend_valid,
                              void* ws, size_t ws_bytes, gs_matches* out, void* stream) {
    GS_REQUIRE(query_feat && rend_feat && out && out->coarse && out->coarse_prob && out->peak && out->prob &&
                   out->ref,
               GS_INVALID_ARG, "gs_match: NULL pointer");
    GS_REQUIRE(n_pairs >= 1 && n_pairs <= 65535, GS_INVALID_ARG, "n_pairs = %d", n_pairs);
    GS_REQUIRE(D == 16 || D == 32 || D == 48 || D == 64, GS_UNSUPPORTED, "gs_match: D = %d (need 16, 32, 48, 64)",
               D);
    GS_REQUIRE(H >= MW && W >= MW && H % MW == 0 && W % MW == 0, GS_INVALID_ARG,
               "gs_match: H = %d, W = %d must be positive multiples of %d (Q31)", H, W, MW);
    GS_REQUIRE((int64_t)H * W * D < (int64_t(1) << 31), GS_UNSUPPORTED, "gs_match: map too large");
    GS_REQUIRE(tau > 0.f && std::isfinite(tau) && std::isfinite(p_min), GS_INVALID_ARG, "gs_match: tau = %g",
               (double)tau);
    GS_REQUIRE(((uintptr_t)query_feat & 15) == 0 && ((uintptr_t)rend_feat & 15) == 0 && ((uintptr_t)ws & 255) == 0,
               GS_INVALID_ARG, "gs_match: feature maps must be 16-byte and ws 256-byte aligned");
    const int Nc = (H / MW) * (W / MW);
    const int Ncp = (int)pad_cells(Nc);
    size_t need = 0;
    MatchWs w = carve(ws, n_pairs, Ncp, D, &need);
    GS_REQUIRE(ws != nullptr && ws_bytes >= need, GS_WORKSPACE_TOO_SMALL, "gs_match workspace %zu < %zu", ws_bytes,
               need);
    cudaStream_t s = (cudaStream_t)stream;
    const float k2 = LOG2E / tau;
    pool_kernel<<<dim3((Ncp + 7) / 8, 2, n_pairs), 256, 0, s>>>(query_feat, rend_feat, D, H, W, Nc, Ncp, w);
    gs_status st = check_launch("pool_kernel");
    if (st != GS_OK) return st;
    switch (D) {
        case 16: st = launch_rows<16>(w, n_pairs, Nc, Ncp, k2, s); break;
        case 32: st = launch_rows<32>(w, n_pairs, Nc, Ncp, k2, s); break;
        case 48: st = launch_rows<48>(w, n_pairs, Nc, Ncp, k2, s); break;
        default: st = launch_rows<64>(w, n_pairs, Nc, Ncp, k2, s); break;
    }
    if (st != GS_OK) return st;
    mnn_kernel<<<dim3((Nc + 255) / 256, n_pairs), 256, 0, s>>>(w, Nc, Ncp, p_min, out->coarse, out->coarse_prob);
    if ((st = check_launch("mnn_kernel")) != GS_OK) return st;
    const int fsmem = (int)sizeof(float) * (std::max(2 * WP * (D + 1), WP * 65) + 3 * WP) + 4 * WP * (D + 8) * 2;
    cudaFuncSetAttribute(fine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    fine_kernel<<<dim3(Nc, n_pairs), 256, fsmem, s>>>(query_feat, rend_feat, D, H, W, Nc, out->coarse, k2, p_min,
                                                      rend_xyz, rend_valid, *out);
    return check_launch("fine_kernel");
}
