// Standalone check of the tcgen05 primitives used by the rasterizer's feature path:
// TMEM alloc, tcgen05.st of A (K-major fp16, M=128 rows = 128 lanes), B in shared
// memory (MN-major fp16, SWIZZLE_NONE canonical layout), tcgen05.mma kind::f16
// (TS: A from TMEM), commit to an mbarrier, tcgen05.ld of D.  D = A B checked on host.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int M = 128, N = 32, K = 16;

__global__ void tc_kernel(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ Dout, int accumulate_twice) {
    __shared__ __align__(1024) __half bs[K * N];     // canonical MN-major: (n/8)*SBO + (k%8)*8 + (k/8)*LBO elements
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // B into the canonical layout: element (k, n) at halves: (n/8)*64 + (k%8)*8 + (k/8)*256 + n%8
    for (int i = tid; i < K * N; i += blockDim.x) {
        const int k = i / N, n = i % N;
        bs[(n / 8) * 64 + (k % 8) * 8 + (k / 8) * 256 + n % 8] = __float2half_rn(B[k * N + n]);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;
    const uint32_t colA = 0, colD = 32;
    // A: row m = lane (32 * warp + lane), K-major fp16 pairs per 32-bit column
    {
        const int m = warp * 32 + lane;
        uint32_t r[8];
        for (int c = 0; c < 8; ++c) {
            const __half2 h = __floats2half2_rn(A[m * K + 2 * c], A[m * K + 2 * c + 1]);
            r[c] = *reinterpret_cast<const uint32_t*>(&h);
        }
        const uint32_t addr = tbase + ((uint32_t)(warp * 32) << 16) + colA;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     :: "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        const uint32_t sbo = 128, lbo = 512;   // bytes
        uint64_t desc = 0;
        desc |= (uint64_t)((smem_u32(bs) >> 4) & 0x3FFF);
        desc |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
        desc |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
        desc |= (uint64_t)1 << 46;                         // version (Blackwell)
        const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (1u << 16) |
                               ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int rep = 0; rep <= accumulate_twice; ++rep) {
            const uint32_t acc = rep > 0 ? 1u : 0u;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}\n"
                         :: "r"(tbase + colD), "r"(tbase + colA), "l"(desc), "r"(idesc), "r"(acc),
                            "r"(0u), "r"(0u), "r"(0u), "r"(0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
    }
    // wait for the MMA
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                 :: "r"(smem_u32(&bar)), "r"(0u) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    {
        const uint32_t addr = tbase + ((uint32_t)(warp * 32) << 16) + colD;
        uint32_t d[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                       "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]),
                       "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]),
                       "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int m = warp * 32 + lane;
        for (int n = 0; n < 32; ++n) Dout[m * N + n] = __uint_as_float(d[n]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "r"(64));
}

// Per-warp lane-masked MMAs: warp w writes rows 32w..32w+31 of A, builds its own
// B_w = (w + 1) B, and issues an M=128 MMA whose disable-output-lane mask leaves
// only its own 32 TMEM lanes writable; two rounds (scale-C 0, then 1).
__global__ void tc_kernel_masked(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ Dout) {
    __shared__ __align__(1024) __half bs[4][K * N];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar[4];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = lane; i < K * N; i += 32) {
        const int k = i / N, n = i % N;
        bs[warp][(n / 8) * 64 + (k % 8) * 8 + (k / 8) * 256 + n % 8] = __float2half_rn(B[k * N + n] * (warp + 1));
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar[warp])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem_base;
    const uint32_t colA = 0, colD = 32;
    for (int round = 0; round < 2; ++round) {
        const int m = warp * 32 + lane;
        uint32_t r[8];
        for (int c = 0; c < 8; ++c) {
            const __half2 h = __floats2half2_rn(A[m * K + 2 * c], A[m * K + 2 * c + 1]);
            r[c] = *reinterpret_cast<const uint32_t*>(&h);
        }
        const uint32_t addr = tbase + ((uint32_t)(warp * 32) << 16) + colA;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     :: "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
            const uint32_t sbo = 128, lbo = 512;
            uint64_t desc = (uint64_t)((smem_u32(bs[warp]) >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                            ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
            const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
            uint32_t mk[4];
            for (int q = 0; q < 4; ++q) mk[q] = q == warp ? 0u : 0xffffffffu;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n}\n"
                         :: "r"(tbase + colD), "r"(tbase + colA), "l"(desc), "r"(idesc), "r"((uint32_t)round),
                            "r"(mk[0]), "r"(mk[1]), "r"(mk[2]), "r"(mk[3]));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar[warp])) : "memory");
        }
        __syncwarp();
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                     :: "r"(smem_u32(&bar[warp])), "r"((uint32_t)round) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    {
        const uint32_t addr = tbase + ((uint32_t)(warp * 32) << 16) + colD;
        uint32_t d[32];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                     "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                     : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                       "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]),
                       "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]),
                       "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int m = warp * 32 + lane;
        for (int n = 0; n < 32; ++n) Dout[m * N + n] = __uint_as_float(d[n]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "r"(64));
}

int main() {
    std::vector<float> A(M * K), B(K * N), D(M * N);
    for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 37) % 17 - 8) / 8.0f;
    for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 11) % 13 - 6) / 4.0f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int twice = 0; twice < 2; ++twice) {
        cudaMemset(dD, 0, D.size() * 4);
        tc_kernel<<<1, 128>>>(dA, dB, dD, twice);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[k * N + n];
                ref *= (twice + 1);
                maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
            }
        printf("accumulate_twice=%d max abs err %g  D[0][0]=%g D[5][7]=%g D[127][31]=%g\n", twice, maxerr, D[0], D[5 * N + 7], D[127 * N + 31]);
    }
    {
        cudaMemset(dD, 0, D.size() * 4);
        tc_kernel_masked<<<1, 128>>>(dA, dB, dD);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[k * N + n];
                ref *= 2 * (m / 32 + 1);
                maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
            }
        printf("masked per-warp max abs err %g  D[0][0]=%g D[100][3]=%g\n", maxerr, D[0], D[100 * N + 3]);
    }
    return 0;
}
