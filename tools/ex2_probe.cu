// ex2_probe.cu -- measures the error of the rasterizer's alpha evaluation
// alpha = o * ex2.approx.ftz.f32(p) (fp32 product rounded to nearest) against the
// oracle's o * 2^p (2^p in fp64, product rounded once to fp32), exhaustively over
// every fp32 p in [-30, 0] and a grid of opacities.  Prints the worst relative
// deviation of ex2.approx from 2^p and of alpha_gpu from alpha_oracle, in units of
// 2^-24, which bounds the O14 alpha band (reading Q20).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ex2_probe.cu -o /tmp/ex2_probe
#include <cstdio>
#include <cstdint>
#include <cmath>

__device__ __forceinline__ float ex2_ftz(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(r) : "f"(x));
    return r;
}

__device__ unsigned long long g_max_ex2, g_max_alpha;   // max rel err * 2^40 (integer for atomicMax)

__global__ void probe(uint32_t lo_bits, uint32_t n, const float* ops, int n_ops) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t bits = lo_bits + i;           // negative floats: bits increase as p decreases
    const float p = __uint_as_float(bits);
    const double ex = exp2((double)p);
    const float e = ex2_ftz(p);
    double r = fabs((double)e - ex) / ex;
    unsigned long long q = (unsigned long long)(r * 1099511627776.0);
    atomicMax(&g_max_ex2, q);
    double ra = 0;
    for (int k = 0; k < n_ops; ++k) {
        const float o = ops[k];
        const float ag = __fmul_rn(o, e);
        const float ao = (float)((double)o * ex);
        if (ao < 1e-30f) continue;
        ra = fmax(ra, fabs((double)ag - (double)ao) / (double)ao);
    }
    atomicMax(&g_max_alpha, (unsigned long long)(ra * 1099511627776.0));
}

int main() {
    const int n_ops = 16;
    float h_ops[n_ops];
    for (int k = 0; k < n_ops; ++k) h_ops[k] = (float)(0.004 + (1.0 - 0.004) * k / (n_ops - 1));
    h_ops[1] = 1.0f / 255.0f * 1.5f;
    float* ops;
    cudaMalloc(&ops, sizeof(h_ops));
    cudaMemcpy(ops, h_ops, sizeof(h_ops), cudaMemcpyHostToDevice);
    // p in [-30, -0]: bit patterns from 0x80000000 (-0) to bits(-30)
    const float lo = -30.0f;
    uint32_t b_hi;
    memcpy(&b_hi, &lo, 4);
    const uint32_t b0 = 0x80000000u;
    const uint64_t total = (uint64_t)b_hi - b0 + 1;
    const uint32_t chunk = 1u << 28;
    for (uint64_t s = 0; s < total; s += chunk) {
        const uint32_t n = (uint32_t)std::min<uint64_t>(chunk, total - s);
        probe<<<(n + 255) / 256, 256>>>(b0 + (uint32_t)s, n, ops, n_ops);
    }
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long me, ma;
    cudaMemcpyFromSymbol(&me, g_max_ex2, 8);
    cudaMemcpyFromSymbol(&ma, g_max_alpha, 8);
    const double re = me / 1099511627776.0, ra = ma / 1099511627776.0;
    printf("{\"p_range\": [-30, 0], \"n_p\": %llu, \"ex2_max_rel\": %.6e, \"ex2_max_rel_in_2^-24\": %.3f, "
           "\"alpha_max_rel\": %.6e, \"alpha_max_rel_in_2^-24\": %.3f, \"cuda\": \"%s\"}\n",
           (unsigned long long)total, re, re * 16777216.0, ra, ra * 16777216.0, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
