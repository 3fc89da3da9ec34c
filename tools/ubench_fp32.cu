// Microbenchmark: FP32 pipe throughput on sm_100a for scalar FFMA, packed FFMA2 (f32x2),
// and a P2P-like mix (FADD/FMUL/FFMA + MUFU.RSQ) in scalar and packed form.
// Prints FMA-lane-ops per SM per clock (clock64-based), which decides the FP32 roofline
// denominator and whether packing helps issue-bound kernels.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters, float a) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, 0.5f * i + 1.0f);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma_reg(float* out, int iters, float a, float b) {
    float x[8], c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 0.001f + i; c[i] = b * i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, c[i]);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters, float a, float b) {
    float2 x[8], c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); c[i] = make_float2(b * i, b + i); }
    const float2 a2 = make_float2(a, a);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], a2, c[i]);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// P2P body, 4 targets, scalar
__global__ void k_p2p_scalar(const float4* src, float* out, int iters) {
    float x[4], y[4], z[4], f[4] = {0, 0, 0, 0}, gx[4] = {0, 0, 0, 0}, gy[4] = {0, 0, 0, 0}, gz[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 4; ++k) { x[k] = threadIdx.x * 1e-3f + k; y[k] = 0.3f * k; z[k] = 0.1f; }
    __shared__ float4 s[256];
    s[threadIdx.x] = src[threadIdx.x];
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        for (int j = 0; j < 256; ++j) {
            const float4 sj = s[j];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float dx = sj.x - x[k], dy = sj.y - y[k], dz = sj.z - z[k];
                const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                const float inv = rsqrtf(r2);
                const float qi = sj.w * inv;
                const float qi3 = qi * (inv * inv);
                f[k] += qi;
                gx[k] = fmaf(qi3, dx, gx[k]);
                gy[k] = fmaf(qi3, dy, gy[k]);
                gz[k] = fmaf(qi3, dz, gz[k]);
            }
        }
    }
    float acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += f[k] + gx[k] + gy[k] + gz[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// P2P body, 4 targets as 2 packed pairs; sources duplicated {x,x,y,y},{z,z,q,q}
__global__ void k_p2p_packed(const float4* src, float* out, int iters) {
    float2 x[2], y[2], z[2], f[2], gx[2], gy[2], gz[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        x[k] = make_float2(-(threadIdx.x * 1e-3f + 2 * k), -(threadIdx.x * 1e-3f + 2 * k + 1));
        y[k] = make_float2(-0.6f * k, -0.6f * k - 0.3f); z[k] = make_float2(-0.1f, -0.1f);  // negated
        f[k] = gx[k] = gy[k] = gz[k] = make_float2(0.f, 0.f);
    }
    __shared__ float4 s[256];
    s[threadIdx.x] = src[threadIdx.x];
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        for (int j = 0; j < 256; ++j) {
            const float4 sj = s[j];
            const float2 sx = make_float2(sj.x, sj.x), sy = make_float2(sj.y, sj.y), sz = make_float2(sj.z, sj.z);
            const float2 sq = make_float2(sj.w, sj.w);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const float2 dx = __fadd2_rn(sx, x[k]), dy = __fadd2_rn(sy, y[k]), dz = __fadd2_rn(sz, z[k]);
                const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
                const float2 inv = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
                const float2 qi = __fmul2_rn(sq, inv);
                const float2 qi3 = __fmul2_rn(qi, __fmul2_rn(inv, inv));
                f[k] = __fadd2_rn(f[k], qi);
                gx[k] = __ffma2_rn(qi3, dx, gx[k]);
                gy[k] = __ffma2_rn(qi3, dy, gy[k]);
                gz[k] = __ffma2_rn(qi3, dz, gz[k]);
            }
        }
    }
    float acc = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) acc += f[k].x + f[k].y + gx[k].x + gy[k].y + gz[k].x + gz[k].y + gx[k].y + gy[k].x;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_rsq(float* out, int iters) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1.0f + threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = rsqrtf(x[i]);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
    int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int nsm = pr.multiProcessorCount;
    printf("%s sms=%d clock_attr=%d kHz\n", pr.name, nsm, clk_khz);
    float* out; cudaMalloc(&out, 1 << 26);
    float4* src; cudaMalloc(&src, 256 * 16); cudaMemset(src, 0, 256 * 16);
    const double ghz = 1.965;
    for (int blocks_per_sm : {4, 8}) {
        const int nb = nsm * blocks_per_sm, nt = 256, it = 4096;
        double lanes = (double)nb * nt;
        float ms = timeit([&] { k_ffma<<<nb, nt>>>(out, it, 0.999f); });
        double fma = lanes * it * 16 * 8;
        printf("FFMA imm     bps=%d: %.3f ms  %.1f FMA/clk/SM (at 1.965 GHz)\n", blocks_per_sm, ms, fma / (ms * 1e-3) / nsm / (ghz * 1e9));
        ms = timeit([&] { k_ffma_reg<<<nb, nt>>>(out, it, 0.999f, 0.5f); });
        printf("FFMA reg     bps=%d: %.3f ms  %.1f FMA/clk/SM\n", blocks_per_sm, ms, fma / (ms * 1e-3) / nsm / (ghz * 1e9));
        ms = timeit([&] { k_ffma2<<<nb, nt>>>(out, it, 0.999f, 0.5f); });
        printf("FFMA2        bps=%d: %.3f ms  %.1f FMA/clk/SM (lane-ops)\n", blocks_per_sm, ms, 2 * fma / (ms * 1e-3) / nsm / (ghz * 1e9));
        ms = timeit([&] { k_rsq<<<nb, nt>>>(out, it / 4); });
        printf("MUFU.RSQ     bps=%d: %.3f ms  %.1f RSQ/clk/SM\n", blocks_per_sm, ms, fma / 4 / (ms * 1e-3) / nsm / (ghz * 1e9));
        const int it2 = 64;
        double inter = lanes * it2 * 256 * 4;
        ms = timeit([&] { k_p2p_scalar<<<nb, nt>>>(src, out, it2); });
        printf("P2P scalar   bps=%d: %.3f ms  %.2f inter/clk/SM  %.3e inter/s\n", blocks_per_sm, ms, inter / (ms * 1e-3) / nsm / (ghz * 1e9), inter / (ms * 1e-3));
        ms = timeit([&] { k_p2p_packed<<<nb, nt>>>(src, out, it2); });
        printf("P2P packed   bps=%d: %.3f ms  %.2f inter/clk/SM  %.3e inter/s\n", blocks_per_sm, ms, inter / (ms * 1e-3) / nsm / (ghz * 1e9), inter / (ms * 1e-3));
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
