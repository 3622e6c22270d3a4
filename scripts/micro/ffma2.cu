// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, int iters, float a, float b) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, int iters, float a, float b) {
    float2 x[4];
    for (int i = 0; i < 4; ++i) x[i] = make_float2(threadIdx.x * 0.001f + i, i + 0.5f);
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = __ffma2_rn(x[i], a2, b2);
    float s = 0; for (int i = 0; i < 4; ++i) s += x[i].x + x[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: 8 FFMA-equivalents as 4 FFMA2 + 4 IMAD per iteration vs 8 FFMA + 4 IMAD
__global__ void k_mix1(float* out, int iters, float a, float b) {
    float x[8]; int y[4];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
    for (int i = 0; i < 4; ++i) y[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
#pragma unroll
        for (int i = 0; i < 4; ++i) y[i] = y[i] * 3 + it;
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + y[0] + y[1] + y[2] + y[3];
}
__global__ void k_mix2(float* out, int iters, float a, float b) {
    float2 x[4]; int y[4];
    for (int i = 0; i < 4; ++i) x[i] = make_float2(threadIdx.x * 0.001f + i, i + 0.5f);
    for (int i = 0; i < 4; ++i) y[i] = threadIdx.x + i;
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = __ffma2_rn(x[i], a2, b2);
#pragma unroll
        for (int i = 0; i < 4; ++i) y[i] = y[i] * 3 + it;
    }
    float s = 0; for (int i = 0; i < 4; ++i) s += x[i].x + x[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + y[0] + y[1] + y[2] + y[3];
}
int main() {
    float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    auto run = [&](const char* name, void (*k)(float*, int, float, float)) {
        k<<<148 * 8, 256>>>(d, iters, 0.999f, 0.001f);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) k<<<148 * 8, 256>>>(d, iters, 0.999f, 0.001f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        const double fma = 148.0 * 8 * 256 * iters * 8;
        printf("%-6s %.3f ms  %.1f T fp32-FMA/s\n", name, ms, fma / ms / 1e9);
    };
    run("ffma", k_ffma); run("ffma2", k_ffma2); run("mix1", k_mix1); run("mix2", k_mix2);
    return 0;
}
