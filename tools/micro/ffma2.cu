// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) throughput on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2 ffma2.cu && ./ffma2
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c)
{
    unsigned long long r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

__global__ void k_scalar(float* out, float m, int iters)
{
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = __fmaf_rn(x[i], m, 0.5f);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_pair(float* out, float m, int iters)
{
    unsigned long long x[8];
    const float2 mm = make_float2(m, m), hh = make_float2(0.5f, 0.5f);
    const unsigned long long M = *(const unsigned long long*)&mm, H = *(const unsigned long long*)&hh;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 v = make_float2(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
        x[i] = *(unsigned long long*)&v;
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], M, H);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 v = *(float2*)&x[i];
        s += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mixed: 8 scalar FFMA + 4 FFMA2 + 8 integer ops per iteration (issue-slot test)
__global__ void k_mix(float* out, float m, int iters, int pair)
{
    float x[8];
    unsigned u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-3f + i; u[i] = threadIdx.x + i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { x[i] = __fmaf_rn(x[i], m, 0.5f); u[i] = u[i] * 3u + 1u; }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i] + (float)u[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    float* d;
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    cudaMalloc(&d, blocks * threads * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a);
        k_scalar<<<blocks, threads>>>(d, 0.999f, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        const double fl = 2.0 * 16 * iters * (double)blocks * threads;
        printf("scalar FFMA : %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(a);
        k_pair<<<blocks, threads>>>(d, 0.999f, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("paired FFMA2: %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    }
    return 0;
}
