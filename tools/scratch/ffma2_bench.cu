// Microbenchmark: FFMA (3-reg) vs FFMA2 (packed f32x2) vs FFMA with immediate
// throughput on one B200 (many warps, independent chains).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void k_ffma(float* out, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < ITERS; ++i) {
        x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
        x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__device__ __forceinline__ unsigned long long pk(float x, float y) {
    unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y)); return r;
}
__global__ void k_ffma2(float* out, float a, float b) {
    float t = threadIdx.x;
    unsigned long long x0 = pk(t, t + 1), x1 = pk(t + 2, t + 3), x2 = pk(t + 4, t + 5), x3 = pk(t + 6, t + 7);
    unsigned long long x4 = pk(t + 8, t + 9), x5 = pk(t + 10, t + 11), x6 = pk(t + 12, t + 13), x7 = pk(t + 14, t + 15);
    const unsigned long long A = pk(a, a), B = pk(b, b);
    for (int i = 0; i < ITERS; ++i) {
#define F(x) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(A), "l"(B));
        F(x0) F(x1) F(x2) F(x3) F(x4) F(x5) F(x6) F(x7)
    }
    float s = 0, u, v;
#define U(x) asm("mov.b64 {%0, %1}, %2;" : "=f"(u), "=f"(v) : "l"(x)); s += u + v;
    U(x0) U(x1) U(x2) U(x3) U(x4) U(x5) U(x6) U(x7)
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); k_ffma<<<148 * 8, 256>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double n = 148.0 * 8 * 256 * ITERS * 8;
        printf("FFMA : %.3f ms  %.2f TFMA/s\n", ms, n / ms / 1e9);
        cudaEventRecord(e0); k_ffma2<<<148 * 8, 256>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        n = 148.0 * 8 * 256 * ITERS * 16;
        printf("FFMA2: %.3f ms  %.2f TFMA/s\n", ms, n / ms / 1e9);
    }
    return 0;
}
