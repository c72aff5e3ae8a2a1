// Microbenchmark: MUFU.EX2 and FFMA throughput per SM (warps x independent chains).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kex(int iters, float* out, unsigned long long* clk) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    __syncthreads();
    const unsigned long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void kfma(int iters, float* out, unsigned long long* clk) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A800000;" : "+f"(x[i]));
    __syncthreads();
    const unsigned long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void kcvt(int iters, float* out, unsigned long long* clk) {
    float x[8]; unsigned int y[8];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-3f + i; y[i] = 0; }
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(y[i]) : "f"(x[i]), "f"(x[(i + 1) & 7]));
    __syncthreads();
    const unsigned long long t1 = clock64();
    unsigned s = 0;
    for (int i = 0; i < 8; ++i) s += y[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) clk[0] = t1 - t0;
}
__global__ void kmix(int iters, float* out, unsigned long long* clk) {  // 1 ex2 : 1 cvt (pairs) : 3 fma
    float x[8]; unsigned int y[4] = {0, 0, 0, 0};
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A800000;" : "+f"(x[i]));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A800000;" : "+f"(x[i]));
            asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0f3A800000;" : "+f"(x[i]));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(y[i]) : "f"(x[2 * i]), "f"(x[2 * i + 1]));
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[threadIdx.x] = s + y[0] + y[1] + y[2] + y[3];
    if (threadIdx.x == 0) clk[0] = t1 - t0;
}
int main() {
    float* o; unsigned long long* c;
    cudaMalloc(&o, 4096 * 4); cudaMalloc(&c, 8);
    for (int w : {4, 8, 16, 32}) {
        const int it = 4096;
        unsigned long long h;
        kex<<<1, w * 32>>>(it, o, c); kex<<<1, w * 32>>>(it, o, c);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("ex2  warps=%2d: %.2f lanes/clk/SM\n", w, (double)it * 8 * w * 32 / h);
        kfma<<<1, w * 32>>>(it, o, c); kfma<<<1, w * 32>>>(it, o, c);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("ffma warps=%2d: %.2f lanes/clk/SM\n", w, (double)it * 8 * w * 32 / h);
        kcvt<<<1, w * 32>>>(it, o, c); kcvt<<<1, w * 32>>>(it, o, c);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("cvt  warps=%2d: %.2f lanes/clk/SM\n", w, (double)it * 8 * w * 32 / h);
        kmix<<<1, w * 32>>>(it, o, c); kmix<<<1, w * 32>>>(it, o, c);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("mix  warps=%2d: %.2f elements/clk/SM (ex2-bound would be 16)\n", w, (double)it * 8 * w * 32 / h);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
