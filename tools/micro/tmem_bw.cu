// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM vs number of warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_17519_b200/csrc/ptx.cuh"
using namespace mgv;

__global__ void k(int iters, int mode, unsigned long long* out, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t colb = (warp >> 2) * 64;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    float acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
            tmem_ld32(tmem + lane_base + colb, r);
            tmem_ld32(tmem + lane_base + colb + 32, r);
            tmem_wait_ld();
            acc += __uint_as_float(r[it & 31]);
        } else {
            tmem_st32(tmem + lane_base + colb, r);
            tmem_st32(tmem + lane_base + colb + 32, r);
            tmem_wait_st();
        }
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[0] = acc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* d;
    float* s;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4);
    for (int mode = 0; mode < 2; ++mode)
        for (int warps : {1, 2, 4, 8, 16}) {
            const int iters = 2000;
            k<<<1, warps * 32>>>(iters, mode, d, s);
            k<<<1, warps * 32>>>(iters, mode, d, s);
            unsigned long long c;
            cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
            const double bytes = (double)iters * warps * 32 * 64 * 4;
            printf("%s warps=%2d: %.1f cycles/iter, %.1f B/clk per SM\n", mode ? "st" : "ld", warps,
                   (double)c / iters, bytes / c);
        }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
}
