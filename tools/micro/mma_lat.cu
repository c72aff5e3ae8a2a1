// Microbenchmark: tcgen05.mma issue->commit latency and back-to-back throughput for the attention shapes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_17519_b200/csrc/ptx.cuh"
using namespace mgv;

__global__ void __launch_bounds__(128, 1) k(int reps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a = smem_u32(sm), b = a + 36864;
    if (threadIdx.x == 0) {
        uint32_t ph = 0;
        constexpr uint32_t id64_ts = idesc_bf16_f32(128, 64, false, true);
        constexpr uint32_t id144 = idesc_bf16_f32(128, 144, false, false);
        for (int mode = 0; mode < 4; ++mode) {
            for (int n : {1, 8}) {  // n groups back to back, then one commit
                unsigned long long best = ~0ull;
                for (int r = 0; r < reps; ++r) {
                    const unsigned long long t0 = clock64();
                    for (int g = 0; g < n; ++g) {
                        if (mode == 0)  // TS, N=64, K=144 (9 MMAs)
                            for (int kk = 0; kk < 9; ++kk)
                                umma_f16_ts(tmem + 64 * (g & 1), tmem + 400 + kk * 8,
                                            smem_desc(b + kk * 2048, 16, 1024, kSwizzle128), id64_ts, kk > 0);
                        else if (mode == 1)  // SS, N=64, K=144
                            for (int kk = 0; kk < 9; ++kk)
                                umma_f16_ss(tmem + 64 * (g & 1),
                                            smem_desc(a + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kSwizzle128),
                                            smem_desc(b + kk * 2048, 16, 1024, kSwizzle128), id64_ts, kk > 0);
                        else if (mode == 2)  // TS, N=144, K=64 (4 MMAs)
                            for (int ks = 0; ks < 4; ++ks)
                                umma_f16_ts(tmem + 128 + 144 * (g & 1), tmem + 400 + ks * 8,
                                            smem_desc(b + ks * 32, 16, 1024, kSwizzle128), id144, ks > 0);
                        else  // SS N=144 K=64
                            for (int ks = 0; ks < 4; ++ks)
                                umma_f16_ss(tmem + 128 + 144 * (g & 1), smem_desc(a + ks * 32, 16, 1024, kSwizzle128),
                                            smem_desc(b + ks * 32, 16, 1024, kSwizzle128), id144, ks > 0);
                    }
                    umma_commit(&bar);
                    mbar_wait(&bar, ph);
                    ph ^= 1;
                    const unsigned long long t1 = clock64();
                    if (t1 - t0 < best) best = t1 - t0;
                }
                out[mode * 2 + (n == 8)] = best;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    k<<<1, 128, 200000>>>(20, d);
    unsigned long long h[8];
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    const char* nm[4] = {"TS N=64 K=144", "SS N=64 K=144", "TS N=144 K=64", "SS N=144 K=64"};
    const double ideal[4] = {288, 288, 288, 288};
    for (int m = 0; m < 4; ++m)
        printf("%-14s latency(1 group) %5llu clk   8 groups %6llu clk -> %.0f clk/group (ideal %.0f)\n", nm[m],
               h[2 * m], h[2 * m + 1], h[2 * m + 1] / 8.0, ideal[m]);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
