// Microbenchmark: how many tcgen05.mma instructions can be outstanding before the issuing thread stalls
// (issue-return clock of each of 48 back-to-back MMAs, 128x64x16 TS ~34 clk and 128x144x16 SS ~107 clk).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_17519_b200/csrc/ptx.cuh"
using namespace mgv;
__global__ void __launch_bounds__(128, 1) k(int ss, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, ss == 2 ? 2 : 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a = smem_u32(sm), b = a + 32768;
    if (ss == 2 && (warp == 1 || warp == 2) && elect_one()) {  // two issuing warps, 24 TS N=64 MMAs each
        const uint32_t id = idesc_bf16_f32(128, 64, false, false);
        const unsigned long long t0 = clock64();
        for (int i = 0; i < 24; ++i)
            umma_f16_ts(tmem + (warp - 1) * 64, tmem + 448 + (i & 3) * 8, smem_desc(b + (i & 3) * 32, 16, 1024, kSwizzle128),
                        id, i > 0);
        const unsigned long long t1 = clock64();
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        const unsigned long long e = clock64();
        out[(warp - 1) * 2] = t1 - t0;
        out[(warp - 1) * 2 + 1] = e - t0;
    }
    if (ss < 2 && warp == 1 && elect_one()) {
        const uint32_t id = idesc_bf16_f32(128, ss ? 144 : 64, false, false);
        unsigned long long t[49];
        t[0] = clock64();
        for (int i = 0; i < 48; ++i) {
            if (ss)
                umma_f16_ss(tmem, smem_desc(a + (i & 3) * 32, 16, 1024, kSwizzle128),
                            smem_desc(b + (i & 3) * 32, 16, 1024, kSwizzle128), id, i > 0);
            else
                umma_f16_ts(tmem, tmem + 448 + (i & 3) * 8, smem_desc(b + (i & 3) * 32, 16, 1024, kSwizzle128), id, i > 0);
            t[i + 1] = clock64();
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        const unsigned long long e = clock64();
        for (int i = 0; i <= 48; ++i) out[i] = t[i] - t[0];
        out[49] = e - t[0];
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    for (int ss = 0; ss < 2; ++ss) {
        unsigned long long h[50];
        k<<<1, 128, 100000>>>(ss, d);
        k<<<1, 128, 100000>>>(ss, d);
        cudaMemcpy(h, d, 50 * 8, cudaMemcpyDeviceToHost);
        printf("%s issue-return clocks:", ss ? "SS N=144" : "TS N=64 ");
        for (int i = 1; i <= 48; ++i) printf(" %llu", h[i]);
        printf("  | complete %llu\n", h[49]);
    }
    {
        unsigned long long h[4];
        k<<<1, 128, 100000>>>(2, d);
        k<<<1, 128, 100000>>>(2, d);
        cudaMemcpy(h, d, 4 * 8, cudaMemcpyDeviceToHost);
        printf("two issuers x 24 TS N=64: issue %llu / %llu clk, complete %llu / %llu (one issuer, 48: see above)\n", h[0],
               h[2], h[1], h[3]);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
