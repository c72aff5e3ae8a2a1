// Microbenchmark: the dK/dV v9 per-step MMA mix as cta_group::2 (M = 256) instructions on a 2-CTA cluster,
// issued back to back by the leader (no waits), vs the same shapes per product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_17519_b200/csrc/ptx.cuh"
using namespace mgv;
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(int what, int steps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    const int rank = static_cast<int>(cluster_ctarank());
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc_pair<512>(&slot);
    tc_fence_before(); cluster_sync(); tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t aK = smem_u32(sm), qs = aK + 36864, os = qs + 9216, qh = os + 9216, oh = qh + 9216, vt = oh + 9216;
    if (rank == 0 && warp == 1) {
        const uint32_t id64 = idesc_bf16_f32(256, 64, false, false), id144 = idesc_bf16_f32(256, 144, false, false);
        auto bdesc = [&](uint32_t b, int kk) {
            return kk < 8 ? smem_desc(b + (kk / 4) * 4096 + (kk % 4) * 32, 16, 1024, kSwizzle128)
                          : smem_desc(b + 8192, 16, 256, kSwizzle32);
        };
        uint32_t ph = 0;
        unsigned long long best = ~0ull;
        for (int r = 0; r < 5; ++r) {
            __syncwarp();
            const unsigned long long t0 = clock64();
            if (elect_one()) {
                for (int s = 0; s < steps; ++s) {
                    if (what & 1) {  // S^T SS
                        for (int kk = 0; kk < 8; ++kk)
                            umma_f16_ss_pair(tmem, smem_desc(aK + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, kSwizzle128),
                                             bdesc(qs, kk), id64, kk > 0);
                        umma_f16_ss_pair(tmem, smem_desc(aK + 32768, 16, 256, kSwizzle32), bdesc(qs, 8), id64, 1);
                    }
                    if (what & 2) {  // dP^T TS + SS tail
                        for (int kk = 0; kk < 8; ++kk) umma_f16_ts_pair(tmem + 96, tmem + 448 + kk * 8, bdesc(os, kk), id64, kk > 0);
                        umma_f16_ss_pair(tmem + 96, smem_desc(vt, 16, 256, kSwizzle32), bdesc(os, 8), id64, 1);
                    }
                    if (what & 4) {  // dV, dK TS N=144
                        for (int ks = 0; ks < 4; ++ks)
                            umma_f16_ts_pair(tmem + 160, tmem + 64 + ks * 8, smem_desc(oh + ks * 32, 16, 1024, kSwizzle128), id144, 1);
                        for (int ks = 0; ks < 4; ++ks)
                            umma_f16_ts_pair(tmem + 304, tmem + 96 + (16 * ks / 32) * 32 + (16 * ks % 32) / 2,
                                             smem_desc(qh + ks * 32, 16, 1024, kSwizzle128), id144, 1);
                    }
                }
                umma_commit_pair_mc(&bar, 0x1);
            }
            __syncwarp();
            mbar_wait(&bar, ph);
            ph ^= 1;
            const unsigned long long t1 = clock64();
            if (t1 - t0 < best) best = t1 - t0;
        }
        if ((threadIdx.x & 31) == 0) out[0] = best;
    }
    tc_fence_before(); cluster_sync(); tc_fence_after();
    if (warp == 0) tmem_dealloc_pair<512>(tmem);
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const char* names[] = {"", "S^T SS pair (9)", "dP^T TS pair (8+1)", "S^T+dP^T", "dV+dK TS pair N=144 (8)", "", "", "all 26"};
    for (int what : {1, 2, 4, 7}) {
        unsigned long long h1, h2;
        k<<<2, 128, 100000>>>(what, 4, d);
        cudaMemcpy(&h1, d, 8, cudaMemcpyDeviceToHost);
        k<<<2, 128, 100000>>>(what, 24, d);
        cudaMemcpy(&h2, d, 8, cudaMemcpyDeviceToHost);
        printf("%-26s %.1f clk per step (single-CTA v8 equivalents: S^T 600, dP^T 337, dV+dK 586, all 1287)\n",
               names[what], (h2 - h1) / 20.0);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
