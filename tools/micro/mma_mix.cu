// Microbenchmark: the per-step tensor-pipe work of the attention backward passes in isolation (one CTA, one
// issuing thread, no TMA, no compute warps), to separate pipe time from in-kernel interference.
//   dkv8: S^T = K Q^T (SS, 8 SW128 k-steps + 1 SW32 tail, B MN-major N=64), dP^T = V dO^T (8 TS + 1 SS),
//         dV += P^T dO (4 TS, N=144, B K-major), dK += dS^T Q (4 TS, N=144)
//   dq:   S = Q K^T (9 TS, N=64, B MN-major), dP = dO V^T (9 TS), dQ += dS K (4 TS, N=144)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_17519_b200/csrc/ptx.cuh"
using namespace mgv;

__device__ volatile int g_stop;
// interf bit 0: 8 warps stream tcgen05.ld (32 cols) + tcgen05.st (16 cols) like the compute warps;
// interf bit 1: 4 warps write shared memory at the TMA rate of the real kernel (36 KB per step, no conflicts)
__global__ void __launch_bounds__(448, 1) k(int mode, int steps, int interf, int fill, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, bar2, bar3;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        mbar_init(&bar3, 1);
        mbar_arrive(&bar3);  // phase 0 complete: waits on it return at once
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    if (fill) {  // random bf16 operands (shared memory and the TMEM A operands), like real data
        uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
        for (int i = threadIdx.x; i < 80000 / 4; i += blockDim.x) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            const uint32_t lo = 0x3C00u | (x & 0x83FFu), hi = 0x3C00u | ((x >> 16) & 0x83FFu);  // ~U(+-1..2) bf16
            reinterpret_cast<uint32_t*>(sm)[i] = lo | (hi << 16);
        }
        if (warp < 4) {
            uint32_t r[32];
            for (int c = 0; c < 32; ++c) {
                x ^= x << 13; x ^= x >> 17; x ^= x << 5;
                r[c] = (0x3C00u | (x & 0x83FFu)) | ((0x3C00u | ((x >> 16) & 0x83FFu)) << 16);
            }
            const uint32_t lb = static_cast<uint32_t>(warp * 32) << 16;
            for (int c0 = 0; c0 < 512; c0 += 32) tmem_st16(tmem + lb + c0, r), tmem_st16(tmem + lb + c0 + 16, r + 16);
            tmem_wait_st();
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    const uint32_t aK = smem_u32(sm);               // 128 x 144 row tile: 2 x 16 KB SW128 + 4 KB SW32
    const uint32_t qt = aK + 36864;                 // 144 x 64 transposed tile (SW128), 18 KB
    const uint32_t dot = qt + 18432;
    const uint32_t vt = dot + 18432;                // 128 x 16 SW32 tail
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (warp >= 6 && (interf & 1)) {  // compute-warp TMEM traffic: lane group g = warp & 3
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const int hf = (warp - 6) >> 2;
        uint32_t r[32];
        for (int i = 0; i < 32; ++i) r[i] = i;
        while (!done) {
            tmem_ld32(tmem + lane_base + 0 + hf * 32, r);
            tmem_wait_ld();
            tmem_st16(tmem + lane_base + 64 + hf * 16, r);
            tmem_wait_st();
            tmem_ld32(tmem + lane_base + 96 + hf * 32, r);
            tmem_wait_ld();
            tmem_st16(tmem + lane_base + 96 + hf * 32, r);
            tmem_wait_st();
        }
    }
    if (warp >= 2 && warp < 6 && (interf & 2)) {  // smem writes into a scratch region
        uint32_t base = smem_u32(sm) + 80000 + (warp - 2) * 4096;
        while (!done) {
            for (int u = 0; u < 8; ++u)
                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + u * 512 + (threadIdx.x & 31) * 16),
                             "r"(u));
            __nanosleep(64);
        }
    }
    if (warp == 1) {
        uint32_t ph = 0;
        unsigned long long best = ~0ull;
        const uint32_t id64 = idesc_bf16_f32(128, 64, false, true), id144 = idesc_bf16_f32(128, 144, false, false);
        for (int r = 0; r < 5; ++r) {
            __syncwarp();
            const unsigned long long t0 = clock64();
            if (elect_one()) {
                auto sep = [&]() {
                    if (interf & 8) umma_commit(&bar2);
                    if (interf & 16) mbar_wait(&bar3, 0);
                    if (interf & 4) tc_fence_after();
                };
                for (int s = 0; s < steps; ++s) {
                    if (mode == 0) {
                        int kk = 0;
                        for (int c = 0; c < 2; ++c)
                            for (int k4 = 0; k4 < 4; ++k4, ++kk)
                                umma_f16_ss(tmem + 0, smem_desc(aK + c * 16384 + k4 * 32, 16, 1024, kSwizzle128),
                                            smem_desc(qt + kk * 2048, 16, 1024, kSwizzle128), id64, kk > 0);
                        umma_f16_ss(tmem + 0, smem_desc(aK + 32768, 16, 256, kSwizzle32),
                                    smem_desc(qt + 8 * 2048, 16, 1024, kSwizzle128), id64, 1);
                        sep();
                        for (int k8 = 0; k8 < 8; ++k8)
                            umma_f16_ts(tmem + 96, tmem + 448 + k8 * 8, smem_desc(dot + k8 * 2048, 16, 1024, kSwizzle128),
                                        id64, k8 > 0);
                        umma_f16_ss(tmem + 96, smem_desc(vt, 16, 256, kSwizzle32),
                                    smem_desc(dot + 8 * 2048, 16, 1024, kSwizzle128), id64, 1);
                        sep();
                        for (int ks = 0; ks < 4; ++ks)
                            umma_f16_ts(tmem + 160, tmem + 64 + ks * 8, smem_desc(dot + ks * 32, 16, 1024, kSwizzle128),
                                        id144, 1);
                        sep();
                        for (int ks = 0; ks < 4; ++ks)
                            umma_f16_ts(tmem + 304, tmem + 96 + (16 * ks / 32) * 32 + (16 * ks % 32) / 2,
                                        smem_desc(qt + ks * 32, 16, 1024, kSwizzle128), id144, 1);
                        sep();
                    } else {
                        for (int b = 0; b < 2; ++b)
                            for (int kk = 0; kk < 9; ++kk)
                                umma_f16_ts(tmem + b * 64, tmem + (b ? 440 : 368) + kk * 8,
                                            smem_desc((b ? dot : qt) + kk * 2048, 16, 1024, kSwizzle128), id64, kk > 0);
                        for (int ks = 0; ks < 4; ++ks)
                            umma_f16_ts(tmem + 224, tmem + 192 + ks * 8, smem_desc(qt + ks * 32, 16, 1024, kSwizzle128),
                                        id144, 1);
                    }
                }
                umma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, ph);
            ph ^= 1;
            const unsigned long long t1 = clock64();
            if (t1 - t0 < best) best = t1 - t0;
        }
        if ((threadIdx.x & 31) == 0) {
            out[blockIdx.x] = best;
            done = 1;
        }
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 296 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    for (int grid : {1, 148})
        for (int fill : {0, 1})
        for (int interf : {0})
            for (int mode = 0; mode < 2; ++mode) {
                unsigned long long h1[296], h2[296];
                const int LONG = 20000;
                k<<<grid, 448, 100000>>>(mode, 4, interf, fill, d);
                cudaMemcpy(h1, d, 8 * grid, cudaMemcpyDeviceToHost);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                k<<<grid, 448, 100000>>>(mode, LONG, interf, fill, d);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(h2, d, 8 * grid, cudaMemcpyDeviceToHost);
                double worst = 0;
                for (int b = 0; b < grid; ++b) worst = worst > (double)(h2[b] - h1[b]) ? worst : (double)(h2[b] - h1[b]);
                printf("fill %d grid %3d %s: %.1f clk per step (%d steps x 5 reps, %.1f ms wall, %.0f MHz effective)\n", fill, grid,
                       mode == 0 ? "dkv v8" : "dq    ", worst / (LONG - 4), LONG, ms,
                       worst * 5.0 / (ms * 1e3) * (grid > 148 ? 0.5 : 1.0));
            }
    // 148 CTAs at once (one per SM): the same, with every SM's tensor pipe busy (power / clock effects excluded:
    // clock64 counts SM cycles)
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
