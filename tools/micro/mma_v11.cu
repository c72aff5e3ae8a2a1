// Microbenchmark: the tensor-pipe work of one 128-query step of the v11 dK/dV pass in isolation (one issuing
// thread, no TMA, no compute warps, operands resident), against sub-mixes, to split pipe time from latency.
//   mode 0: S^T (9 SS, N=128, B MN-major over two tiles) + dP^T (9 SS) + dV (8 TS, N=144) + dK (8 TS, N=144)
//   mode 1: the 18 SS MMAs only;  mode 2: the 16 TS MMAs only;  mode 3: the 18 SS MMAs at N=64 (v8 shape)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_17519_b200/csrc/ptx.cuh"
using namespace mgv;

constexpr int TT = 144 * 128;  // one HD x 64-token transposed tile
__global__ void __launch_bounds__(128, 1) k(int mode, int steps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    for (int i = threadIdx.x; i < 150000 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3C003C00u;
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t aK = smem_u32(sm), aV = aK + 36864, qt = aV + 36864, dot = qt + 2 * TT;
    if (warp == 1) {
        const uint32_t id128 = idesc_bf16_f32(128, 128, false, true), id64 = idesc_bf16_f32(128, 64, false, true);
        const uint32_t id144 = idesc_bf16_f32(128, 144, false, false);
        unsigned long long best = ~0ull;
        uint32_t ph = 0;
        for (int r = 0; r < 3; ++r) {
            __syncwarp();
            const unsigned long long t0 = clock64();
            if (elect_one()) {
                for (int s = 0; s < steps; ++s) {
                    if (mode != 2)
                        for (int p = 0; p < 2; ++p) {
                            const uint32_t a = p ? aV : aK, b = p ? dot : qt;
                            const uint32_t id = mode == 3 ? id64 : id128;
                            int kk = 0;
                            for (int c = 0; c < 2; ++c)
                                for (int k4 = 0; k4 < 4; ++k4, ++kk)
                                    umma_f16_ss(tmem, smem_desc(a + c * 16384 + k4 * 32, 16, 1024, kSwizzle128),
                                                smem_desc(b + kk * 2048, TT, 1024, kSwizzle128), id, kk > 0);
                            umma_f16_ss(tmem, smem_desc(a + 32768, 16, 256, kSwizzle32),
                                        smem_desc(b + 8 * 2048, TT, 1024, kSwizzle128), id, 1);
                        }
                    if (mode == 0 || mode == 2)
                        for (int p = 0; p < 2; ++p)
                            for (int ks = 0; ks < 8; ++ks)
                                umma_f16_ts(tmem + 192 + p * 144, tmem + 128 + ks * 8,
                                            smem_desc((p ? qt : dot) + (ks >> 2) * TT + (ks & 3) * 32, 16, 1024, kSwizzle128),
                                            id144, 1);
                }
                umma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, ph);
            ph ^= 1;
            const unsigned long long t1 = clock64();
            if (t1 - t0 < best) best = t1 - t0;
        }
        if ((threadIdx.x & 31) == 0) out[blockIdx.x] = best;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    const int SM = 150000;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
    const char* names[4] = {"v11 step (18 SS N128 + 16 TS N144)", "18 SS N=128 only", "16 TS N=144 only",
                            "18 SS N=64 (v8 shape)"};
    const double pipe[4] = {18 * 64 + 16 * 72, 18 * 64, 16 * 72, 18 * 32};
    for (int grid : {1, 148})
        for (int mode = 0; mode < 4; ++mode) {
            unsigned long long h1[148], h2[148];
            k<<<grid, 128, SM>>>(mode, 4, d);
            cudaMemcpy(h1, d, 8 * grid, cudaMemcpyDeviceToHost);
            k<<<grid, 128, SM>>>(mode, 2004, d);
            cudaMemcpy(h2, d, 8 * grid, cudaMemcpyDeviceToHost);
            double worst = 0;
            for (int b = 0; b < grid; ++b) worst = worst > (double)(h2[b] - h1[b]) ? worst : (double)(h2[b] - h1[b]);
            printf("grid %3d %-38s %7.1f clk/step (ideal pipe %5.0f)\n", grid, names[mode], worst / 2000, pipe[mode]);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
