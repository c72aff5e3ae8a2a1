// Microbenchmark: tcgen05.mma kind::f16 throughput (clk per 128xNx16 MMA) vs N, operand majors, A source,
// and accumulate-chain dependence.  One CTA, one issuing thread, 64 MMAs then one commit.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2510_17519_b200/csrc/ptx.cuh"
using namespace mgv;
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

struct Cfg { int N; bool ts; bool a_mn; bool b_mn; bool chain; };

__global__ void __launch_bounds__(128, 1) k(Cfg c, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&slot);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a = smem_u32(sm), b = a + 65536;
    if (warp == 1) {
        const uint32_t id = idesc_bf16_f32(128, c.N, c.a_mn, c.b_mn);
        const uint64_t bd0 = smem_desc(b, c.b_mn ? 8192 : 16, 1024, kSwizzle128);
        const uint64_t ad0 = smem_desc(a, c.a_mn ? 8192 : 16, 1024, kSwizzle128);
        const uint32_t bstep = c.b_mn ? (2048 >> 4) : (32 >> 4), astep = c.a_mn ? (2048 >> 4) : (32 >> 4);
        uint32_t ph = 0;
        unsigned long long best = ~0ull;
        for (int r = 0; r < 10; ++r) {
            __syncwarp();
            const unsigned long long t0 = clock64();
            if (elect_one()) {
                for (int o = 0; o < 4; ++o) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const uint32_t d = tmem + (c.chain ? 0 : (i & 1) * 256);
                        const uint64_t bd = bd0 + (i & 3) * bstep;
                        if (c.ts)
                            umma_f16_ts(d, tmem + 480 + (i & 3) * 8, bd, id, c.chain ? (o + i > 0) : 0);
                        else
                            umma_f16_ss(d, ad0 + (i & 3) * astep, bd, id, c.chain ? (o + i > 0) : 0);
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
        if (lane_id() == 0) out[0] = best;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    printf("%-4s %-3s %-5s %-5s %-6s  clk/MMA  ideal  eff\n", "N", "A", "A_mn", "B_mn", "chain");
    for (int N : {64, 128, 144, 256})
        for (int ts = 1; ts >= 0; --ts)
            for (int amn = 0; amn < (ts ? 1 : 2); ++amn)
                for (int bmn = 0; bmn < 2; ++bmn)
                    for (int ch = 1; ch >= 0; --ch) {
                        if (N > 256 / (ch ? 1 : 1) && 0) continue;
                        Cfg c{N, ts != 0, amn != 0, bmn != 0, ch != 0};
                        if (!ch && N > 240) continue;  // two D buffers must fit
                        k<<<1, 128, 200000>>>(c, d);
                        unsigned long long h;
                        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                        const double per = (h - 700.0) / 64.0, ideal = 128.0 * N / 256.0;
                        printf("%-4d %-3s %-5d %-5d %-6d  %6.1f  %5.1f  %4.0f%%\n", N, ts ? "tm" : "sm", amn, bmn, ch, per,
                               ideal, 100.0 * ideal / per);
                    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
