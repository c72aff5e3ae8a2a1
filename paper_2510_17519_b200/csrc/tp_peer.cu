// Peer-memory tensor-parallel exchange kernels (protocol in tp_peer.h).  HBM / NVLink bound:
// the owner reads P slots of rpr x H fp32 and writes rpr x H to each of the P result regions.
#include "tp_peer.h"

#include "gemm.cuh"

namespace mgv {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void tp_signal_kernel(TpFlagPtrs f, int n, unsigned long long epoch) {
    __threadfence_system();  // the previous kernel's peer stores are visible before the flag
    if (threadIdx.x < n) st_release_sys(f.f[threadIdx.x], epoch);
}

__global__ void tp_wait_kernel(const unsigned long long* flags, int P, unsigned long long epoch) {
    if (threadIdx.x < P)
        while (ld_acquire_sys(flags + threadIdx.x) < epoch) __nanosleep(64);
    __syncthreads();
}

// All P slot loads of an element are issued before the adds (P <= kMaxTp, compile-time unrolled), the sum
// is taken in rank order.  Peer-written data is read with ld.global.cg (L2, no L1 allocation).
template <int PM>
__global__ void __launch_bounds__(256) tp_reduce_gather_kernel(const float* __restrict__ mbox, int P, int64_t slot4,
                                                               int64_t n4, TpDstPtrs dst, int ndst,
                                                               const unsigned long long* flags,
                                                               unsigned long long epoch) {
    if (threadIdx.x < P)
        while (ld_acquire_sys(flags + threadIdx.x) < epoch) __nanosleep(64);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(mbox);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 b[PM];
#pragma unroll
        for (int k = 0; k < PM; ++k)
            if (k < P) b[k] = __ldcg(src + k * slot4 + i);
        float4 a = b[0];
#pragma unroll
        for (int k = 1; k < PM; ++k)
            if (k < P) {
                a.x += b[k].x;
                a.y += b[k].y;
                a.z += b[k].z;
                a.w += b[k].w;
            }
        for (int j = 0; j < ndst; ++j) __stcg(reinterpret_cast<float4*>(dst.p[j]) + i, a);
    }
}

void tp_signal(const TpFlagPtrs& f, int n, uint64_t epoch, cudaStream_t s) {
    tp_signal_kernel<<<1, 32, 0, s>>>(f, n, epoch);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

void tp_wait(const unsigned long long* flags, int P, uint64_t epoch, cudaStream_t s) {
    tp_wait_kernel<<<1, 32, 0, s>>>(flags, P, epoch);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

void tp_reduce_gather(const float* mbox, int P, int64_t rpr, int64_t rows, int64_t H, const TpDstPtrs& dst, int ndst,
                      const unsigned long long* flags, uint64_t epoch, cudaStream_t s) {
    const int64_t n4 = rows > 0 ? rows * H / 4 : 0;
    const int64_t want = (n4 + 255) / 256;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 8LL * num_sms())));
    if (P <= 2)
        tp_reduce_gather_kernel<2><<<grid, 256, 0, s>>>(mbox, P, rpr * H / 4, n4, dst, ndst, flags, epoch);
    else if (P <= 4)
        tp_reduce_gather_kernel<4><<<grid, 256, 0, s>>>(mbox, P, rpr * H / 4, n4, dst, ndst, flags, epoch);
    else
        tp_reduce_gather_kernel<kMaxTp><<<grid, 256, 0, s>>>(mbox, P, rpr * H / 4, n4, dst, ndst, flags, epoch);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

}  // namespace mgv
