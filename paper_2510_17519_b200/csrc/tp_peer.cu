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

__global__ void __launch_bounds__(256) tp_reduce_gather_kernel(const float* __restrict__ mbox, int P, int64_t slot4,
                                                               int64_t n4, TpDstPtrs dst, int ndst,
                                                               const unsigned long long* flags,
                                                               unsigned long long epoch) {
    if (threadIdx.x < P)
        while (ld_acquire_sys(flags + threadIdx.x) < epoch) __nanosleep(64);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(mbox);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 a = __ldcv(src + i);  // written by peers over NVLink: bypass L1
        for (int k = 1; k < P; ++k) {
            const float4 b = __ldcv(src + k * slot4 + i);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        for (int j = 0; j < ndst; ++j) reinterpret_cast<float4*>(dst.p[j])[i] = a;
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
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 4LL * num_sms())));
    tp_reduce_gather_kernel<<<grid, 256, 0, s>>>(mbox, P, rpr * H / 4, n4, dst, ndst, flags, epoch);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

}  // namespace mgv
