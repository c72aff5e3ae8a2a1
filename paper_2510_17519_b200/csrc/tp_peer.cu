// Peer-memory tensor-parallel exchange kernels (protocol in tp_peer.h).  HBM / NVLink bound:
// the owner reads P slots of rpr x H payload (fp32 or bf16) and writes rpr x H to each of the P result regions.
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
// One 16-byte vector: 4 fp32 or 8 bf16 elements of a slot / result row.
template <class E>
struct TpVec;
template <>
struct TpVec<float> {
    static constexpr int kElems = 4;
    __device__ static void load(const uint4& u, float* f) {
        f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y); f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
    }
    __device__ static uint4 store(const float* f) {
        return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
    }
};
template <>
struct TpVec<__nv_bfloat16> {
    static constexpr int kElems = 8;
    __device__ static void load(const uint4& u, float* f) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
            f[2 * j] = t.x;
            f[2 * j + 1] = t.y;
        }
    }
    __device__ static uint4 store(const float* f) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
            w[j] = *reinterpret_cast<uint32_t*>(&b);
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};

// E: payload element (fp32 or bf16); the sum is always taken in fp32, in rank order.
template <int PM, class E>
__global__ void __launch_bounds__(256) tp_reduce_gather_kernel(const void* __restrict__ mbox, int P, int64_t slot_v,
                                                               int64_t nv, TpDstPtrs dst, int ndst,
                                                               const unsigned long long* flags,
                                                               unsigned long long epoch) {
    constexpr int NE = TpVec<E>::kElems;
    if (threadIdx.x < P)
        while (ld_acquire_sys(flags + threadIdx.x) < epoch) __nanosleep(64);
    __syncthreads();
    const uint4* src = static_cast<const uint4*>(mbox);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
        uint4 b[PM];
#pragma unroll
        for (int k = 0; k < PM; ++k)
            if (k < P) b[k] = __ldcg(src + k * slot_v + i);
        float a[NE], t[NE];
        TpVec<E>::load(b[0], a);
#pragma unroll
        for (int k = 1; k < PM; ++k)
            if (k < P) {
                TpVec<E>::load(b[k], t);
#pragma unroll
                for (int e = 0; e < NE; ++e) a[e] += t[e];
            }
        const uint4 o = TpVec<E>::store(a);
        for (int j = 0; j < ndst; ++j) __stcg(static_cast<uint4*>(dst.p[j]) + i, o);
    }
}

__global__ void tp_bf16_to_f32_kernel(const uint4* __restrict__ in, int64_t nv, float4* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
        float f[8];
        TpVec<__nv_bfloat16>::load(in[i], f);
        out[2 * i] = make_float4(f[0], f[1], f[2], f[3]);
        out[2 * i + 1] = make_float4(f[4], f[5], f[6], f[7]);
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

template <class E>
static void reduce_gather_launch(const void* mbox, int P, int64_t rpr, int64_t rows, int64_t H, const TpDstPtrs& dst,
                                 int ndst, const unsigned long long* flags, uint64_t epoch, cudaStream_t s) {
    constexpr int NE = TpVec<E>::kElems;
    const int64_t nv = rows > 0 ? rows * H / NE : 0, slot_v = rpr * H / NE;
    const int64_t want = (nv + 255) / 256;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, 8LL * num_sms())));
    if (P <= 2)
        tp_reduce_gather_kernel<2, E><<<grid, 256, 0, s>>>(mbox, P, slot_v, nv, dst, ndst, flags, epoch);
    else if (P <= 4)
        tp_reduce_gather_kernel<4, E><<<grid, 256, 0, s>>>(mbox, P, slot_v, nv, dst, ndst, flags, epoch);
    else
        tp_reduce_gather_kernel<kMaxTp, E><<<grid, 256, 0, s>>>(mbox, P, slot_v, nv, dst, ndst, flags, epoch);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

void tp_reduce_gather(const void* mbox, bool bf16, int P, int64_t rpr, int64_t rows, int64_t H, const TpDstPtrs& dst,
                      int ndst, const unsigned long long* flags, uint64_t epoch, cudaStream_t s) {
    if (bf16)
        reduce_gather_launch<__nv_bfloat16>(mbox, P, rpr, rows, H, dst, ndst, flags, epoch, s);
    else
        reduce_gather_launch<float>(mbox, P, rpr, rows, H, dst, ndst, flags, epoch, s);
}

void tp_bf16_to_f32(const void* in, int64_t n, float* out, cudaStream_t s) {
    const int64_t nv = n / 8;
    if (nv <= 0) return;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((nv + 255) / 256, 8LL * num_sms())));
    tp_bf16_to_f32_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(in), nv, reinterpret_cast<float4*>(out));
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

}  // namespace mgv
