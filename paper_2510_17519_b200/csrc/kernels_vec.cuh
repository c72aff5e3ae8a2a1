// Vectorised row kernels for the bf16 path (H % 8 == 0): each thread owns 8-column groups
// g = tid, tid + 256 (16-byte bf16 / 2 x 16-byte fp32 accesses) and two rows are processed per
// block reduction.  Same math and the same fixed-order reductions as the scalar kernels in
// kernels_elem.cu (which remain the fp32-mode / odd-width path).
#pragma once
#include <cuda_bf16.h>

#include "epilogue.cuh"

namespace mgv {
namespace vec {

constexpr int RT = 256;
constexpr int VG = 2;  // 8-column groups per thread -> H <= 4096
constexpr int R = 2;   // rows per block reduction

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* v) {
    const uint4 x = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
        v[2 * j] = f.x;
        v[2 * j + 1] = f.y;
    }
}
__device__ __forceinline__ void ld8(const float* p, float* v) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        w[j] = *reinterpret_cast<uint32_t*>(&b);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ void st8(float* p, const float* v) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// R-wide fixed-order block sum (all threads get the same values)
__device__ __forceinline__ void block_sum_r(float* v, float (*red)[RT / 32]) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[r] += __shfl_xor_sync(0xffffffff, v[r], o);
    const int w = threadIdx.x / 32;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int r = 0; r < R; ++r) red[r][w] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        float s = 0.0f;
#pragma unroll
        for (int i = 0; i < RT / 32; ++i) s += red[r][i];
        v[r] = s;
    }
    __syncthreads();
}

}  // namespace vec
}  // namespace mgv
