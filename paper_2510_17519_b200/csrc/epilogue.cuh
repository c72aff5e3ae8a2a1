// GEMM epilogue functors.  Every GEMM in the block (tcgen05 bf16 path and the
// IEEE-fp32 SIMT parity path) hands each output row segment
// (row m, columns n0 .. n0+cnt-1, fp32 accumulators) to one of these, so the
// bias / activation / gate / residual work of dit.cpp:288-311 is fused into
// the GEMM that produces the values.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace mgv {

template <class T> __device__ __forceinline__ T to_t(float v);
template <> __device__ __forceinline__ float to_t<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 to_t<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + expf(-x)); }

// out[m, n] = alpha * (acc + bias[n])                     (plain linear + bias)
template <class T>
struct EpiStore {
    T* out;
    int64_t ldo;
    const float* bias;  // may be null
    float alpha;
    int M, N;
    __device__ __forceinline__ void operator()(int m, int n0, const float* v, int cnt) const {
        if (m >= M) return;
        T* o = out + (int64_t)m * ldo;
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) o[n] = to_t<T>(alpha * (v[j] + (bias ? bias[n] : 0.0f)));
        }
    }
};

// fp32 output, optionally accumulating into what is there (dgrad into dX, wgrad over samples)
struct EpiF32 {
    float* out;
    int64_t ldo;
    const float* bias;
    float alpha;
    int accumulate;
    int M, N;
    __device__ __forceinline__ void operator()(int m, int n0, const float* v, int cnt) const {
        if (m >= M) return;
        float* o = out + (int64_t)m * ldo;
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float r = alpha * (v[j] + (bias ? bias[n] : 0.0f));
                o[n] = accumulate ? o[n] + r : r;
            }
        }
    }
};

// z = acc + b ; h = silu(z)  (dit.cpp:309; autodiff.cpp:263-266)
template <class T>
struct EpiBiasSilu {
    T* z;
    T* h;
    int64_t ld;
    const float* bias;
    int M, N;
    __device__ __forceinline__ void operator()(int m, int n0, const float* v, int cnt) const {
        if (m >= M) return;
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float zz = v[j] + bias[n];
                z[(int64_t)m * ld + n] = to_t<T>(zz);
                h[(int64_t)m * ld + n] = to_t<T>(zz * sigmoidf_(zz));
            }
        }
    }
};

// y = acc + b ; X += y * gate[mod_id[m], n]   (dit.cpp:295-297, 310-311)
// y is kept (bf16/fp32) for the gate gradient of the backward pass.
template <class T>
struct EpiGateResid {
    const float* Xin;
    float* X;  // out (may alias Xin)
    int64_t ldx;
    T* y;  // may be null
    int64_t ldy;
    const float* bias;
    const float* gate;  // row u of the modulation table, pre-offset to the gate chunk
    int64_t gate_ld;
    const int32_t* mod_id;
    int M, N;
    __device__ __forceinline__ void operator()(int m, int n0, const float* v, int cnt) const {
        if (m >= M) return;
        const float* g = gate + (int64_t)mod_id[m] * gate_ld;
        float* x = X + (int64_t)m * ldx;
        const float* xi = Xin + (int64_t)m * ldx;
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float yy = v[j] + bias[n];
                if (y) y[(int64_t)m * ldy + n] = to_t<T>(yy);
                x[n] = xi[n] + yy * g[n];
            }
        }
    }
};

// dz = acc * silu'(z)   (autodiff.cpp:267-275), the FFN-in backward fused into the FFN-out dgrad
template <class T>
struct EpiSiluBwd {
    T* out;
    const T* z;
    int64_t ld;
    int M, N;
    __device__ __forceinline__ void operator()(int m, int n0, const float* v, int cnt) const {
        if (m >= M) return;
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float zz = to_f(z[(int64_t)m * ld + n]);
                float s = sigmoidf_(zz);
                out[(int64_t)m * ld + n] = to_t<T>(v[j] * (s + zz * s * (1.0f - s)));
            }
        }
    }
};

}  // namespace mgv
