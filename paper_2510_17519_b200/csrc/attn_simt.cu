// Flash-style attention with fp32 math on CUDA cores: the IEEE-fp32 parity
// path for any head_dim <= 256 and any sequence lengths.
// Online softmax with exp (not exp2) so fp32 results track the fp64 oracle to
// ~1e-7 relative.
#include <cfloat>

#include "attn.h"
#include "epilogue.cuh"
#include "gemm.cuh"

namespace mgv {

namespace {
constexpr int BQ = 32, BK = 32, NT = 256;

template <class T>
__device__ __forceinline__ float ld_el(const void* p, int64_t idx) {
    return to_f(static_cast<const T*>(p)[idx]);
}

inline size_t fwd_smem(int hd) { return sizeof(float) * (2 * BQ * hd + BK * (hd + 1) + BK * hd + BQ * (BK + 1) + 3 * BQ); }
inline size_t bwd_smem(int hd) {
    // Q, dO (BQ x hd) ; K (+1 pad), V (BK x hd) ; S/P, dS (BQ x BK+1) ; acc (BQ or BK x hd, x2) ; lse, D
    return sizeof(float) * (2 * BQ * hd + BK * (hd + 1) + BK * (hd + 1) + 2 * BQ * (BK + 1) + 2 * BK * hd + 2 * BQ);
}
}  // namespace

template <class T>
__global__ void __launch_bounds__(NT) attn_fwd_simt_kernel(AttnProblem p) {
    extern __shared__ float sm[];
    const int hd = p.hd, h = blockIdx.y, q0 = blockIdx.x * BQ, tid = threadIdx.x;
    const int klo = p.seg ? p.seg[2 * (q0 / 128)] : 0, khi = p.seg ? p.seg[2 * (q0 / 128) + 1] : p.Nk;
    float* sQ = sm;
    float* sO = sQ + BQ * hd;
    float* sK = sO + BQ * hd;
    float* sV = sK + BK * (hd + 1);
    float* sS = sV + BK * hd;
    float* sM = sS + BQ * (BK + 1);
    float* sL = sM + BQ;
    float* sA = sL + BQ;
    for (int e = tid; e < BQ * hd; e += NT) {
        const int i = e / hd, d = e % hd, q = q0 + i;
        sQ[e] = q < p.Nq ? ld_el<T>(p.q, (int64_t)q * p.q_ld + h * hd + d) : 0.0f;
        sO[e] = 0.0f;
    }
    if (tid < BQ) {
        sM[tid] = -FLT_MAX;
        sL[tid] = 0.0f;
    }
    for (int k0 = klo; k0 < khi; k0 += BK) {
        __syncthreads();
        for (int e = tid; e < BK * hd; e += NT) {
            const int j = e / hd, d = e % hd, kk = k0 + j;
            const bool in = kk < khi;
            sK[j * (hd + 1) + d] = in ? ld_el<T>(p.k, (int64_t)kk * p.k_ld + h * hd + d) : 0.0f;
            sV[e] = in ? ld_el<T>(p.v, (int64_t)kk * p.v_ld + h * hd + d) : 0.0f;
        }
        __syncthreads();
        for (int e = tid; e < BQ * BK; e += NT) {
            const int i = e / BK, j = e % BK;
            float acc = 0.0f;
            for (int d = 0; d < hd; ++d) acc = fmaf(sQ[i * hd + d], sK[j * (hd + 1) + d], acc);
            sS[i * (BK + 1) + j] = (k0 + j < khi) ? acc : -FLT_MAX;
        }
        __syncthreads();
        if (tid < BQ) {
            float* row = sS + tid * (BK + 1);
            float mx = sM[tid];
            for (int j = 0; j < BK; ++j) mx = fmaxf(mx, row[j]);
            const float alpha = expf(sM[tid] - mx);
            float sum = 0.0f;
            for (int j = 0; j < BK; ++j) {
                const float pj = (k0 + j < khi) ? expf(row[j] - mx) : 0.0f;
                row[j] = pj;
                sum += pj;
            }
            sL[tid] = sL[tid] * alpha + sum;
            sM[tid] = mx;
            sA[tid] = alpha;
        }
        __syncthreads();
        for (int e = tid; e < BQ * hd; e += NT) {
            const int i = e / hd, d = e % hd;
            float o = sO[e] * sA[i];
            const float* row = sS + i * (BK + 1);
            for (int j = 0; j < BK; ++j) o = fmaf(row[j], sV[j * hd + d], o);
            sO[e] = o;
        }
    }
    __syncthreads();
    for (int e = tid; e < BQ * hd; e += NT) {
        const int i = e / hd, d = e % hd, q = q0 + i;
        if (q < p.Nq) static_cast<T*>(p.o)[(int64_t)q * p.o_ld + h * hd + d] = to_t<T>(sO[e] / sL[i]);
    }
    if (tid < BQ && q0 + tid < p.Nq) p.lse[(int64_t)h * lse_stride(p) + q0 + tid] = sM[tid] + logf(sL[tid]);
}

// D[h][q] = sum_d dO * O
template <class T>
__global__ void attn_bwd_dvec_kernel(AttnBwdProblem p) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    const int hd = p.f.hd;
    if (w >= (int64_t)p.f.Nq * p.f.heads) return;
    const int h = static_cast<int>(w % p.f.heads);
    const int64_t q = w / p.f.heads;
    float acc = 0.0f;
    for (int d = lane; d < hd; d += 32)
        acc += ld_el<T>(p.dO, q * p.do_ld + h * hd + d) * ld_el<T>(p.f.o, q * p.f.o_ld + h * hd + d);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
    if (lane == 0) p.Dvec[(int64_t)h * lse_stride(p.f) + q] = acc;
}

// Shared tile math for both backward passes: given sQ, sdO (BQ rows), sK, sV (BK rows), lse/D for the q rows,
// compute P (into sP) and dS (into sdS).
__device__ __forceinline__ void bwd_tile_p_ds(const float* sQ, const float* sdO, const float* sK, const float* sV,
                                              const float* sLse, const float* sD, float* sP, float* sdS, int hd,
                                              int q0, int Nq, int k0, int Nk) {
    for (int e = threadIdx.x; e < BQ * BK; e += NT) {
        const int i = e / BK, j = e % BK;
        float s = 0.0f, dp = 0.0f;
        for (int d = 0; d < hd; ++d) {
            s = fmaf(sQ[i * hd + d], sK[j * (hd + 1) + d], s);
            dp = fmaf(sdO[i * hd + d], sV[j * (hd + 1) + d], dp);
        }
        const bool valid = (q0 + i < Nq) && (k0 + j < Nk);
        const float pr = valid ? expf(s - sLse[i]) : 0.0f;
        sP[i * (BK + 1) + j] = pr;
        sdS[i * (BK + 1) + j] = pr * (dp - sD[i]);  // autodiff.cpp:820
    }
}

template <class T>
__device__ __forceinline__ void load_rows(float* dst, int stride, const void* src, int64_t ld, int r0, int nrows,
                                          int rmax, int h, int hd) {
    for (int e = threadIdx.x; e < nrows * hd; e += NT) {
        const int i = e / hd, d = e % hd, r = r0 + i;
        dst[i * stride + d] = r < rmax ? ld_el<T>(src, (int64_t)r * ld + h * hd + d) : 0.0f;
    }
}

template <class T>
__global__ void __launch_bounds__(NT) attn_bwd_dq_simt_kernel(AttnBwdProblem p) {
    extern __shared__ float sm[];
    const AttnProblem& f = p.f;
    const int hd = f.hd, h = blockIdx.y, q0 = blockIdx.x * BQ, tid = threadIdx.x;
    const int klo = f.seg ? f.seg[2 * (q0 / 128)] : 0, khi = f.seg ? f.seg[2 * (q0 / 128) + 1] : f.Nk;
    float* sQ = sm;
    float* sdO = sQ + BQ * hd;
    float* sK = sdO + BQ * hd;
    float* sV = sK + BK * (hd + 1);
    float* sP = sV + BK * (hd + 1);
    float* sdS = sP + BQ * (BK + 1);
    float* sAcc = sdS + BQ * (BK + 1);
    float* sLse = sAcc + 2 * BK * hd;
    float* sD = sLse + BQ;
    load_rows<T>(sQ, hd, f.q, f.q_ld, q0, BQ, f.Nq, h, hd);
    load_rows<T>(sdO, hd, p.dO, p.do_ld, q0, BQ, f.Nq, h, hd);
    for (int e = tid; e < BQ * hd; e += NT) sAcc[e] = 0.0f;
    if (tid < BQ) {
        const int q = q0 + tid;
        sLse[tid] = q < f.Nq ? f.lse[(int64_t)h * lse_stride(f) + q] : 0.0f;
        sD[tid] = q < f.Nq ? p.Dvec[(int64_t)h * lse_stride(f) + q] : 0.0f;
    }
    for (int k0 = klo; k0 < khi; k0 += BK) {
        __syncthreads();
        load_rows<T>(sK, hd + 1, f.k, f.k_ld, k0, BK, khi, h, hd);
        load_rows<T>(sV, hd + 1, f.v, f.v_ld, k0, BK, khi, h, hd);
        __syncthreads();
        bwd_tile_p_ds(sQ, sdO, sK, sV, sLse, sD, sP, sdS, hd, q0, f.Nq, k0, khi);
        __syncthreads();
        for (int e = tid; e < BQ * hd; e += NT) {  // dQ += dS K
            const int i = e / hd, d = e % hd;
            float acc = sAcc[e];
            for (int j = 0; j < BK; ++j) acc = fmaf(sdS[i * (BK + 1) + j], sK[j * (hd + 1) + d], acc);
            sAcc[e] = acc;
        }
    }
    __syncthreads();
    for (int e = tid; e < BQ * hd; e += NT) {
        const int i = e / hd, d = e % hd, q = q0 + i;
        if (q < f.Nq) static_cast<T*>(p.dq)[(int64_t)q * p.dq_ld + h * hd + d] = to_t<T>(sAcc[e]);
    }
}

template <class T>
__global__ void __launch_bounds__(NT) attn_bwd_dkv_simt_kernel(AttnBwdProblem p) {
    extern __shared__ float sm[];
    const AttnProblem& f = p.f;
    const int hd = f.hd, h = blockIdx.y, k0 = blockIdx.x * BK, split = blockIdx.z, tid = threadIdx.x;
    float* sQ = sm;
    float* sdO = sQ + BQ * hd;
    float* sK = sdO + BQ * hd;
    float* sV = sK + BK * (hd + 1);
    float* sP = sV + BK * (hd + 1);
    float* sdS = sP + BQ * (BK + 1);
    float* sdK = sdS + BQ * (BK + 1);
    float* sdV = sdK + BK * hd;
    float* sLse = sdV + BK * hd;
    float* sD = sLse + BQ;
    load_rows<T>(sK, hd + 1, f.k, f.k_ld, k0, BK, f.Nk, h, hd);
    load_rows<T>(sV, hd + 1, f.v, f.v_ld, k0, BK, f.Nk, h, hd);
    for (int e = tid; e < BK * hd; e += NT) sdK[e] = sdV[e] = 0.0f;
    const int qlo = f.seg ? f.seg[2 * (k0 / 128)] : 0, qhi = f.seg ? f.seg[2 * (k0 / 128) + 1] : f.Nq;
    const int qtiles = (qhi - qlo + BQ - 1) / BQ;
    const int per = (qtiles + p.q_splits - 1) / p.q_splits;
    const int t0 = split * per, t1 = min(qtiles, t0 + per);
    for (int qt = t0; qt < t1; ++qt) {
        const int q0 = qlo + qt * BQ;
        __syncthreads();
        load_rows<T>(sQ, hd, f.q, f.q_ld, q0, BQ, qhi, h, hd);
        load_rows<T>(sdO, hd, p.dO, p.do_ld, q0, BQ, qhi, h, hd);
        if (tid < BQ) {
            const int q = q0 + tid;
            sLse[tid] = q < qhi ? f.lse[(int64_t)h * lse_stride(f) + q] : 0.0f;
            sD[tid] = q < qhi ? p.Dvec[(int64_t)h * lse_stride(f) + q] : 0.0f;
        }
        __syncthreads();
        // packed segments: keys past the tile's own segment end are padding rows (P = 0, so dK = dV = 0 there)
        bwd_tile_p_ds(sQ, sdO, sK, sV, sLse, sD, sP, sdS, hd, q0, qhi, k0, f.seg ? qhi : f.Nk);
        __syncthreads();
        for (int e = tid; e < BK * hd; e += NT) {  // dV += P^T dO ; dK += dS^T Q
            const int j = e / hd, d = e % hd;
            float av = sdV[e], ak = sdK[e];
            for (int i = 0; i < BQ; ++i) {
                av = fmaf(sP[i * (BK + 1) + j], sdO[i * hd + d], av);
                ak = fmaf(sdS[i * (BK + 1) + j], sQ[i * hd + d], ak);
            }
            sdV[e] = av;
            sdK[e] = ak;
        }
    }
    __syncthreads();
    for (int e = tid; e < BK * hd; e += NT) {
        const int j = e / hd, d = e % hd, kk = k0 + j;
        if (kk >= f.Nk) continue;
        if (p.q_splits > 1) {
            float* part = p.dkv_part + (((int64_t)split * f.heads + h) * f.Nk + kk) * 2 * hd;
            part[d] = sdK[e];
            part[hd + d] = sdV[e];
        } else {
            static_cast<T*>(p.dk)[(int64_t)kk * p.dk_ld + h * hd + d] = to_t<T>(sdK[e]);
            static_cast<T*>(p.dv)[(int64_t)kk * p.dv_ld + h * hd + d] = to_t<T>(sdV[e]);
        }
    }
}

template <class T>
__global__ void attn_dkv_reduce_kernel(AttnBwdProblem p) {
    const AttnProblem& f = p.f;
    const int hd = f.hd;
    const int64_t total = (int64_t)f.heads * f.Nk * 2 * hd;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (int s = 0; s < p.q_splits; ++s) acc += p.dkv_part[(int64_t)s * total + e];
        const int c = static_cast<int>(e % (2 * hd));
        const int64_t kk = (e / (2 * hd)) % f.Nk;
        const int h = static_cast<int>(e / (2 * hd * (int64_t)f.Nk));
        if (c < hd)
            static_cast<T*>(p.dk)[kk * p.dk_ld + h * hd + c] = to_t<T>(acc);
        else
            static_cast<T*>(p.dv)[kk * p.dv_ld + h * hd + c - hd] = to_t<T>(acc);
    }
}

template <class T>
void attn_fwd_simt(const AttnProblem& p, cudaStream_t s) {
    const size_t smem = fwd_smem(p.hd);
    ensure_smem(attn_fwd_simt_kernel<T>, 200 * 1024);
    dim3 grid((p.Nq + BQ - 1) / BQ, p.heads);
    attn_fwd_simt_kernel<T><<<grid, NT, smem, s>>>(p); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

template <class T>
void attn_bwd_simt(const AttnBwdProblem& p, cudaStream_t s) {
    const size_t smem = bwd_smem(p.f.hd);
    ensure_smem(attn_bwd_dq_simt_kernel<T>, 200 * 1024);
    ensure_smem(attn_bwd_dkv_simt_kernel<T>, 200 * 1024);
    const int64_t rows = (int64_t)p.f.Nq * p.f.heads;
    attn_bwd_dvec_kernel<T><<<(int)((rows * 32 + 255) / 256), 256, 0, s>>>(p); ::mgv::note_launch();
    attn_bwd_dq_simt_kernel<T><<<dim3((p.f.Nq + BQ - 1) / BQ, p.f.heads), NT, smem, s>>>(p); ::mgv::note_launch();
    attn_bwd_dkv_simt_kernel<T><<<dim3((p.f.Nk + BK - 1) / BK, p.f.heads, p.q_splits), NT, smem, s>>>(p); ::mgv::note_launch();
    if (p.q_splits > 1) {
        const int64_t total = (int64_t)p.f.heads * p.f.Nk * 2 * p.f.hd;
        attn_dkv_reduce_kernel<T><<<(int)((total + 255) / 256), 256, 0, s>>>(p); ::mgv::note_launch();
    }
    MGV_CUDA(cudaGetLastError());
}

// bf16, head_dim % 8 == 0, 16-byte aligned rows: a warp per (query, head), one 16-byte load per lane per operand
__global__ void attn_bwd_dvec_vec_kernel(AttnBwdProblem p) {
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    const int hd = p.f.hd;
    if (w >= (int64_t)p.f.Nq * p.f.heads) return;
    const int h = static_cast<int>(w % p.f.heads);
    const int64_t q = w / p.f.heads;
    float acc = 0.0f;
    for (int c = lane; c < hd / 8; c += 32) {
        const uint4 a = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.dO) + q * p.do_ld + h * hd + 8 * c);
        const uint4 b = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.f.o) + q * p.f.o_ld + h * hd + 8 * c);
        const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&aw[j]));
            const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bw[j]));
            acc = fmaf(fa.x, fb.x, acc);
            acc = fmaf(fa.y, fb.y, acc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
    if (lane == 0) p.Dvec[(int64_t)h * lse_stride(p.f) + q] = acc;
}

void attn_bwd_dvec(const AttnBwdProblem& p, cudaStream_t s) {
    const int64_t rows = (int64_t)p.f.Nq * p.f.heads;
    const bool vec = p.f.hd % 8 == 0 && p.do_ld % 8 == 0 && p.f.o_ld % 8 == 0 &&
                     (reinterpret_cast<uintptr_t>(p.dO) | reinterpret_cast<uintptr_t>(p.f.o)) % 16 == 0;
    if (vec)
        attn_bwd_dvec_vec_kernel<<<(int)((rows * 32 + 255) / 256), 256, 0, s>>>(p);
    else
        attn_bwd_dvec_kernel<__nv_bfloat16><<<(int)((rows * 32 + 255) / 256), 256, 0, s>>>(p);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

template void attn_fwd_simt<float>(const AttnProblem&, cudaStream_t);
template void attn_fwd_simt<__nv_bfloat16>(const AttnProblem&, cudaStream_t);
template void attn_bwd_simt<float>(const AttnBwdProblem&, cudaStream_t);
template void attn_bwd_simt<__nv_bfloat16>(const AttnBwdProblem&, cudaStream_t);

}  // namespace mgv
