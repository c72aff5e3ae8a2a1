// GEMM epilogue functors.  Every GEMM in the block (tcgen05 bf16 path and the
// IEEE-fp32 SIMT parity path) hands each output row segment
// (row m, columns n0 .. n0+cnt-1, fp32 accumulators) to one of these, so the
// bias / activation / gate / residual work of dit.cpp:288-311 is fused into
// the GEMM that produces the values.
//
// The tensor-core epilogue calls them with cnt == 16 and n0 % 16 == 0; a
// vector path (16-byte loads/stores) is taken whenever the row segment is in
// range and 16-byte aligned, the scalar path otherwise.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace mgv {

template <class T> __device__ __forceinline__ T to_t(float v);
template <> __device__ __forceinline__ float to_t<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 to_t<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float sigmoidf_(float x) { return 1.0f / (1.0f + __expf(-x)); }

__device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// 16 contiguous values <-> registers
template <class T> struct Vec16;
template <> struct Vec16<float> {
    __device__ static void load(const float* p, float* v) {
        const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float4 x = q[i];
            v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
        }
    }
    __device__ static void store(float* p, const float* v) {
        float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
};
template <> struct Vec16<__nv_bfloat16> {
    __device__ static void load(const __nv_bfloat16* p, float* v) {
        const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            uint4 x = q[i];
            const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[j]);
                float2 f = __bfloat1622float2(b);
                v[8 * i + 2 * j] = f.x;
                v[8 * i + 2 * j + 1] = f.y;
            }
        }
    }
    __device__ static void store(__nv_bfloat16* p, const float* v) {
        uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                __nv_bfloat162 b = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
                w[j] = *reinterpret_cast<uint32_t*>(&b);
            }
            q[i] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
};

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
        T* o = out + (int64_t)m * ldo + n0;
        if (cnt == 16 && n0 + 16 <= N && al16(o) && (!bias || al16(bias + n0))) {
            float r[16], b[16];
            if (bias) Vec16<float>::load(bias + n0, b);
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = alpha * (v[j] + (bias ? b[j] : 0.0f));
            Vec16<T>::store(o, r);
            return;
        }
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) o[j] = to_t<T>(alpha * (v[j] + (bias ? bias[n] : 0.0f)));
        }
    }
};

// EpiStore (bf16) that also writes the transposed copy outT[n * ldT + m] (the attention kernels' [heads*hd][tokens]
// operands: V^T, the cross-attention q'^T, dO^T), the same rounded values, so no separate transpose pass is needed.
// Lanes of a warp hold consecutive rows m: each transposed column is one 64-byte coalesced store per warp.
struct EpiStoreT {
    __nv_bfloat16* out;
    int64_t ldo;
    const float* bias;  // may be null
    float alpha;
    int M, N;
    __nv_bfloat16* outT;
    int64_t ldT;
    __device__ __forceinline__ void operator()(int m, int n0, const float* v, int cnt) const {
        if (m >= M) return;
        __nv_bfloat16* o = out + (int64_t)m * ldo + n0;
        float r[16];
        const int c = cnt < 16 ? cnt : 16;
        for (int j = 0; j < c; ++j) r[j] = alpha * (v[j] + (bias && n0 + j < N ? bias[n0 + j] : 0.0f));
        if (cnt == 16 && n0 + 16 <= N && al16(o)) {
            Vec16<__nv_bfloat16>::store(o, r);
        } else {
            for (int j = 0; j < c; ++j)
                if (n0 + j < N) o[j] = __float2bfloat16_rn(r[j]);
        }
        for (int j = 0; j < c; ++j)
            if (n0 + j < N) outT[(int64_t)(n0 + j) * ldT + m] = __float2bfloat16_rn(r[j]);
    }
};

// Tensor-parallel row-parallel GEMM (attn.out / xattn.out / ffn.out and their dgrad conjugates):
// the epilogue performs the reduce-scatter transfer of the TP exchange tile by tile.  Row m of this rank's
// fp32 partial goes straight into this rank's slot of the mailbox of the rank that owns rows
// [o*rpr, (o+1)*rpr), over NVLink peer memory for o != self (tp_peer.cu sums the slots in rank order).
constexpr int kMaxTp = 8;
struct EpiF32Peer {
    void* box[kMaxTp];  // box[o]: this rank's slot (rpr x ldo) in owner o's mailbox
    int64_t ldo;
    float alpha;
    int rpr, M, N;
    int bf16;  // payload: 0 fp32 (the bits EpiF32 writes), 1 bf16 (half the NVLink bytes)
    __device__ __forceinline__ void operator()(int m, int n0, const float* v, int cnt) const {
        if (m >= M) return;
        const int o = m / rpr;
        const int64_t off = (int64_t)(m - o * rpr) * ldo + n0;
        float r[16];
        const int c = cnt < 16 ? cnt : 16;
        for (int j = 0; j < c; ++j) r[j] = alpha * (v[j] + 0.0f);
        if (bf16) {
            __nv_bfloat16* p = static_cast<__nv_bfloat16*>(box[o]) + off;
            if (cnt == 16 && n0 + 16 <= N && al16(p)) {
                Vec16<__nv_bfloat16>::store(p, r);
                return;
            }
            for (int j = 0; j < c; ++j)
                if (n0 + j < N) p[j] = __float2bfloat16_rn(r[j]);
            return;
        }
        float* p = static_cast<float*>(box[o]) + off;
        if (cnt == 16 && n0 + 16 <= N && al16(p)) {
            Vec16<float>::store(p, r);
            return;
        }
        for (int j = 0; j < c; ++j)
            if (n0 + j < N) p[j] = r[j];
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
        float* o = out + (int64_t)m * ldo + n0;
        if (cnt == 16 && n0 + 16 <= N && al16(o) && (!bias || al16(bias + n0))) {
            float r[16], b[16], prev[16];
            if (bias) Vec16<float>::load(bias + n0, b);
            if (accumulate) Vec16<float>::load(o, prev);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                r[j] = alpha * (v[j] + (bias ? b[j] : 0.0f));
                if (accumulate) r[j] = __fadd_rn(r[j], prev[j]);  // no FMA: the sum of rounded partials
            }
            Vec16<float>::store(o, r);
            return;
        }
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float r = alpha * (v[j] + (bias ? bias[n] : 0.0f));
                o[j] = accumulate ? __fadd_rn(o[j], r) : r;
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
        T* zo = z + (int64_t)m * ld + n0;
        T* ho = h + (int64_t)m * ld + n0;
        if (cnt == 16 && n0 + 16 <= N && al16(zo) && al16(ho) && al16(bias + n0)) {
            float b[16], zz[16], hh[16];
            Vec16<float>::load(bias + n0, b);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                zz[j] = v[j] + b[j];
                hh[j] = zz[j] * sigmoidf_(zz[j]);
            }
            Vec16<T>::store(zo, zz);
            Vec16<T>::store(ho, hh);
            return;
        }
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float zz = v[j] + bias[n];
                zo[j] = to_t<T>(zz);
                ho[j] = to_t<T>(zz * sigmoidf_(zz));
            }
        }
    }
};

// y = acc + b ; X = Xin + y * gate[mod_id[m], n]   (dit.cpp:295-297, 310-311)
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
        const float* g = gate + (int64_t)mod_id[m] * gate_ld + n0;
        float* x = X + (int64_t)m * ldx + n0;
        const float* xi = Xin + (int64_t)m * ldx + n0;
        T* yo = y ? y + (int64_t)m * ldy + n0 : nullptr;
        if (cnt == 16 && n0 + 16 <= N && al16(x) && al16(xi) && al16(g) && al16(bias + n0) && (!yo || al16(yo))) {
            float b[16], gg[16], xx[16], yy[16];
            Vec16<float>::load(bias + n0, b);
            Vec16<float>::load(g, gg);
            Vec16<float>::load(xi, xx);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                yy[j] = v[j] + b[j];
                xx[j] = xx[j] + yy[j] * gg[j];
            }
            if (yo) Vec16<T>::store(yo, yy);
            Vec16<float>::store(x, xx);
            return;
        }
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float yy = v[j] + bias[n];
                if (yo) yo[j] = to_t<T>(yy);
                x[j] = xi[j] + yy * g[j];
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
        T* o = out + (int64_t)m * ld + n0;
        const T* zi = z + (int64_t)m * ld + n0;
        if (cnt == 16 && n0 + 16 <= N && al16(o) && al16(zi)) {
            float zz[16], r[16];
            Vec16<T>::load(zi, zz);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float s = sigmoidf_(zz[j]);
                r[j] = v[j] * (s + zz[j] * s * (1.0f - s));
            }
            Vec16<T>::store(o, r);
            return;
        }
        for (int j = 0; j < cnt; ++j) {
            int n = n0 + j;
            if (n < N) {
                float zz = to_f(zi[j]);
                float s = sigmoidf_(zz);
                o[j] = to_t<T>(v[j] * (s + zz * s * (1.0f - s)));
            }
        }
    }
};

}  // namespace mgv

namespace mgv {

// ---- whole-tile epilogues: the GEMM hands the functor one output row of a BN-column tile through a chunk
// loader (ld(c, v): 16 fp32 accumulators of columns [16c, 16c+16), executed by all 32 lanes of the warp, so
// the functor's control flow around it must be warp-uniform) instead of 16-column segments.
template <class Epi>
struct IsTileEpi {
    static constexpr bool value = false;
};

// Rotation of one (x0, x1) pair, explicit roundings so every kernel that applies it (this epilogue and
// qk_norm_rope_vec) produces the same bits:  (x0 c - x1 s, x0 s + x1 c)   (autodiff.cpp:864-865)
__device__ __forceinline__ void rope_pair(float x0, float x1, float c, float sn, float& o0, float& o1) {
    o0 = __fmaf_rn(x0, c, -__fmul_rn(x1, sn));
    o1 = __fmaf_rn(x0, sn, __fmul_rn(x1, c));
}

// QKV projection with the QK-L2-norm x temperature and the 3-D RoPE fused into its epilogue (dit.cpp:288-294,
// SURVEY K6).  The GEMM runs with BN = head_dim (HD), so every output tile is one whole head of q, k or v for
// 128 tokens; each epilogue thread owns one token row of it:
//   pass 1  raw = bf16(acc + bias)  -> qkv (kept for the backward and for V);  q/k: the 18 lane partials of
//           sum(raw^2) that qk_norm_rope_vec forms (lane l: fmaf over elements [8l, 8l+8)), then its xor
//           butterfly order, so iq / ik and the rotated output are bit-identical to the separate kernel;
//   pass 2  (q/k only) re-read the accumulators, raw * (1/|raw| [* temp_h]), rotate pairs with the row's
//           (cos, sin) table -> qk.
// V tiles take pass 1 only.  Layout as QKLayout: raw q|k|v chunks of Hl columns at stride ld, rotated q|k at
// stride qk_ld (k at qk_koff), inverse norms at iq / ik [m * i_ld + head].
template <int HD>
struct EpiQKNormRope {
    __nv_bfloat16* qkv;
    int64_t ld;
    const float* bias;
    __nv_bfloat16* qk;
    int64_t qk_ld, qk_koff;
    int64_t hl;  // columns per q|k|v chunk (heads * HD)
    const float* temp;
    const float2* cs;  // (N, HD/2) (cos, sin)
    float* iq;
    float* ik;
    int64_t i_ld;
    int M;
    __nv_bfloat16* qkT;  // optional: rotated q | k transposed ([2 hl][ldT]), the attention backward's Q^T / K^T
    int64_t ldT;
    // ldi(c, r): issue the tcgen05.ld of accumulator chunk c into r (16 x u32); wt(): wait for the issued loads.
    // Both passes keep the next chunk's TMEM load (and its bias / RoPE rows) in flight under the current chunk's math.
    template <class LDI, class WT>
    __device__ __forceinline__ void tile_row(int m, int n0, LDI&& ldi, WT&& wt) const {
        constexpr int NC = HD / 16, NP = HD / 8;  // 16-column chunks; 8-element lane partials
        static_assert(HD % 16 == 0 && NP <= 32, "head_dim");
        const int region = static_cast<int>(n0 / hl);  // 0 q, 1 k, 2 v (warp-uniform)
        const int h = static_cast<int>((n0 - region * hl) / HD);
        const bool ok = m < M;
        const float4* bias4 = reinterpret_cast<const float4*>(bias + n0);
        float part[NP];
        uint32_t r[2][16];
        float4 b[2][4];
        ldi(0, r[0]);
#pragma unroll
        for (int q = 0; q < 4; ++q) b[0][q] = bias4[q];
        wt();
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int cur = c & 1, nxt = cur ^ 1;
            if (c + 1 < NC) {
                ldi(c + 1, r[nxt]);
#pragma unroll
                for (int q = 0; q < 4; ++q) b[nxt][q] = bias4[4 * (c + 1) + q];
            }
            const float* bb = reinterpret_cast<const float*>(b[cur]);
            float v[16];
            uint32_t w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                __nv_bfloat162 p2 = __floats2bfloat162_rn(__uint_as_float(r[cur][2 * j]) + bb[2 * j],
                                                          __uint_as_float(r[cur][2 * j + 1]) + bb[2 * j + 1]);
                w[j] = *reinterpret_cast<uint32_t*>(&p2);
                const float2 f = __bfloat1622float2(p2);
                v[2 * j] = f.x;
                v[2 * j + 1] = f.y;
            }
            if (ok) {
                uint4* o = reinterpret_cast<uint4*>(qkv + (int64_t)m * ld + n0 + 16 * c);
                o[0] = make_uint4(w[0], w[1], w[2], w[3]);
                o[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                float ss = 0.0f;
#pragma unroll
                for (int e = 0; e < 8; ++e) ss = fmaf(v[8 * hh + e], v[8 * hh + e], ss);
                part[2 * c + hh] = ss;
            }
            if (c + 1 < NC) wt();
        }
        if (region == 2) return;
        // the xor butterfly of a 32-lane warp_sum as seen by lane 0 (lanes >= NP contribute 0)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int l = 0; l < o; ++l)
                if (l + o < NP) part[l] = part[l] + part[l + o];
        const float iv = 1.0f / sqrtf(part[0] + 1e-6f);  // autodiff.cpp:727
        if (ok) (region == 0 ? iq : ik)[(int64_t)m * i_ld + h] = iv;
        const float sc = region == 0 ? iv * temp[h] : iv;  // dit.cpp:292
        const float4* csr = reinterpret_cast<const float4*>(cs + (int64_t)(ok ? m : 0) * (HD / 2));
        float4 t[2][4];
        ldi(0, r[0]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            b[0][q] = bias4[q];
            t[0][q] = csr[q];
        }
        wt();
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int cur = c & 1, nxt = cur ^ 1;
            if (c + 1 < NC) {
                ldi(c + 1, r[nxt]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    b[nxt][q] = bias4[4 * (c + 1) + q];
                    t[nxt][q] = csr[4 * (c + 1) + q];
                }
            }
            const float* bb = reinterpret_cast<const float*>(b[cur]);
            float o[16];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float2 f = __bfloat1622float2(__floats2bfloat162_rn(__uint_as_float(r[cur][2 * k]) + bb[2 * k],
                                                                          __uint_as_float(r[cur][2 * k + 1]) + bb[2 * k + 1]));
                const float4 tt = t[cur][k >> 1];
                const float cc = (k & 1) ? tt.z : tt.x, sn = (k & 1) ? tt.w : tt.y;
                rope_pair(__fmul_rn(f.x, sc), __fmul_rn(f.y, sc), cc, sn, o[2 * k], o[2 * k + 1]);
            }
            if (ok) {
                Vec16<__nv_bfloat16>::store(qk + (int64_t)m * qk_ld + region * qk_koff + h * HD + 16 * c, o);
                if (qkT) {
                    __nv_bfloat16* tp = qkT + (region * hl + h * HD + 16 * c) * ldT + m;
#pragma unroll
                    for (int j = 0; j < 16; ++j) tp[j * ldT] = __float2bfloat16_rn(o[j]);
                }
            }
            if (c + 1 < NC) wt();
        }
    }
};
template <int HD>
struct IsTileEpi<EpiQKNormRope<HD>> {
    static constexpr bool value = true;
};

}  // namespace mgv
