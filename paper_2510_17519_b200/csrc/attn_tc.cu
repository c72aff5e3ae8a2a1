// tcgen05 flash attention forward for sm_100a (bf16 operands, fp32 softmax and
// accumulation) -- Tape::mha forward (autodiff.cpp:755-793) at head_dim 144.
//
// One CTA per (128-query tile, head):
//   warp 0      TMA producer: Q once, then K and V^T tiles (128 keys) through a
//               2-stage ring
//   warp 1      MMA issuer: S_j = Q K_j^T into TMEM buffer j%2, then
//               O += P_{j-1} V_{j-1} with P read straight from TMEM (the TS form)
//   warp 2      TMEM allocator: columns [0,128) S/P 0, [128,256) S/P 1, [256,256+hd) O
//   warps 4..7  softmax, thread i = query row i = TMEM lane i: tcgen05.ld S ->
//               online softmax in the log2 domain (ex2.approx) -> bf16 P written
//               back over S with tcgen05.st -> signal.  O is rescaled in TMEM only
//               when the running max grows by more than 2^8 (stale-max trick); the
//               epilogue normalises O and writes lse.
//
// P lives in TMEM in the buffer its S came from, so softmax(j+1) never waits for
// the P.V product of step j (only a rare O rescale does); the tensor core runs
// S_{j+1} and PV_j back to back while the softmax warps work.
//
// head_dim 144 = 64 + 64 + 16: Q and K tiles are 64-column SW128 chunks plus a
// 16-column SW32 tail (S = Q K^T walks 9 K-steps across them); V is consumed
// transposed (V^T tile = hd rows x 128 keys, K-major) so O += P V is ONE
// N = 144 MMA per 16-key step.
#include <cfloat>

#include "attn.h"
#include "gemm.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace mgv {

namespace {

constexpr int BM = 128;  // queries per CTA
constexpr int BN = 128;  // keys per tile
constexpr float kLog2e = 1.4426950408889634f;

template <int HD>
struct FwdCfg {
    static constexpr int NF = HD / 64;
    static constexpr int TAIL = HD % 64;
    static_assert(TAIL == 0 || TAIL == 16, "head_dim must be 64k or 64k+16");
    static constexpr int QK_TILE = NF * 16384 + (TAIL ? 4096 : 0);  // 128 rows x HD (K-major over hd)
    static constexpr int VT_CHUNK = HD * 128;                        // HD rows x 64 keys (SW128)
    static constexpr int VT_TILE = 2 * VT_CHUNK;                     // HD rows x 128 keys
    static constexpr int STAGE = QK_TILE + VT_TILE;
    static constexpr int SMEM = QK_TILE + 2 * STAGE + 1024 + 256;
    static constexpr int O_COL = 256;
};

struct FwdMaps {
    CUtensorMap q128, q32, k128, k32, vt;
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

template <int HD>
__device__ __forceinline__ void load_qk_tile(uint8_t* dst, const CUtensorMap* m128, const CUtensorMap* m32,
                                             uint64_t* bar, int col0, int row0) {
    using C = FwdCfg<HD>;
#pragma unroll
    for (int c = 0; c < C::NF; ++c) tma_load_2d(dst + c * 16384, m128, bar, col0 + c * 64, row0);
    if (C::TAIL) tma_load_2d(dst + C::NF * 16384, m32, bar, col0 + C::NF * 64, row0);
}

}  // namespace

template <int HD>
__global__ void __launch_bounds__(256, 1) attn_fwd_tc_kernel(const __grid_constant__ FwdMaps tm, AttnProblem p) {
    using C = FwdCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sStage = sQ + C::QK_TILE;  // [2] x (K tile | V^T tile)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + 2 * C::STAGE);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;    // [2]
    uint64_t* v_full = bars + 3;    // [2]
    uint64_t* kv_empty = bars + 5;  // [2]
    uint64_t* s_full = bars + 7;    // [2]
    uint64_t* p_full = bars + 9;    // [2]
    uint64_t* pv_done = bars + 11;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BM;
    const int nkv = (p.Nk + BN - 1) / BN;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
        }
        mbar_init(pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            tma_prefetch(&tm.q128);
            tma_prefetch(&tm.k128);
            tma_prefetch(&tm.vt);
            mbar_arrive_expect_tx(q_full, C::QK_TILE);
            load_qk_tile<HD>(sQ, &tm.q128, &tm.q32, q_full, col, q0);
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                if (j >= 2) mbar_wait(&kv_empty[st], ((j - 2) >> 1) & 1);
                uint8_t* sK = sStage + st * C::STAGE;
                uint8_t* sVt = sK + C::QK_TILE;
                mbar_arrive_expect_tx(&k_full[st], C::QK_TILE);
                load_qk_tile<HD>(sK, &tm.k128, &tm.k32, &k_full[st], col, j * BN);
                mbar_arrive_expect_tx(&v_full[st], C::VT_TILE);
                tma_load_2d(sVt, &tm.vt, &v_full[st], j * BN, col);
                tma_load_2d(sVt + C::VT_CHUNK, &tm.vt, &v_full[st], j * BN + 64, col);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idS = idesc_bf16_f32(BM, BN, false, false);
        constexpr uint32_t idO = idesc_bf16_f32(BM, HD, false, false);
        const uint32_t aQ = smem_u32(sQ);
        mbar_wait(q_full, 0);
        for (int j = 0; j <= nkv; ++j) {
            if (j < nkv) {
                const int st = j & 1;
                const uint32_t aK = smem_u32(sStage + st * C::STAGE);
                mbar_wait(&k_full[st], (j >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    // S_j -> TMEM buffer j%2 (P_{j-2} there was consumed by PV_{j-2}, issued earlier)
                    const uint32_t d = tmem + st * BN;
                    int kk = 0;
#pragma unroll
                    for (int c = 0; c < C::NF; ++c)
#pragma unroll
                        for (int k = 0; k < 4; ++k, ++kk)
                            umma_f16_ss(d, smem_desc(aQ + c * 16384 + k * 32, 16, 1024, kSwizzle128),
                                        smem_desc(aK + c * 16384 + k * 32, 16, 1024, kSwizzle128), idS, kk > 0);
                    if (C::TAIL)
                        umma_f16_ss(d, smem_desc(aQ + C::NF * 16384, 16, 256, kSwizzle32),
                                    smem_desc(aK + C::NF * 16384, 16, 256, kSwizzle32), idS, 1);
                    umma_commit(&s_full[st]);
                }
                __syncwarp();
            }
            if (j >= 1) {
                const int jp = j - 1, sp = jp & 1;
                mbar_wait(&p_full[sp], (jp >> 1) & 1);
                mbar_wait(&v_full[sp], (jp >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t aVt = smem_u32(sStage + sp * C::STAGE + C::QK_TILE);
                    const uint32_t pt = tmem + sp * BN;  // bf16 P packed 2 per column
#pragma unroll
                    for (int ks = 0; ks < BN / 16; ++ks)
                        umma_f16_ts(tmem + C::O_COL, pt + ks * 8,
                                    smem_desc(aVt + (ks >> 2) * C::VT_CHUNK + (ks & 3) * 32, 16, 1024, kSwizzle128),
                                    idO, (jp > 0 || ks > 0) ? 1u : 0u);
                    umma_commit(pv_done);
                    umma_commit(&kv_empty[sp]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        const int wq = warp - 4;
        const int row = wq * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
        float m2 = -FLT_MAX;  // running max (log2 domain)
        float l = 0.0f;
        for (int j = 0; j < nkv; ++j) {
            const int sb = j & 1;
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            tc_fence_after();
            float s[BN];
#pragma unroll
            for (int c = 0; c < BN / 32; ++c)
                tmem_ld32(tmem + lane_base + sb * BN + c * 32, reinterpret_cast<uint32_t*>(s + c * 32));
            tmem_wait_ld();
            const int kv0 = j * BN;
            if (kv0 + BN > p.Nk) {
#pragma unroll
                for (int c = 0; c < BN; ++c)
                    if (kv0 + c >= p.Nk) s[c] = -FLT_MAX;
            }
            // row max over raw logits with 8 independent chains (short dependency depth)
            float mx8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx8[e] = s[e];
#pragma unroll
            for (int c = 8; c < BN; c += 8)
#pragma unroll
                for (int e = 0; e < 8; ++e) mx8[e] = fmaxf(mx8[e], s[c + e]);
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * kLog2e;
            float alpha = 1.0f, m_use = m2;
            if (j == 0) {
                m_use = mx;
            } else if (mx > m2 + 8.0f) {
                m_use = mx;
                alpha = ex2(m2 - mx);
            }
            // p = 2^(s*log2e - m): one FFMA + one MUFU per element; 8 independent partial sums
            float ps8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) ps8[e] = 0.0f;
            uint32_t pk[BN / 2];
#pragma unroll
            for (int c = 0; c < BN; c += 2) {
                const float p0 = ex2(fmaf(s[c], kLog2e, -m_use)), p1 = ex2(fmaf(s[c + 1], kLog2e, -m_use));
                ps8[(c / 2) & 7] += p0 + p1;
                pk[c / 2] = pack_bf16(p0, p1);
            }
            const float ps = ((ps8[0] + ps8[1]) + (ps8[2] + ps8[3])) + ((ps8[4] + ps8[5]) + (ps8[6] + ps8[7]));
            if (j >= 1 && __any_sync(0xffffffff, alpha != 1.0f)) {
                // O must hold exactly PV_0..PV_{j-1} before it is rescaled
                mbar_wait(pv_done, (j - 1) & 1);
                tc_fence_after();
                const uint32_t ob = tmem + lane_base + C::O_COL;
#pragma unroll 1
                for (int c = 0; c < HD / 16; ++c) {
                    uint32_t r[16];
                    tmem_ld16(ob + c * 16, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
                    tmem_st16(ob + c * 16, r);
                }
            }
            l = l * alpha + ps;
            m2 = m_use;
            // P (bf16) over S in the same TMEM buffer: 64 packed columns
            tmem_st32(tmem + lane_base + sb * BN, pk);
            tmem_st32(tmem + lane_base + sb * BN + 32, pk + 32);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[sb]);
        }
        if (nkv > 0) {
            mbar_wait(pv_done, (nkv - 1) & 1);
            tc_fence_after();
        }
        const int q = q0 + row;
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.o) + (int64_t)q * p.o_ld + col;
#pragma unroll 1
        for (int c = 0; c < HD / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(tmem + lane_base + C::O_COL + c * 16, r);
            tmem_wait_ld();
            if (q < p.Nq) {
                uint32_t o[8];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    o[e] = pack_bf16(__uint_as_float(r[2 * e]) * inv, __uint_as_float(r[2 * e + 1]) * inv);
                uint4* dst = reinterpret_cast<uint4*>(out + c * 16);
                dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
                dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
            }
        }
        if (q < p.Nq) p.lse[(int64_t)h * p.Nq + q] = (m2 + __log2f(l)) * 0.6931471805599453f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host
bool attn_tc_supported(int hd, int Nk) {
    (void)Nk;
    return hd == 64 || hd == 128 || hd == 144;
}

template <int HD>
static void launch_fwd(const AttnProblem& p, const void* vt, int64_t vt_ld, cudaStream_t s) {
    using C = FwdCfg<HD>;
    FwdMaps tm;
    const uint64_t W = (uint64_t)p.heads * HD;
    make_tmap_sw(&tm.q128, p.q, W, p.Nq, p.q_ld, 64, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&tm.q32, p.q, W, p.Nq, p.q_ld, 16, BM, CU_TENSOR_MAP_SWIZZLE_32B);
    make_tmap_sw(&tm.k128, p.k, W, p.Nk, p.k_ld, 64, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&tm.k32, p.k, W, p.Nk, p.k_ld, 16, BN, CU_TENSOR_MAP_SWIZZLE_32B);
    // V^T: rows = heads*HD (dims), cols = keys; box = 64 keys x HD dims
    make_tmap_sw(&tm.vt, vt, p.Nk, W, vt_ld, 64, HD, CU_TENSOR_MAP_SWIZZLE_128B);
    static bool set = false;
    if (!set) {
        MGV_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        set = true;
    }
    dim3 grid((p.Nq + BM - 1) / BM, p.heads);
    attn_fwd_tc_kernel<HD><<<grid, 256, C::SMEM, s>>>(tm, p); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

void attn_fwd_tc(const AttnProblem& p, cudaStream_t s) {
    const void* vt = p.vt;
    int64_t vt_ld = p.vt_ld;
    __nv_bfloat16* tmp = nullptr;
    if (!vt) {  // transpose V here (callers that keep V^T for the backward pass supply it)
        vt_ld = (p.Nk + 7) / 8 * 8;
        MGV_CUDA(cudaMallocAsync(&tmp, sizeof(__nv_bfloat16) * vt_ld * p.heads * p.hd, s));
        transpose_bf16(static_cast<const __nv_bfloat16*>(p.v), p.v_ld, p.Nk, p.heads * p.hd, tmp, vt_ld, s);
        vt = tmp;
    }
    switch (p.hd) {
        case 64: launch_fwd<64>(p, vt, vt_ld, s); break;
        case 128: launch_fwd<128>(p, vt, vt_ld, s); break;
        case 144: launch_fwd<144>(p, vt, vt_ld, s); break;
        default: throw std::runtime_error("attn_fwd_tc: unsupported head_dim");
    }
    if (tmp) MGV_CUDA(cudaFreeAsync(tmp, s));
}

}  // namespace mgv

extern "C" {
// Op-level entry for tests / roofline: bf16 operands, token-major with row strides; tc != 0 selects tcgen05.
int mgv_dev_attn_fwd(int tc, const void* q, int64_t q_ld, const void* k, int64_t k_ld, const void* v, int64_t v_ld,
                     void* o, int64_t o_ld, float* lse, int Nq, int Nk, int heads, int hd, void* stream) {
    try {
        mgv::AttnProblem p{q, q_ld, k, k_ld, v, v_ld, o, o_ld, lse, Nq, Nk, heads, hd};
        if (tc)
            mgv::attn_fwd_tc(p, static_cast<cudaStream_t>(stream));
        else
            mgv::attn_fwd_simt<__nv_bfloat16>(p, static_cast<cudaStream_t>(stream));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
int mgv_dev_attn_bwd(int tc, const void* q, int64_t q_ld, const void* k, int64_t k_ld, const void* v, int64_t v_ld,
                     const void* o, int64_t o_ld, const float* lse, const void* dO, int64_t do_ld, float* Dvec,
                     void* dq, int64_t dq_ld, void* dk, int64_t dk_ld, void* dv, int64_t dv_ld, float* dkv_part,
                     int q_splits, int Nq, int Nk, int heads, int hd, void* stream) {
    try {
        mgv::AttnBwdProblem p{mgv::AttnProblem{q, q_ld, k, k_ld, v, v_ld, const_cast<void*>(o), o_ld,
                                               const_cast<float*>(lse), Nq, Nk, heads, hd},
                              dO, do_ld, Dvec, dq, dq_ld, dk, dk_ld, dv, dv_ld, dkv_part, q_splits};
        if (tc)
            mgv::attn_bwd_tc(p, static_cast<cudaStream_t>(stream));
        else
            mgv::attn_bwd_simt<__nv_bfloat16>(p, static_cast<cudaStream_t>(stream));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
}
