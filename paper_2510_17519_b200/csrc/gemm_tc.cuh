// tcgen05 BF16 GEMM for sm_100a: C[M,N] = sum_k A[m,k] * B[n,k], fp32 accumulate
// in TMEM, fused epilogue functor (epilogue.cuh).
//
//   A, B each K-major ("row-major, K contiguous") or MN-major ("M/N contiguous"):
//     forward  X W^T : A K-major (activations), B K-major (weights)
//     dgrad    dY W  : A K-major, B MN-major (weights read as stored)
//     wgrad    dY^T X: A MN-major, B MN-major (activations read as stored)
//   so no transposed copies are ever made.
//
// Persistent, warp specialised, one CTA per SM:
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      MMA issuer (one elected lane), 128 x BN x 16 UMMAs
//   warp 2      TMEM allocator (2 x BN fp32 accumulator columns, double buffer)
//   warps 4..7  epilogue: tcgen05.ld -> registers -> functor -> global
// Tiles are 128 x BN x 64 with the 128-byte swizzle on both operands.
#pragma once
#include "epilogue.cuh"
#include "ptx.cuh"

namespace mgv {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
// Epilogue warps per CTA: 4 (one per TMEM lane group) for the light epilogues; the SiLU epilogues
// (two exponentials-worth of MUFU work and two outputs per element) use 8, two per lane group, each
// draining half of the columns.  Extra warps cost power in the power-capped GEMMs, so they are only
// spent where the epilogue would otherwise outlast the main loop.
template <class Epi>
struct EpiWarps {
    static constexpr int value = 4;
};
template <class T>
struct EpiWarps<EpiBiasSilu<T>> {
    static constexpr int value = 8;
};
template <class T>
struct EpiWarps<EpiSiluBwd<T>> {
    static constexpr int value = 8;
};
constexpr int kGemmThreadsMax = 128 + 32 * 8;
template <class Epi>
constexpr int gemm_threads() {
    return 128 + 32 * EpiWarps<Epi>::value;
}

// Grouped rasterisation: tiles are walked in groups of kRasterGroup M-tiles x all N-tiles, so the
// concurrently resident tiles share a few A slabs and a few B slabs (L2 reuse in both operands).
constexpr int kRasterGroup = 8;
__device__ __forceinline__ void raster(int t, int num_m, int num_n, int& mt, int& nt) {
    const int gsz = kRasterGroup * num_n;
    const int g = t / gsz, r = t % gsz;
    const int rows = min(kRasterGroup, num_m - g * kRasterGroup);
    mt = g * kRasterGroup + r % rows;
    nt = r / rows;
}

// Drain one accumulator: epilogue warp wq reads TMEM lane group (wq % 4) and column half (wq / 4) of
// the BN-column tile, 16 columns per tcgen05.ld, loading the next chunk while the current one is in
// the epilogue functor.
template <int BN, class Epi>
__device__ __forceinline__ void epilogue_rows(uint32_t acc_base, int wq, int lane, int m0, int n0, const Epi& epi) {
    constexpr int W = BN / (EpiWarps<Epi>::value / 4), NCH = W / 16;
    const int g = wq & 3, hf = wq >> 2;
    const int row = m0 + g * 32 + lane;
    const uint32_t base = acc_base + hf * W + (static_cast<uint32_t>(g * 32) << 16);
    if constexpr (IsTileEpi<Epi>::value) {  // whole-row functor (BN = one head): chunks on demand
        static_assert(EpiWarps<Epi>::value == 4, "tile epilogues own whole rows");
        epi.tile_row(
            row, n0, [&](int c, uint32_t* q) { tmem_ld16(base + c * 16, q); }, [] { tmem_wait_ld(); });
    } else {
        uint32_t r[2][16];
        tmem_ld16(base, r[0]);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            tmem_wait_ld();
            if (c + 1 < NCH) tmem_ld16(base + (c + 1) * 16, r[(c + 1) & 1]);
            epi(row, n0 + hf * W + c * 16, reinterpret_cast<const float*>(r[c & 1]), 16);
        }
    }
}

template <int BN>
struct GemmCfg {
    static constexpr int STAGES = BN >= 256 ? 4 : 6;
    static constexpr int A_BYTES = kGemmBM * kGemmBK * 2;  // 16 KB
    static constexpr int B_BYTES = BN * kGemmBK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                     : (2 * BN <= 256) ? 256 : 512;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// MC = 2: CTA pairs (a 2-CTA cluster) work on vertically adjacent tiles (m, m+1) of the same N block and
// share the B (weight) tile: each CTA TMA-loads half of it with .multicast::cluster into both CTAs'
// shared memory, and every MMA commit releases the stage in both CTAs.  L2->SM traffic per FLOP drops
// by a third (the kernel is otherwise L2-bandwidth-bound); the MMA / TMEM / epilogue path is unchanged.
template <int BN, bool A_MN, bool B_MN, int MC, class Epi>
__global__ void __launch_bounds__(kGemmThreadsMax, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                        int N, int K, Epi epi) {
    using C = GemmCfg<BN>;
    constexpr int BM = kGemmBM, BK = kGemmBK, STAGES = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * C::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
    const int num_mp = (num_m + MC - 1) / MC;  // M-tile groups (pairs when MC = 2)
    const int tiles = num_mp * num_n, kblocks = (K + BK - 1) / BK;
    const int rank = MC == 2 ? static_cast<int>(cluster_ctarank()) : 0;
    const int cid = blockIdx.x / MC, nclusters = gridDim.x / MC;
    constexpr uint16_t kPair = 0x3;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MC);  // released by the MMA of every CTA that reads the stage
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], EpiWarps<Epi>::value);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    if (MC == 2)
        cluster_sync();  // peer barriers initialised before any multicast lands
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // m fastest: consecutive CTAs share the B (weight) tile
    if (warp == 0) {
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < tiles; t += nclusters) {
                int mt_, nt_;
                raster(t, num_mp, num_n, mt_, nt_);
                const int m0 = (mt_ * MC + rank) * BM, n0 = nt_ * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = sA + stage * C::A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
                    const int k0 = kb * BK;
                    if (A_MN) {
#pragma unroll
                        for (int c = 0; c < BM / 64; ++c) tma_load_2d(a + c * 8192, &tmA, &full[stage], m0 + 64 * c, k0);
                    } else {
                        tma_load_2d(a, &tmA, &full[stage], k0, m0);
                    }
                    if (MC == 2) {  // this CTA's half of the shared B tile, multicast to both CTAs
                        if (B_MN) {
#pragma unroll
                            for (int c = rank * (BN / 128); c < (rank + 1) * (BN / 128); ++c)
                                tma_load_2d_mc(b + c * 8192, &tmB, &full[stage], n0 + 64 * c, k0, kPair);
                        } else {
                            tma_load_2d_mc(b + rank * (BN / 2) * 128, &tmB, &full[stage], k0, n0 + rank * (BN / 2), kPair);
                        }
                    } else if (B_MN) {
#pragma unroll
                        for (int c = 0; c < BN / 64; ++c) tma_load_2d(b + c * 8192, &tmB, &full[stage], n0 + 64 * c, k0);
                    } else {
                        tma_load_2d(b, &tmB, &full[stage], k0, n0);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t aphase = 0;
        for (int t = cid; t < tiles; t += nclusters) {
            mbar_wait(&tempty[acc], aphase ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + acc * BN;
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a = smem_u32(sA + stage * C::A_BYTES);
                    const uint32_t b = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // K-major: advance 16 elements = 32 bytes inside the 128B swizzle atom.
                        // MN-major: advance 16 K-rows = 2048 bytes (two 8-row groups).
                        const uint64_t ad = A_MN ? smem_desc(a + k * 2048, 8192, 1024, kSwizzle128)
                                                 : smem_desc(a + k * 32, 16, 1024, kSwizzle128);
                        const uint64_t bd = B_MN ? smem_desc(b + k * 2048, 8192, 1024, kSwizzle128)
                                                 : smem_desc(b + k * 32, 16, 1024, kSwizzle128);
                        umma_f16_ss(d, ad, bd, idesc, (kb | k) != 0);
                    }
                    if (MC == 2)
                        umma_commit_mc(&empty[stage], kPair);  // the stage holds data for both CTAs
                    else
                        umma_commit(&empty[stage]);
                    if (kb == kblocks - 1) umma_commit(&tfull[acc]);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++acc == 2) {
                acc = 0;
                aphase ^= 1;
            }
        }
    } else if (warp >= 4) {
        const int wq = warp - 4;  // epilogue warp index
        int acc = 0;
        uint32_t aphase = 0;
        for (int t = cid; t < tiles; t += nclusters) {
            int mt_, nt_;
                raster(t, num_mp, num_n, mt_, nt_);
                const int m0 = (mt_ * MC + rank) * BM, n0 = nt_ * BN;
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            epilogue_rows<BN>(tmem + acc * BN, wq, lane, m0, n0, epi);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                aphase ^= 1;
            }
        }
    }
    tc_fence_before();
    if (MC == 2)
        cluster_sync();  // no CTA leaves while its peer may still multicast into it
    else
        __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem);
}


// ------------------------------------------------------------------------------------------------
// CTA-pair GEMM (cta_group::2): a 2-CTA cluster computes a 256 x BN tile with M=256 UMMAs issued by
// the leader CTA.  Each CTA stages only its own 128 rows of A and its BN/2 rows of B (32 KB per stage
// for BN = 256, so 6 stages fit), both CTAs' TMA loads complete on the leader's barrier, the leader's
// commits release the stage / accumulator in both CTAs, and each CTA's epilogue drains the 128 TMEM
// lanes it owns, then arrives on the leader's accumulator-empty barrier.
template <int BN>
struct Gemm2Cfg {
    static constexpr int STAGES = BN >= 256 ? 6 : 8;
    static constexpr int A_BYTES = kGemmBM * kGemmBK * 2;        // this CTA's 128 rows
    static constexpr int B_BYTES = (BN / 2) * kGemmBK * 2;        // this CTA's BN/2 rows
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(kGemmThreadsMax, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                         int N, int K, Epi epi) {
    using C = Gemm2Cfg<BN>;
    constexpr int BM = kGemmBM, BK = kGemmBK, STAGES = C::STAGES, HB = BN / 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * C::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rank = static_cast<int>(cluster_ctarank());
    const bool leader = rank == 0;
    const int num_mp = (M + 2 * BM - 1) / (2 * BM), num_n = (N + BN - 1) / BN;
    const int tiles = num_mp * num_n, kblocks = (K + BK - 1) / BK;
    const int cid = blockIdx.x / 2, nclusters = gridDim.x / 2;
    constexpr uint16_t kPair = 0x3;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 2 * EpiWarps<Epi>::value);  // epilogue warps of both CTAs (leader's is used)
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            const uint32_t full_leader = mapa(smem_u32(full), 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < tiles; t += nclusters) {
                int mt_, nt_;
                raster(t, num_mp, num_n, mt_, nt_);
                const int m0 = mt_ * 2 * BM + rank * BM, n0 = nt_ * BN + rank * HB;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* a = sA + stage * C::A_BYTES;
                    uint8_t* b = sB + stage * C::B_BYTES;
                    const uint32_t fb = full_leader + stage * 8;
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
                    const int k0 = kb * BK;
                    if (A_MN) {
#pragma unroll
                        for (int c = 0; c < BM / 64; ++c) tma_load_2d_pair(a + c * 8192, &tmA, fb, m0 + 64 * c, k0);
                    } else {
                        tma_load_2d_pair(a, &tmA, fb, k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int c = 0; c < HB / 64; ++c) tma_load_2d_pair(b + c * 8192, &tmB, fb, n0 + 64 * c, k0);
                    } else {
                        tma_load_2d_pair(b, &tmB, fb, k0, n0);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            constexpr uint32_t idesc = idesc_bf16_f32(2 * BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int t = cid; t < tiles; t += nclusters) {
                mbar_wait(&tempty[acc], aphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t a = smem_u32(sA + stage * C::A_BYTES);
                        const uint32_t b = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            const uint64_t ad = A_MN ? smem_desc(a + k * 2048, 8192, 1024, kSwizzle128)
                                                     : smem_desc(a + k * 32, 16, 1024, kSwizzle128);
                            const uint64_t bd = B_MN ? smem_desc(b + k * 2048, 8192, 1024, kSwizzle128)
                                                     : smem_desc(b + k * 32, 16, 1024, kSwizzle128);
                            umma_f16_ss_pair(d, ad, bd, idesc, (kb | k) != 0);
                        }
                        umma_commit_pair_mc(&empty[stage], kPair);
                        if (kb == kblocks - 1) umma_commit_pair_mc(&tfull[acc], kPair);
                    }
                    __syncwarp();
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (++acc == 2) {
                    acc = 0;
                    aphase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        const int wq = warp - 4;  // epilogue warp index
        const uint32_t tempty_leader = mapa(smem_u32(tempty), 0);
        int acc = 0;
        uint32_t aphase = 0;
        for (int t = cid; t < tiles; t += nclusters) {
            int mt_, nt_;
            raster(t, num_mp, num_n, mt_, nt_);
            const int m0 = mt_ * 2 * BM + rank * BM, n0 = nt_ * BN;
            mbar_wait(&tfull[acc], aphase);
            tc_fence_after();
            epilogue_rows<BN>(tmem + acc * BN, wq, lane, m0, n0, epi);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
            if (++acc == 2) {
                acc = 0;
                aphase ^= 1;
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 2) tmem_dealloc_pair<C::TMEM_COLS>(tmem);
}

}  // namespace mgv
