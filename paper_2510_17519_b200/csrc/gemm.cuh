// Host-side GEMM dispatch: tcgen05 bf16 (performance mode) or IEEE-fp32 SIMT
// (parity mode: single-pass TF32/BF16 cannot meet 1e-4).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "epilogue.cuh"
#include "gemm_tc.cuh"

namespace mgv {

enum class Major { K = 0, MN = 1 };

// Element (i, k) of an operand: K-major -> p[i*ld + k]; MN-major -> p[k*ld + i].
struct Mat {
    const void* p;
    int64_t ld;
    Major major;
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define MGV_CUDA(x)                                                                                      \
    do {                                                                                                 \
        cudaError_t e_ = (x);                                                                            \
        if (e_ != cudaSuccess)                                                                           \
            throw ::mgv::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + ":" + \
                                   std::to_string(__LINE__));                                            \
    } while (0)

int num_sms();
void ensure_smem_attr(const void* kern, int bytes);  // per (kernel, device), thread-safe
template <class K>
inline void ensure_smem(K* kern, int bytes) {
    ensure_smem_attr(reinterpret_cast<const void*>(kern), bytes);
}
// kernel-launch accounting (bench: gpu_launches)
void note_launch();
int64_t launch_count();
void make_tmap_sw(CUtensorMap* m, const void* p, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_c,
                  uint32_t box_r, CUtensorMapSwizzle sw);
void make_tmap_bf16(CUtensorMap* m, const void* p, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                    uint32_t box_inner, uint32_t box_outer);

// ------------------------------------------------------------ fp32 SIMT path
template <bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(256) gemm_f32_simt_kernel(const float* __restrict__ A, int64_t lda,
                                                            const float* __restrict__ B, int64_t ldb, int M, int N,
                                                            int K, Epi epi) {
    __shared__ float sA[16][68];
    __shared__ float sB[16][68];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int k0 = 0; k0 < K; k0 += 16) {
        for (int i = threadIdx.x; i < 1024; i += 256) {
            int mm = A_MN ? i % 64 : i / 16, kk = A_MN ? i / 64 : i % 16;
            int m = m0 + mm, k = k0 + kk;
            sA[kk][mm] = (m < M && k < K) ? (A_MN ? A[(int64_t)k * lda + m] : A[(int64_t)m * lda + k]) : 0.0f;
            int nn = B_MN ? i % 64 : i / 16, kb = B_MN ? i / 64 : i % 16;
            int n = n0 + nn, k2 = k0 + kb;
            sB[kb][nn] = (n < N && k2 < K) ? (B_MN ? B[(int64_t)k2 * ldb + n] : B[(int64_t)n * ldb + k2]) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) epi(m0 + ty * 4 + i, n0 + tx * 4, acc[i], 4);
}

template <bool A_MN, bool B_MN, class Epi>
void gemm_f32_launch(const Mat& A, const Mat& B, int M, int N, int K, const Epi& epi, cudaStream_t s) {
    dim3 grid((N + 63) / 64, (M + 63) / 64);
    gemm_f32_simt_kernel<A_MN, B_MN, Epi><<<grid, 256, 0, s>>>(static_cast<const float*>(A.p), A.ld,
                                                               static_cast<const float*>(B.p), B.ld, M, N, K, epi); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------ tcgen05 path
template <int BN, bool A_MN, bool B_MN, class Epi>
void gemm_tc_launch(const Mat& A, const Mat& B, int M, int N, int K, const Epi& epi, cudaStream_t s) {
    using C = GemmCfg<BN>;
    const int num_m = (M + kGemmBM - 1) / kGemmBM, num_n = (N + BN - 1) / BN;
    const int MC = num_m >= 2 ? 2 : 1;  // B-tile multicast over CTA pairs
    CUtensorMap ta, tb;
    if (A_MN)
        make_tmap_bf16(&ta, A.p, M, K, A.ld, 64, kGemmBK);
    else
        make_tmap_bf16(&ta, A.p, K, M, A.ld, kGemmBK, kGemmBM);
    if (B_MN)
        make_tmap_bf16(&tb, B.p, N, K, B.ld, 64, kGemmBK);
    else
        make_tmap_bf16(&tb, B.p, K, N, B.ld, kGemmBK, BN / MC);
    if (MC == 1) {
        auto kern = gemm_bf16_tc_kernel<BN, A_MN, B_MN, 1, Epi>;
        ensure_smem(kern, C::SMEM);
        const int tiles = num_m * num_n;
        const int grid = tiles < num_sms() ? tiles : num_sms();
        kern<<<grid, gemm_threads<Epi>(), C::SMEM, s>>>(ta, tb, M, N, K, epi); ::mgv::note_launch();
    } else {
        auto kern = gemm_bf16_tc_kernel<BN, A_MN, B_MN, 2, Epi>;
        ensure_smem(kern, C::SMEM);
        const int pair_tiles = ((num_m + 1) / 2) * num_n;
        const int clusters = pair_tiles < num_sms() / 2 ? pair_tiles : num_sms() / 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * clusters);
        cfg.blockDim = dim3(gemm_threads<Epi>());
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MGV_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, epi));
        note_launch();
    }
    MGV_CUDA(cudaGetLastError());
}

template <int BN, bool A_MN, bool B_MN, class Epi>
void gemm_tc2_launch(const Mat& A, const Mat& B, int M, int N, int K, const Epi& epi, cudaStream_t s) {
    using C = Gemm2Cfg<BN>;
    CUtensorMap ta, tb;
    if (A_MN)
        make_tmap_bf16(&ta, A.p, M, K, A.ld, 64, kGemmBK);
    else
        make_tmap_bf16(&ta, A.p, K, M, A.ld, kGemmBK, kGemmBM);
    if (B_MN)
        make_tmap_bf16(&tb, B.p, N, K, B.ld, 64, kGemmBK);
    else
        make_tmap_bf16(&tb, B.p, K, N, B.ld, kGemmBK, BN / 2);
    auto kern = gemm_bf16_tc2_kernel<BN, A_MN, B_MN, Epi>;
    ensure_smem(kern, C::SMEM);
    const int tiles = ((M + 2 * kGemmBM - 1) / (2 * kGemmBM)) * ((N + BN - 1) / BN);
    const int clusters = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(gemm_threads<Epi>());
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MGV_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, M, N, K, epi));
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

extern int g_gemm_mode;  // 0: 1-CTA (+B multicast pairs), 1: CTA-pair UMMA (default)
// Benchmark-only phase timing of the tensor-core GEMMs: when set (Model, profiling on), called with
// begin = true and the GEMM's 2 M N K before the launch and with begin = false after it.
extern void (*g_gemm_prof_hook)(bool begin, double flops, cudaStream_t s);

struct GemmProfScope {
    cudaStream_t s;
    GemmProfScope(double f, cudaStream_t st) : s(st) {
        if (g_gemm_prof_hook) g_gemm_prof_hook(true, f, s);
    }
    ~GemmProfScope() {
        if (g_gemm_prof_hook) g_gemm_prof_hook(false, 0.0, s);
    }
};

// bf16 tcgen05 GEMM, both operands K-major, with an explicit N tile: the whole-tile epilogues need BN = one
// head (EpiQKNormRope: BN = head_dim).
template <int BN, class Epi>
void gemm_tc_bn(const Mat& A, const Mat& B, int M, int N, int K, const Epi& epi, cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    if (A.major != Major::K || B.major != Major::K) throw std::runtime_error("gemm_tc_bn: K-major operands only");
    GemmProfScope prof_scope(2.0 * M * N * K, s);
    if (g_gemm_mode == 1 && M > kGemmBM)
        gemm_tc2_launch<BN, false, false>(A, B, M, N, K, epi, s);
    else
        gemm_tc_launch<BN, false, false>(A, B, M, N, K, epi, s);
}

// Dispatch on precision and operand majors.  bf16: A/B are __nv_bfloat16; fp32: float.
template <class Epi>
void gemm(bool bf16, const Mat& A, const Mat& B, int M, int N, int K, const Epi& epi, cudaStream_t s) {
    if (M <= 0 || N <= 0) return;
    const bool am = A.major == Major::MN, bm = B.major == Major::MN;
    if (!bf16) {
        if (!am && !bm) gemm_f32_launch<false, false>(A, B, M, N, K, epi, s);
        else if (!am && bm) gemm_f32_launch<false, true>(A, B, M, N, K, epi, s);
        else if (am && bm) gemm_f32_launch<true, true>(A, B, M, N, K, epi, s);
        else gemm_f32_launch<true, false>(A, B, M, N, K, epi, s);
        return;
    }
    GemmProfScope prof_scope(2.0 * M * N * K, s);
    if (g_gemm_mode == 1 && M > kGemmBM) {
        if (!am && !bm) gemm_tc2_launch<256, false, false>(A, B, M, N, K, epi, s);
        else if (!am && bm) gemm_tc2_launch<256, false, true>(A, B, M, N, K, epi, s);
        else if (am && bm) gemm_tc2_launch<256, true, true>(A, B, M, N, K, epi, s);
        else throw std::runtime_error("gemm: MN-major A with K-major B is not used");
        return;
    }
    if (!am && !bm) gemm_tc_launch<256, false, false>(A, B, M, N, K, epi, s);
    else if (!am && bm) gemm_tc_launch<256, false, true>(A, B, M, N, K, epi, s);
    else if (am && bm) gemm_tc_launch<256, true, true>(A, B, M, N, K, epi, s);
    else throw std::runtime_error("gemm: MN-major A with K-major B is not used");
}

}  // namespace mgv
