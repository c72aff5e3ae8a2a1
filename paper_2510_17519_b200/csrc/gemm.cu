// GEMM host helpers (tensor maps, SM count) and the op-level GEMM entry points
// exported for tests / roofline measurement.
#include "gemm.cuh"

#include <atomic>
#include <map>
#include <mutex>

namespace mgv {

static std::atomic<int64_t> g_launches{0};
int g_gemm_mode = 1;
void (*g_gemm_prof_hook)(bool, double, cudaStream_t) = nullptr;
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

// SM count of the CURRENT device (a process may hold contexts on several GPUs)
int num_sms() {
    constexpr int kMaxDev = 64;
    static std::atomic<int> cache[kMaxDev] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) dev = 0;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n = v > 0 ? v : 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device context: remember, per (kernel, device), the
// largest size already set; thread-safe.
void ensure_smem_attr(const void* kern, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;
    int dev = 0;
    MGV_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    int& have = done[{kern, dev}];
    if (have >= bytes) return;
    MGV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

// 2-D bf16 tensor map, 128-byte swizzle: inner dim contiguous, outer dim strided by ld.
void make_tmap_bf16(CUtensorMap* m, const void* p, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                    uint32_t box_inner, uint32_t box_outer) {
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ") inner=" +
                        std::to_string(inner) + " outer=" + std::to_string(outer) + " ld=" + std::to_string(ld_elems));
}

// bf16 2-D map over a token-major matrix (rows x cols, row stride ld elements) with a chosen swizzle/box.
void make_tmap_sw(CUtensorMap* m, const void* p, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_c,
                  uint32_t box_r, CUtensorMapSwizzle sw) {
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {box_c, box_r};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("tensor map encode failed: " + std::to_string(int(r)));
}

}  // namespace mgv

using namespace mgv;

extern "C" {

// C[M,N] (fp32, ldc) (+)= alpha * sum_k A(m,k) B(n,k).  bf16 != 0: tcgen05 path on bf16
// operands; else IEEE fp32 SIMT path on fp32 operands.  Returns 0 or a CUDA error code.
// 0: 1-CTA tcgen05 GEMM (+ weight-tile multicast over CTA pairs), 1: CTA-pair (cta_group::2) GEMM
void mgv_dev_set_gemm_mode(int mode) { g_gemm_mode = mode; }

int mgv_dev_gemm(int bf16, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn, int M, int N,
                 int K, float* C, int64_t ldc, float alpha, int accumulate, void* stream) {
    try {
        EpiF32 e{C, ldc, nullptr, alpha, accumulate, M, N};
        gemm(bf16 != 0, Mat{A, lda, a_mn ? Major::MN : Major::K}, Mat{B, ldb, b_mn ? Major::MN : Major::K}, M, N,
             K, e, static_cast<cudaStream_t>(stream));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

}  // extern "C"
