// Memory-bound kernels of the DiT block: patchify, interpolation / masking,
// RoPE tables, modulation table, modulated RMSNorm, QK-norm + temperature +
// 3-D RoPE, post-norm residual, flow loss, and all their backward passes.
//
// Row kernels use one CTA per chunk of kRowsPerChunk rows with threads mapped
// to columns (thread j owns columns j, j+256, ...): loads are coalesced across
// the CTA, per-row statistics use a fixed-order block reduction, and
// per-column gradient partials stay in registers for the whole chunk, so every
// reduction is run-to-run bit-deterministic (no float atomics anywhere).
#include <cmath>

#include "gemm.cuh"
#include "kernels.h"

#include <type_traits>

namespace mgv {
// vectorised bf16 row kernels (defined at the end of this file)
bool use_vec(int H);
void rms_fwd_vec_launch(const float* X, int N, int H, const float* table, int64_t tld, int sh_off, int sc_off,
                        const int32_t* mod_id, const float* g, __nv_bfloat16* out, float* r, cudaStream_t s);
void postnorm_resid_vec_launch(const float* X1, const __nv_bfloat16* co, int N, int H, const float* g, float* X2,
                               float* rc, cudaStream_t s);
void postnorm_resid_mod_vec_launch(const float* X1, const __nv_bfloat16* co, int N, int H, const float* g, float* X2,
                                   float* rc, const float* table, int64_t tld, int sh_off, int sc_off,
                                   const int32_t* mod_id, __nv_bfloat16* f, float* r2, cudaStream_t s);
void gate_bwd_vec_launch(const float* dX, const __nv_bfloat16* y, const float* table, int64_t tld, int gate_off,
                         const int32_t* mod_id, int n_u, int N, int H, __nv_bfloat16* dY, float* part_dgate,
                         float* part_db, cudaStream_t s);
void rms_bwd_vec_launch(int mode, const __nv_bfloat16* dA, const float* X, const float* r, const float* table,
                        int64_t tld, int sc_off, const int32_t* mod_id, int n_u, const float* g, int N, int H, float* dX,
                        int accumulate, float* part_a, float* part_b, cudaStream_t s);
void postnorm_bwd_vec_launch(const float* dX, const __nv_bfloat16* co, const float* rc, const float* g, int N, int H,
                             __nv_bfloat16* dco, float* part_dg, cudaStream_t s);
void qk_norm_rope_vec_launch(const __nv_bfloat16* qkv, const QKLayout& L, int N, int hd, int heads,
                             const float* temp, const float2* cs, __nv_bfloat16* qk, float* iq, float* ik,
                             cudaStream_t s);
void qk_norm_rope_bwd_vec_launch(__nv_bfloat16* dqkv, const __nv_bfloat16* qkv, const QKLayout& L, int N, int hd,
                                 int heads, const float* temp, const float2* cs, const float* iq, const float* ik,
                                 float* part_dtemp, cudaStream_t s);
bool qk_vec_ok(const void* a, const void* b, const QKLayout& L, int hd);
void colsum_vec_launch(const __nv_bfloat16* Y, int64_t ld, int N, int C, float* part, cudaStream_t s);
template <class T>
constexpr bool is_bf16() { return std::is_same<T, __nv_bfloat16>::value; }
}  // namespace mgv

namespace mgv {

namespace {

constexpr int RT = 256;          // threads per row CTA
constexpr int MAXC = 16;         // columns per thread -> H <= 4096
constexpr double kEps = 1e-6;    // dit.cpp:13

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}
// Every thread returns the same value, summed in the same order.
__device__ __forceinline__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x / 32;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < RT / 32; ++i) s += red[i];
    __syncthreads();
    return s;
}
__device__ __forceinline__ double block_sum_d(double v, double* red) {
    v = warp_sum_d(v);
    const int w = threadIdx.x / 32;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < RT / 32; ++i) s += red[i];
    __syncthreads();
    return s;
}

inline int grid_for(int64_t n, int threads = 256) {
    int64_t g = (n + threads - 1) / threads;
    return static_cast<int>(g < (1 << 30) ? g : (1 << 30));
}

}  // namespace

// ============================================================ K1: sample prep
template <class T>
__global__ void prep_flow_sample_kernel(const double* clean, const double* noise, const uint8_t* cond,
                                        const double* cond_lat, int N, int D, double t, T* rows, float* vt,
                                        uint8_t* lmask, int32_t* mod_id, int id_t, int id_0) {
    const int64_t total = (int64_t)N * D;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(e / D);
        const bool c = cond && cond[i];  // apply_condition_mask (flowtrain.cpp:83-100), any unit-aligned mask
        const double x = clean[e], n = noise[e];
        // interpolate (flowtrain.cpp:16); conditioned rows <- condition_latents (flowtrain.cpp:95)
        const double xt = c ? (cond_lat ? cond_lat[e] : x) : (1.0 - t) * x + t * n;
        rows[e] = to_t<T>(static_cast<float>(xt));
        vt[e] = static_cast<float>(n - x);
        if (e % D == 0) {
            lmask[i] = c ? 0 : 1;
            mod_id[i] = c ? id_0 : id_t;  // modulation-table rows of tau = t and tau = 0 (flowtrain.cpp:96)
        }
    }
}
template <class T>
void prep_flow_sample(const double* clean, const double* noise, const uint8_t* cond, const double* cond_lat, int N,
                      int D, double t, T* rows, float* vt, uint8_t* lmask, int32_t* mod_id, cudaStream_t s, int id_t,
                      int id_0) {
    prep_flow_sample_kernel<T><<<grid_for((int64_t)N * D), 256, 0, s>>>(clean, noise, cond, cond_lat, N, D, t, rows,
                                                                        vt, lmask, mod_id, id_t, id_0);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

template <class T>
__global__ void convert_rows_kernel(const double* src, int64_t n, T* dst) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = to_t<T>(static_cast<float>(src[e]));
}
template <class T>
void convert_rows(const double* src, int64_t n, T* dst, cudaStream_t s) {
    convert_rows_kernel<T><<<grid_for(n), 256, 0, s>>>(src, n, dst); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
template <class T>
__global__ void convert_f32_kernel(const float* src, int64_t n, T* dst) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = to_t<T>(src[e]);
}
// 8 elements per thread (2 x 16-byte loads, one 16-byte bf16 store) when both pointers are 16-byte aligned
__global__ void convert_f32_bf16_vec8(const float4* src, int64_t n8, uint4* dst) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = src[2 * e], b = src[2 * e + 1];
        const __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w),
                             p2 = __floats2bfloat162_rn(b.x, b.y), p3 = __floats2bfloat162_rn(b.z, b.w);
        dst[e] = make_uint4(*reinterpret_cast<const uint32_t*>(&p0), *reinterpret_cast<const uint32_t*>(&p1),
                            *reinterpret_cast<const uint32_t*>(&p2), *reinterpret_cast<const uint32_t*>(&p3));
    }
}
template <class T>
void convert_f32(const float* src, int64_t n, T* dst, cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (n % 8 == 0 && (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16 == 0) {
            convert_f32_bf16_vec8<<<grid_for(n / 8), 256, 0, s>>>(reinterpret_cast<const float4*>(src), n / 8,
                                                                 reinterpret_cast<uint4*>(dst));
            ::mgv::note_launch();
            MGV_CUDA(cudaGetLastError());
            return;
        }
    }
    convert_f32_kernel<T><<<grid_for(n), 256, 0, s>>>(src, n, dst); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ patchify index math
__global__ void latent_rows_kernel(const double* grid, int U, int h, int w, int C, double* rows, int32_t* coords) {
    const int Hp = h / 2, Wp = w / 2, D = 4 * C;
    const int64_t N = (int64_t)U * Hp * Wp, total = N * D;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / D;
        const int j = static_cast<int>(e % D);
        const int c = j % C, q = j / C, dy = q / 2, dx = q % 2;
        const int64_t t = i / ((int64_t)Hp * Wp);
        const int py = static_cast<int>((i / Wp) % Hp), px = static_cast<int>(i % Wp);
        rows[e] = grid[((t * h + 2 * py + dy) * w + 2 * px + dx) * C + c];  // dit.cpp:108-109
        if (j == 0) {
            coords[3 * i] = static_cast<int32_t>(t);
            coords[3 * i + 1] = py;
            coords[3 * i + 2] = px;
        }
    }
}
void latent_rows_gather(const double* grid, int U, int h, int w, int C, double* rows, int32_t* coords, cudaStream_t s) {
    const int64_t total = (int64_t)U * (h / 2) * (w / 2) * 4 * C;
    latent_rows_kernel<<<grid_for(total), 256, 0, s>>>(grid, U, h, w, C, rows, coords); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

__global__ void rows_to_grid_check_kernel(const int32_t* coords, int N, int U, int Hp, int Wp, int32_t* seen,
                                          int32_t* status) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const int t = coords[3 * i], py = coords[3 * i + 1], px = coords[3 * i + 2];
        if (t < 0 || t >= U || py < 0 || py >= Hp || px < 0 || px >= Wp) {
            atomicMax(status, 1);
            continue;
        }
        const int64_t slot = ((int64_t)t * Hp + py) * Wp + px;
        if (atomicAdd(&seen[slot], 1) != 0) atomicMax(status, 2);
    }
}
__global__ void rows_to_grid_kernel(const double* rows, const int32_t* coords, int N, int U, int Hp, int Wp, int C,
                                    double* grid, const int32_t* status) {
    if (*status != 0) return;
    const int D = 4 * C;
    const int64_t total = (int64_t)N * D;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / D;
        const int j = static_cast<int>(e % D);
        const int c = j % C, q = j / C, dy = q / 2, dx = q % 2;
        const int64_t t = coords[3 * i], py = coords[3 * i + 1], px = coords[3 * i + 2];
        grid[((t * 2 * Hp + 2 * py + dy) * 2 * Wp + 2 * px + dx) * C + c] = rows[e];  // dit.cpp:137-138
    }
}
void rows_to_grid_scatter(const double* rows, const int32_t* coords, int N, int U, int Hp, int Wp, int C, double* grid,
                          int32_t* seen, int32_t* status, cudaStream_t s) {
    MGV_CUDA(cudaMemsetAsync(seen, 0, sizeof(int32_t) * (size_t)U * Hp * Wp, s));
    MGV_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t), s));
    rows_to_grid_check_kernel<<<grid_for(N), 256, 0, s>>>(coords, N, U, Hp, Wp, seen, status); ::mgv::note_launch();
    rows_to_grid_kernel<<<grid_for((int64_t)N * 4 * C), 256, 0, s>>>(rows, coords, N, U, Hp, Wp, C, grid, status); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ RoPE table
// pair p of a head vector: axis a with offset o_a (in pairs) -> theta = pos_a * 10000^(-2i/d_a)  (autodiff.cpp:856-866)
__global__ void rope_table_kernel(const int32_t* coords, int N, int s0, int s1, int s2, float2* cs) {
    const int P = (s0 + s1 + s2) / 2;
    const int64_t total = (int64_t)N * P;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t n = e / P;
        int p = static_cast<int>(e % P);
        int axis = 0, d = s0;
        if (p >= s0 / 2) {
            p -= s0 / 2;
            axis = 1;
            d = s1;
            if (p >= s1 / 2) {
                p -= s1 / 2;
                axis = 2;
                d = s2;
            }
        }
        const double freq = pow(10000.0, -2.0 * static_cast<double>(p) / static_cast<double>(d));
        const double th = static_cast<double>(coords[3 * n + axis]) * freq;
        double sn, c;
        sincos(th, &sn, &c);
        cs[e] = make_float2(static_cast<float>(c), static_cast<float>(sn));
    }
}
void rope_table(const int32_t* coords, int N, int s0, int s1, int s2, float2* cs, cudaStream_t s) {
    rope_table_kernel<<<grid_for((int64_t)N * (s0 + s1 + s2) / 2), 256, 0, s>>>(coords, N, s0, s1, s2, cs); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ global embedding (fp64)
// phi rows: 0..n_u-1 = sinusoid(1000 tau_u), n_u = sinusoid(fps)   (dit.cpp:27-34, 242-244)
__global__ void sinusoid_kernel(const double* taus, int n_u, double fps, double* phi) {
    const int r = blockIdx.x, i = threadIdx.x;  // 16 threads
    if (i >= 16) return;
    const double s = r < n_u ? 1000.0 * taus[r] : fps;
    const double freq = exp(-(log(10000.0) * static_cast<double>(i)) / 16.0);
    phi[r * 32 + i] = cos(s * freq);
    phi[r * 32 + 16 + i] = sin(s * freq);
}
// out[r, j] = act(sum_k in[r, k] W[j, k] + b[j]) ; one warp per (r, j), fp64 accumulate
template <int ACT>  // 0 none, 1 silu (stores pre-act to z)
__global__ void gemv_rows_f64(const double* in, int rows, int K, const float* W, const float* b, int J, double* z,
                              double* out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
    if (warp >= rows * J) return;
    const int r = warp / J, j = warp % J;
    double acc = 0.0;
    for (int k = lane; k < K; k += 32) acc += in[(int64_t)r * K + k] * static_cast<double>(W[(int64_t)j * K + k]);
    acc = warp_sum_d(acc);
    if (lane == 0) {
        acc += b ? static_cast<double>(b[j]) : 0.0;
        if (ACT == 1) {
            z[(int64_t)r * J + j] = acc;
            out[(int64_t)r * J + j] = acc / (1.0 + exp(-acc));
        } else {
            out[(int64_t)r * J + j] = acc;
        }
    }
}
__global__ void add_fps_row(double* g, int n_u, int H) {  // g_u += g_fps (row n_u)
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_u * H; e += gridDim.x * blockDim.x)
        g[e] += g[(int64_t)n_u * H + e % H];
}
void global_embed(const double* taus, int n_u, double fps, const float* w_in, const float* b_in, const float* w_out,
                  const float* b_out, int H, double* phi, double* z_in, double* h_in, double* g, cudaStream_t s) {
    const int R = n_u + 1;
    sinusoid_kernel<<<R, 32, 0, s>>>(taus, n_u, fps, phi); ::mgv::note_launch();
    gemv_rows_f64<1><<<grid_for((int64_t)R * H * 32), 256, 0, s>>>(phi, R, 32, w_in, b_in, H, z_in, h_in); ::mgv::note_launch();
    gemv_rows_f64<0><<<grid_for((int64_t)R * H * 32), 256, 0, s>>>(h_in, R, H, w_out, b_out, H, nullptr, g); ::mgv::note_launch();
    add_fps_row<<<grid_for((int64_t)n_u * H), 256, 0, s>>>(g, n_u, H); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
__global__ void mul_gscale(const double* g, const float* gs, int n_u, int H, double* gb) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_u * H; e += gridDim.x * blockDim.x)
        gb[e] = g[e] * static_cast<double>(gs[e % H]);
}
__global__ void gemv_rows_f64_to_f32(const double* in, int rows, int K, const float* W, const float* b, int J,
                                     float* out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
    if (warp >= rows * J) return;
    const int r = warp / J, j = warp % J;
    double acc = 0.0;
    for (int k = lane; k < K; k += 32) acc += in[(int64_t)r * K + k] * static_cast<double>(W[(int64_t)j * K + k]);
    acc = warp_sum_d(acc);
    if (lane == 0) out[(int64_t)r * J + j] = static_cast<float>(acc + static_cast<double>(b[j]));
}
void modulation_table(const double* g, const float* gscale, const float* w_mod, const float* b_mod, int n_u, int H,
                      double* gb, float* table, cudaStream_t s) {
    mul_gscale<<<grid_for((int64_t)n_u * H), 256, 0, s>>>(g, gscale, n_u, H, gb); ::mgv::note_launch();
    gemv_rows_f64_to_f32<<<grid_for((int64_t)n_u * 6 * H * 32), 256, 0, s>>>(gb, n_u, H, w_mod, b_mod, 6 * H, table); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ forward row kernels
template <class T>
__global__ void __launch_bounds__(RT) rms_mod_kernel(const float* X, int N, int H, const float* table, int64_t tld,
                                                     int sh_off, int sc_off, const int32_t* mod_id, int use_gain,
                                                     const float* g, T* out, float* r) {
    __shared__ float red[RT / 32];
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    for (int i = r0; i < r1; ++i) {
        const float* x = X + (int64_t)i * H;
        float v[MAXC];
        float ss = 0.0f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            v[c] = j < H ? x[j] : 0.0f;
            ss = fmaf(v[c], v[c], ss);
        }
        ss = block_sum(ss, red);
        const float rr = 1.0f / sqrtf(ss / static_cast<float>(H) + static_cast<float>(kEps));
        if (threadIdx.x == 0) r[i] = rr;
        const float* tb = use_gain ? nullptr : table + (int64_t)mod_id[i] * tld;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            if (j < H) {
                const float n = v[c] * rr;
                const float o = use_gain ? n * g[j] : n * (1.0f + tb[sc_off + j]) + tb[sh_off + j];
                out[(int64_t)i * H + j] = to_t<T>(o);
            }
        }
    }
}
template <class T>
void rms_mod(const float* X, int N, int H, const float* table, int64_t tld, int sh_off, int sc_off,
             const int32_t* mod_id, T* out, float* r, cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H)) return rms_fwd_vec_launch(X, N, H, table, tld, sh_off, sc_off, mod_id, nullptr, out, r, s);
    }
    rms_mod_kernel<T><<<row_chunks(N), RT, 0, s>>>(X, N, H, table, tld, sh_off, sc_off, mod_id, 0, nullptr, out, r); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
template <class T>
void rms_gain(const float* X, int N, int H, const float* g, T* out, float* r, cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H)) return rms_fwd_vec_launch(X, N, H, nullptr, 0, 0, 0, nullptr, g, out, r, s);
    }
    rms_mod_kernel<T><<<row_chunks(N), RT, 0, s>>>(X, N, H, nullptr, 0, 0, 0, nullptr, 1, g, out, r); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

template <class T>
__global__ void __launch_bounds__(RT) postnorm_resid_kernel(const float* X1, const T* co, int N, int H, const float* g,
                                                            float* X2, float* rc) {
    __shared__ float red[RT / 32];
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    for (int i = r0; i < r1; ++i) {
        float v[MAXC];
        float ss = 0.0f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            v[c] = j < H ? to_f(co[(int64_t)i * H + j]) : 0.0f;
            ss = fmaf(v[c], v[c], ss);
        }
        ss = block_sum(ss, red);
        const float rr = 1.0f / sqrtf(ss / static_cast<float>(H) + static_cast<float>(kEps));
        if (threadIdx.x == 0) rc[i] = rr;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            if (j < H) X2[(int64_t)i * H + j] = X1[(int64_t)i * H + j] + v[c] * rr * g[j];
        }
    }
}
template <class T>
void postnorm_resid(const float* X1, const T* co, int N, int H, const float* g, float* X2, float* rc, cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H)) return postnorm_resid_vec_launch(X1, co, N, H, g, X2, rc, s);
    }
    postnorm_resid_kernel<T><<<row_chunks(N), RT, 0, s>>>(X1, co, N, H, g, X2, rc); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

template <class T>
bool postnorm_resid_mod(const float* X1, const T* co, int N, int H, const float* g, float* X2, float* rc,
                        const float* table, int64_t tld, int sh_off, int sc_off, const int32_t* mod_id, T* f, float* r2,
                        cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H)) {
            postnorm_resid_mod_vec_launch(X1, co, N, H, g, X2, rc, table, tld, sh_off, sc_off, mod_id, f, r2, s);
            return true;
        }
    }
    return false;
}

// One warp per (token, head, q|k); lane owns rotation pairs lane, lane+32, lane+64 (hd <= 192).
template <class T>
__global__ void __launch_bounds__(256) qk_norm_rope_kernel(const T* qkv, QKLayout Lq, int N, int H, int heads,
                                                           const float* temp, const float2* cs, T* qk, float* iq,
                                                           float* ik) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    const int hd = H / heads, P = hd / 2;
    if (gw >= (int64_t)N * heads * 2) return;
    const int which = static_cast<int>(gw % 2);  // 0 q, 1 k
    const int h = static_cast<int>((gw / 2) % heads);
    const int64_t n = gw / (2 * heads);
    const T* src = qkv + n * Lq.in_ld + which * Lq.in_koff + h * hd;
    float a[3], b[3];
    float ss = 0.0f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int p = lane + 32 * c;
        a[c] = p < P ? to_f(src[2 * p]) : 0.0f;
        b[c] = p < P ? to_f(src[2 * p + 1]) : 0.0f;
        ss = fmaf(a[c], a[c], fmaf(b[c], b[c], ss));
    }
    ss = warp_sum(ss);
    const float iv = 1.0f / sqrtf(ss + static_cast<float>(kEps));  // autodiff.cpp:727
    if (lane == 0) (which == 0 ? iq : ik)[n * Lq.i_ld + h] = iv;
    const float sc = which == 0 ? iv * temp[h] : iv;  // mul_head_scalar on q (dit.cpp:292)
    T* dst = qk + n * Lq.out_ld + which * Lq.out_koff + h * hd;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int p = lane + 32 * c;
        if (p < P) {
            const float2 r = cs[n * P + p];
            const float x0 = a[c] * sc, x1 = b[c] * sc;
            dst[2 * p] = to_t<T>(x0 * r.x - x1 * r.y);  // autodiff.cpp:864-865
            dst[2 * p + 1] = to_t<T>(x0 * r.y + x1 * r.x);
        }
    }
}
template <class T>
void qk_norm_rope(const T* qkv, const QKLayout& L, int N, int H, int heads, const float* temp, const float2* cs, T* qk,
                  float* iq, float* ik, cudaStream_t s) {
    if constexpr (is_bf16<T>())
        if (qk_vec_ok(qkv, qk, L, H / heads))
            return qk_norm_rope_vec_launch(qkv, L, N, H / heads, heads, temp, cs, qk, iq, ik, s);
    const int64_t warps = (int64_t)N * heads * 2;
    qk_norm_rope_kernel<T><<<grid_for(warps * 32), 256, 0, s>>>(qkv, L, N, H, heads, temp, cs, qk, iq, ik); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ flow loss
template <class T>
__global__ void __launch_bounds__(RT) flow_loss_fwd_kernel(const float* V, const float* vt, const uint8_t* mask, int N,
                                                           int D, double* part) {
    __shared__ double red[RT / 32];
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    double acc = 0.0;
    for (int i = r0; i < r1; ++i) {
        if (!mask[i]) continue;
        for (int j = threadIdx.x; j < D; j += RT) {
            const double d = static_cast<double>(V[(int64_t)i * D + j]) - static_cast<double>(vt[(int64_t)i * D + j]);
            acc += d * d;
        }
    }
    acc = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
template <class T>
void flow_loss_fwd(const float* V, const float* vt, const uint8_t* mask, int N, int D, double* part, cudaStream_t s) {
    flow_loss_fwd_kernel<T><<<row_chunks(N), RT, 0, s>>>(V, vt, mask, N, D, part); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
template <class T>
__global__ void flow_loss_bwd_kernel(const float* V, const float* vt, const uint8_t* mask, int N, int D, float base,
                                     const int* count, T* dV) {
    const int64_t total = (int64_t)N * D;
    const int cnt = *count;
    const float coef = cnt > 0 ? static_cast<float>(static_cast<double>(base) / (static_cast<double>(cnt) * D)) : 0.0f;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(e / D);
        dV[e] = to_t<T>(mask[i] ? coef * (V[e] - vt[e]) : 0.0f);
    }
}
template <class T>
void flow_loss_bwd(const float* V, const float* vt, const uint8_t* mask, int N, int D, float base, const int* count,
                   T* dV, cudaStream_t s) {
    flow_loss_bwd_kernel<T><<<grid_for((int64_t)N * D), 256, 0, s>>>(V, vt, mask, N, D, base, count, dV); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
__global__ void count_mask_kernel(const uint8_t* mask, int N, int* count) {
    __shared__ float red[RT / 32];
    float c = 0.0f;  // exact for N < 2^24 per thread partial
    int acc = 0;
    for (int i = threadIdx.x; i < N; i += RT) acc += mask[i] ? 1 : 0;
    c = block_sum(static_cast<float>(acc), red);
    if (threadIdx.x == 0) *count = static_cast<int>(c);
}
void count_mask(const uint8_t* mask, int N, int* count, cudaStream_t s) {
    count_mask_kernel<<<1, RT, 0, s>>>(mask, N, count); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
__global__ void sum_double_kernel(const double* part, int n, double* out) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
}
__global__ void flow_loss_acc_kernel(const double* part, int n, const int* count, int D, double* acc) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    const int c = *count;
    if (c > 0) acc[0] += s / (static_cast<double>(c) * D);
}
void flow_loss_accumulate(const double* part, int n, const int* count, int D, double* acc, cudaStream_t s) {
    flow_loss_acc_kernel<<<1, 1, 0, s>>>(part, n, count, D, acc); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
void sum_double(const double* part, int n, double* out, cudaStream_t s) {
    sum_double_kernel<<<1, 1, 0, s>>>(part, n, out); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ backward row kernels
constexpr int MAXU = 2;  // distinct modulation rows per 64-row chunk (tau = t and tau = 0)

// The (at most two) modulation-table rows of chunk [r0, r1): ua = the first row's, ub = the other one (= ua when
// the chunk has one).  An unpacked sample uses rows {0, 1}; a varlen-packed batch (Model::flow_step_packed) uses
// {k, B} inside sample k's 256-row-aligned segment (its padding rows take k), so no 64-row chunk sees a third.
__device__ __forceinline__ void chunk_rows(const int32_t* mod_id, int r0, int r1, int& ua, int& ub) {
    ua = mod_id[r0];
    ub = ua;
    for (int i = r0 + 1; i < r1; ++i) {
        const int u = mod_id[i];
        if (u != ua) ub = u;
    }
}

template <class T>
__global__ void __launch_bounds__(RT) gate_bwd_kernel(const float* dX, const T* y, const float* table, int64_t tld,
                                                      int gate_off, const int32_t* mod_id, int n_u, int N, int H,
                                                      T* dY, float* part_dgate, float* part_db) {
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float pg[MAXU][MAXC], pb[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        pb[c] = 0.0f;
#pragma unroll
        for (int u = 0; u < MAXU; ++u) pg[u][c] = 0.0f;
    }
    int ua, ub;
    chunk_rows(mod_id, r0, r1, ua, ub);
    for (int i = r0; i < r1; ++i) {
        const int u = mod_id[i];
        const float* gt = table + (int64_t)u * tld + gate_off;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            if (j < H) {
                const int64_t e = (int64_t)i * H + j;
                const float dx = dX[e];
                const float d = dx * gt[j];
                dY[e] = to_t<T>(d);
                pb[c] += d;
                const float gg = dx * to_f(y[e]);
                if (u == ua)
                    pg[0][c] += gg;
                else
                    pg[1][c] += gg;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const int j = threadIdx.x + c * RT;
        if (j < H) {
            part_db[(int64_t)blockIdx.x * H + j] = pb[c];
            for (int u = 0; u < n_u; ++u)
                part_dgate[((int64_t)blockIdx.x * n_u + u) * H + j] =
                    u == ua ? pg[0][c] : (u == ub ? pg[1][c] : 0.0f);
        }
    }
}
template <class T>
void gate_bwd(const float* dX, const T* y, const float* table, int64_t tld, int gate_off, const int32_t* mod_id,
              int n_u, int N, int H, T* dY, float* part_dgate, float* part_db, cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H))
            return gate_bwd_vec_launch(dX, y, table, tld, gate_off, mod_id, n_u, N, H, dY, part_dgate, part_db, s);
    }
    gate_bwd_kernel<T><<<row_chunks(N), RT, 0, s>>>(dX, y, table, tld, gate_off, mod_id, n_u, N, H, dY, part_dgate,
                                                   part_db); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// rms backward (autodiff.cpp:702-716): dx = dn*r - x * (sum(dn*x) * r^3 / D)
template <class T, int MODE>  // MODE 0: modulated (dn = dA (1+sc)), 1: gain (dn = dA g)
__global__ void __launch_bounds__(RT) rms_bwd_kernel(const T* dA, const float* X, const float* r, const float* table,
                                                     int64_t tld, int sh_off, int sc_off, const int32_t* mod_id,
                                                     int n_u, const float* g, int N, int H, float* dX, int accumulate,
                                                     float* part_a, float* part_b) {
    __shared__ float red[RT / 32];
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float pa[MAXU][MAXC], pbv[MAXU][MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
#pragma unroll
        for (int u = 0; u < MAXU; ++u) pa[u][c] = pbv[u][c] = 0.0f;
    int ua = 0, ub = 0;
    if (MODE == 0) chunk_rows(mod_id, r0, r1, ua, ub);
    for (int i = r0; i < r1; ++i) {
        const int u = MODE == 0 ? mod_id[i] : 0;
        const int slot = u == ua ? 0 : 1;
        const float* tb = MODE == 0 ? table + (int64_t)u * tld : nullptr;
        const float rr = r[i];
        float xv[MAXC], dn[MAXC];
        float dot = 0.0f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            xv[c] = 0.0f;
            dn[c] = 0.0f;
            if (j < H) {
                const int64_t e = (int64_t)i * H + j;
                const float da = to_f(dA[e]);
                xv[c] = X[e];
                const float n = xv[c] * rr;
                if (MODE == 0) {
                    dn[c] = da * (1.0f + tb[sc_off + j]);
#pragma unroll
                    for (int uu = 0; uu < MAXU; ++uu)
                        if (uu == slot) {
                            pa[uu][c] += da;       // d shift
                            pbv[uu][c] += da * n;  // d scale
                        }
                } else {
                    dn[c] = da * g[j];
                    pa[0][c] += da * n;  // d gain
                }
                dot = fmaf(dn[c], xv[c], dot);
            }
        }
        dot = block_sum(dot, red);
        const float k = dot * rr * rr * rr / static_cast<float>(H);
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            if (j < H) {
                const int64_t e = (int64_t)i * H + j;
                const float d = dn[c] * rr - xv[c] * k;
                dX[e] = accumulate ? dX[e] + d : d;
            }
        }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const int j = threadIdx.x + c * RT;
        if (j < H) {
            if (MODE == 0) {
                for (int u = 0; u < n_u; ++u) {
                    part_a[((int64_t)blockIdx.x * n_u + u) * H + j] = u == ua ? pa[0][c] : (u == ub ? pa[1][c] : 0.0f);
                    part_b[((int64_t)blockIdx.x * n_u + u) * H + j] = u == ua ? pbv[0][c] : (u == ub ? pbv[1][c] : 0.0f);
                }
            } else {
                part_a[(int64_t)blockIdx.x * H + j] = pa[0][c];
            }
        }
    }
}
template <class T>
void rms_mod_bwd(const T* dA, const float* X, const float* r, const float* table, int64_t tld, int sh_off, int sc_off,
                 const int32_t* mod_id, int n_u, int N, int H, float* dX, float* part_dsh, float* part_dsc,
                 cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H))
            return rms_bwd_vec_launch(0, dA, X, r, table, tld, sc_off, mod_id, n_u, nullptr, N, H, dX, 1, part_dsh,
                                      part_dsc, s);
    }
    rms_bwd_kernel<T, 0><<<row_chunks(N), RT, 0, s>>>(dA, X, r, table, tld, sh_off, sc_off, mod_id, n_u, nullptr, N, H,
                                                     dX, 1, part_dsh, part_dsc); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
template <class T>
void rms_gain_bwd(const T* dA, const float* X, const float* r, const float* g, int N, int H, float* dX, int accumulate,
                  float* part_dg, cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H))
            return rms_bwd_vec_launch(1, dA, X, r, nullptr, 0, 0, nullptr, 1, g, N, H, dX, accumulate, part_dg, nullptr, s);
    }
    rms_bwd_kernel<T, 1><<<row_chunks(N), RT, 0, s>>>(dA, X, r, nullptr, 0, 0, 0, nullptr, 1, g, N, H, dX, accumulate,
                                                     part_dg, nullptr); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// post-norm backward: X2 = X1 + n(co) g -> dg += dX n ; dco = rms_bwd(co, rc, dX g)
template <class T>
__global__ void __launch_bounds__(RT) postnorm_bwd_kernel(const float* dX, const T* co, const float* rc,
                                                          const float* g, int N, int H, T* dco, float* part_dg) {
    __shared__ float red[RT / 32];
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float pg[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) pg[c] = 0.0f;
    for (int i = r0; i < r1; ++i) {
        const float rr = rc[i];
        float xv[MAXC], dn[MAXC];
        float dot = 0.0f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            xv[c] = dn[c] = 0.0f;
            if (j < H) {
                const int64_t e = (int64_t)i * H + j;
                xv[c] = to_f(co[e]);
                const float dx = dX[e];
                pg[c] += dx * xv[c] * rr;
                dn[c] = dx * g[j];
                dot = fmaf(dn[c], xv[c], dot);
            }
        }
        dot = block_sum(dot, red);
        const float k = dot * rr * rr * rr / static_cast<float>(H);
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int j = threadIdx.x + c * RT;
            if (j < H) dco[(int64_t)i * H + j] = to_t<T>(dn[c] * rr - xv[c] * k);
        }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
        const int j = threadIdx.x + c * RT;
        if (j < H) part_dg[(int64_t)blockIdx.x * H + j] = pg[c];
    }
}
template <class T>
void postnorm_bwd(const float* dX, const T* co, const float* rc, const float* g, int N, int H, T* dco, float* part_dg,
                  cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (use_vec(H)) return postnorm_bwd_vec_launch(dX, co, rc, g, N, H, dco, part_dg, s);
    }
    postnorm_bwd_kernel<T><<<row_chunks(N), RT, 0, s>>>(dX, co, rc, g, N, H, dco, part_dg); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// QK-norm + temperature + RoPE backward.  CTA = chunk of rows; warp w owns heads w, w+8, ... (deterministic dtemp).
template <class T>
__global__ void __launch_bounds__(256) qk_norm_rope_bwd_kernel(T* dqkv, const T* qkv, QKLayout Lq, int N, int H,
                                                               int heads, const float* temp, const float2* cs,
                                                               const float* iq, const float* ik, float* part_dtemp) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int hd = H / heads, P = hd / 2;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    for (int h = warp; h < heads; h += 8) {
        float dtemp = 0.0f;
        for (int n = r0; n < r1; ++n) {
#pragma unroll 1
            for (int which = 0; which < 2; ++which) {
                const T* x = qkv + (int64_t)n * Lq.in_ld + which * Lq.in_koff + h * hd;
                T* dx = dqkv + (int64_t)n * Lq.in_ld + which * Lq.in_koff + h * hd;
                const float iv = (which == 0 ? iq : ik)[(int64_t)n * Lq.i_ld + h];
                float xa[3], xb[3], ga[3], gb[3];
                float dot = 0.0f, tdot = 0.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int p = lane + 32 * c;
                    xa[c] = xb[c] = ga[c] = gb[c] = 0.0f;
                    if (p < P) {
                        const float2 r = cs[(int64_t)n * P + p];
                        const float d0 = to_f(dx[2 * p]), d1 = to_f(dx[2 * p + 1]);
                        // inverse rotation (autodiff.cpp:888-898)
                        ga[c] = d0 * r.x + d1 * r.y;
                        gb[c] = -d0 * r.y + d1 * r.x;
                        xa[c] = to_f(x[2 * p]);
                        xb[c] = to_f(x[2 * p + 1]);
                        if (which == 0) tdot += (ga[c] * xa[c] + gb[c] * xb[c]) * iv;  // d temp = sum dqt * qn
                    }
                }
                const float sc = which == 0 ? temp[h] : 1.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    ga[c] *= sc;
                    gb[c] *= sc;
                    dot += ga[c] * xa[c] + gb[c] * xb[c];
                }
                dot = warp_sum(dot);
                if (which == 0) dtemp += warp_sum(tdot);
                const float k = dot * iv * iv * iv;  // autodiff.cpp:746-748
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int p = lane + 32 * c;
                    if (p < P) {
                        dx[2 * p] = to_t<T>(ga[c] * iv - xa[c] * k);
                        dx[2 * p + 1] = to_t<T>(gb[c] * iv - xb[c] * k);
                    }
                }
            }
        }
        if (lane == 0) part_dtemp[(int64_t)blockIdx.x * heads + h] = dtemp;
    }
}
template <class T>
void qk_norm_rope_bwd(T* dqkv, const T* qkv, const QKLayout& L, int N, int H, int heads, const float* temp,
                      const float2* cs, const float* iq, const float* ik, float* part_dtemp, cudaStream_t s) {
    if constexpr (is_bf16<T>())
        if (qk_vec_ok(dqkv, qkv, L, H / heads))
            return qk_norm_rope_bwd_vec_launch(dqkv, qkv, L, N, H / heads, heads, temp, cs, iq, ik, part_dtemp, s);
    qk_norm_rope_bwd_kernel<T><<<row_chunks(N), 256, 0, s>>>(dqkv, qkv, L, N, H, heads, temp, cs, iq, ik, part_dtemp); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// column sums: CTA (chunk, column block of 256) ; thread = column
template <class T>
__global__ void colsum_kernel(const T* Y, int64_t ld, int N, int C, float* part) {
    const int j = blockIdx.y * blockDim.x + threadIdx.x;
    if (j >= C) return;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float acc = 0.0f;
    for (int i = r0; i < r1; ++i) acc += to_f(Y[(int64_t)i * ld + j]);
    part[(int64_t)blockIdx.x * C + j] = acc;
}
template <class T>
void colsum(const T* Y, int64_t ld, int N, int C, float* part, cudaStream_t s) {
    if constexpr (is_bf16<T>()) {
        if (C % 8 == 0 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0)
            return colsum_vec_launch(Y, ld, N, C, part, s);
    }
    dim3 grid(row_chunks(N), (C + 255) / 256);
    colsum_kernel<T><<<grid, 256, 0, s>>>(Y, ld, N, C, part); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
// Block = 32 consecutive (group, column) entries x kRcWarps warps.  Warp r sums chunks r, r + kRcWarps, ... and
// the partial sums are then added in warp order: a fixed reduction tree, so the result is deterministic while
// kRcWarps x total/32 warps share the (chunks x total) reads (16 warps: 57 sequential loads each at 900 chunks;
// with 8 the 108-CTA launches for H-wide gradients were latency-bound at ~20 us).
constexpr int kRcWarps = 16;
__global__ void __launch_bounds__(32 * kRcWarps) reduce_chunks_kernel(const float* part, int chunks, int groups,
                                                                     int C, float* out, int64_t out_stride,
                                                                     float alpha, int accumulate) {
    __shared__ float red[kRcWarps][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t total = (int64_t)groups * C;
    const int64_t e = blockIdx.x * 32LL + tx;
    float acc = 0.0f;
    if (e < total) {
        int c = ty;
#pragma unroll 4
        for (; c < chunks; c += kRcWarps) acc += part[(int64_t)c * total + e];
    }
    red[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && e < total) {
        float sum = 0.0f;
#pragma unroll
        for (int r = 0; r < kRcWarps; ++r) sum += red[r][tx];
        const int gidx = static_cast<int>(e / C), j = static_cast<int>(e % C);
        float* o = out + gidx * out_stride + j;
        *o = accumulate ? *o + alpha * sum : alpha * sum;
    }
}
void reduce_chunks(const float* part, int chunks, int C, float* out, float alpha, int accumulate, cudaStream_t s) {
    reduce_chunks_kernel<<<(C + 31) / 32, 32 * kRcWarps, 0, s>>>(part, chunks, 1, C, out, 0, alpha, accumulate); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
void reduce_chunks_grouped(const float* part, int chunks, int groups, int C, float* out, int64_t out_stride,
                           float alpha, int accumulate, cudaStream_t s) {
    reduce_chunks_kernel<<<static_cast<int>(((int64_t)groups * C + 31) / 32), 32 * kRcWarps, 0, s>>>(
        part, chunks, groups, C, out, out_stride, alpha, accumulate); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ modulation / gmlp backward
// dW_mod[k, j] += sum_u dm[u, k] gb[u, j] ; db_mod[k] += sum_u dm[u, k]
__global__ void mod_wgrad_kernel(const float* dm, const double* gb, int n_u, int H, float* dw, float* db) {
    const int64_t total = (int64_t)6 * H * H;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / H;
        const int j = static_cast<int>(e % H);
        double acc = 0.0;
        for (int u = 0; u < n_u; ++u) acc += static_cast<double>(dm[(int64_t)u * 6 * H + k]) * gb[(int64_t)u * H + j];
        dw[e] += static_cast<float>(acc);
        if (j == 0) {
            double b = 0.0;
            for (int u = 0; u < n_u; ++u) b += dm[(int64_t)u * 6 * H + k];
            db[k] += static_cast<float>(b);
        }
    }
}
// The same update with one grid row per output row k and 4 columns per thread (no 64-bit index division,
// 16-byte dW accesses); identical per-element arithmetic, so identical results.
__global__ void mod_wgrad_rows_kernel(const float* dm, const double* gb, int n_u, int H, float* dw, float* db) {
    const int64_t k = blockIdx.y;
    const int j = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (j < H) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int u = 0; u < n_u; ++u) {
            const double d = static_cast<double>(dm[(int64_t)u * 6 * H + k]);
            const double* g = gb + (int64_t)u * H + j;
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[c] += d * g[c];
        }
        float4* o = reinterpret_cast<float4*>(dw + k * H + j);
        float4 v = *o;
        v.x += static_cast<float>(acc[0]);
        v.y += static_cast<float>(acc[1]);
        v.z += static_cast<float>(acc[2]);
        v.w += static_cast<float>(acc[3]);
        *o = v;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double b = 0.0;
        for (int u = 0; u < n_u; ++u) b += dm[(int64_t)u * 6 * H + k];
        db[k] += static_cast<float>(b);
    }
}
// out[r, j] = sum_k in[r, k] W[k, j] for R <= 3 rows per launch, fp64 accumulation, split over K:
// thread = column j of one K-slice; all rows share each W read.  part[ks][r][j], then a
// fixed-order reduce over the slices (deterministic).
constexpr int VM_KS = 48;
template <class TI, int R>
__global__ void vecmat_part_kernel(const TI* in, int64_t in_ld, int rows, const float* W, int K, int J, double* part) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int ks = blockIdx.y;
    if (j >= J) return;
    const int per = (K + VM_KS - 1) / VM_KS;
    const int k0 = ks * per, k1 = min(K, k0 + per);
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    // unrolled so that several W rows are in flight per thread (the loop was load-latency bound at ~1.4 TB/s);
    // the accumulation order is unchanged
#pragma unroll 8
    for (int k = k0; k < k1; ++k) {
        const double w = static_cast<double>(W[(int64_t)k * J + j]);
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (r < rows) acc[r] += static_cast<double>(in[(int64_t)r * in_ld + k]) * w;
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (r < rows) part[((int64_t)ks * R + r) * J + j] = acc[r];
}
// out[r, j] = sum_ks part[ks][r][j]  (x silu'(z[r, j]) when z != null)
template <int R>
__global__ void vecmat_reduce_kernel(const double* part, int rows, int J, const double* z, double* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= J) return;
    for (int r = 0; r < rows; ++r) {
        double acc = 0.0;
        for (int ks = 0; ks < VM_KS; ++ks) acc += part[((int64_t)ks * R + r) * J + j];
        if (z) {
            const double zz = z[(int64_t)r * J + j];
            const double sg = 1.0 / (1.0 + exp(-zz));
            acc *= sg + zz * sg * (1.0 - sg);
        }
        out[(int64_t)r * J + j] = acc;
    }
}
template <class TI>
static void vecmat(const TI* in, int64_t in_ld, int rows, const float* W, int K, int J, const double* z, double* out,
                   cudaStream_t s) {
    double* part = nullptr;
    MGV_CUDA(cudaMallocAsync(&part, sizeof(double) * VM_KS * 3 * (size_t)J, s));
    for (int r0 = 0; r0 < rows; r0 += 3) {  // row blocks of 3 (a packed batch has one timestep row per sample)
        const int rb = rows - r0 < 3 ? rows - r0 : 3;
        vecmat_part_kernel<TI, 3><<<dim3((J + 255) / 256, VM_KS), 256, 0, s>>>(in + (int64_t)r0 * in_ld, in_ld, rb, W,
                                                                                K, J, part);
        ::mgv::note_launch();
        vecmat_reduce_kernel<3><<<(J + 255) / 256, 256, 0, s>>>(part, rb, J, z ? z + (int64_t)r0 * J : nullptr,
                                                                 out + (int64_t)r0 * J);
        ::mgv::note_launch();
    }
    MGV_CUDA(cudaFreeAsync(part, s));
    MGV_CUDA(cudaGetLastError());
}
void modulation_bwd(const float* dm, const double* gb, const float* w_mod, int n_u, int H, float* dw_mod,
                    float* db_mod, double* dgb, cudaStream_t s) {
    if (H % 4 == 0) {
        mod_wgrad_rows_kernel<<<dim3((H / 4 + 255) / 256, 6 * H), 256, 0, s>>>(dm, gb, n_u, H, dw_mod, db_mod);
    } else {
        mod_wgrad_kernel<<<grid_for((int64_t)6 * H * H), 256, 0, s>>>(dm, gb, n_u, H, dw_mod, db_mod);
    }
    ::mgv::note_launch();
    vecmat<float>(dm, 6 * H, n_u, w_mod, 6 * H, H, nullptr, dgb, s);  // dgb = dm W_mod
    MGV_CUDA(cudaGetLastError());
}
__global__ void gscale_bwd_kernel(const double* dgb, const double* g, const float* gs, int n_u, int H, float* dgs,
                                  double* dg) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= H) return;
    double acc = 0.0;
    for (int u = 0; u < n_u; ++u) {
        acc += dgb[(int64_t)u * H + j] * g[(int64_t)u * H + j];
        dg[(int64_t)u * H + j] += dgb[(int64_t)u * H + j] * static_cast<double>(gs[j]);
    }
    dgs[j] += static_cast<float>(acc);
}
void gscale_bwd(const double* dgb, const double* g, const float* gscale, int n_u, int H, float* dgscale, double* dg,
                cudaStream_t s) {
    gscale_bwd_kernel<<<(H + 255) / 256, 256, 0, s>>>(dgb, g, gscale, n_u, H, dgscale, dg); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
// rows R = n_u + 1 (last = fps row, gradient = sum_u dg_u)
__global__ void gmlp_out_bwd_kernel(const double* dg, int n_u, const double* h_in, int H, float* dw_out, float* db_out) {
    const int64_t total = (int64_t)H * H;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / H;
        const int j = static_cast<int>(e % H);
        double acc = 0.0, dgf = 0.0;
        for (int u = 0; u < n_u; ++u) {
            const double d = dg[(int64_t)u * H + k];
            acc += d * h_in[(int64_t)u * H + j];
            dgf += d;
        }
        acc += dgf * h_in[(int64_t)n_u * H + j];
        dw_out[e] += static_cast<float>(acc);
        if (j == 0) db_out[k] += static_cast<float>(2.0 * dgf);  // both MLP evaluations add b_out
    }
}
// rows of the gmlp output gradient: dg_u (u < n_u) and the fps row sum_u dg_u
__global__ void gmlp_rows_kernel(const double* dg, int n_u, int H, double* rows) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= H) return;
    double f = 0.0;
    for (int u = 0; u < n_u; ++u) {
        rows[(int64_t)u * H + k] = dg[(int64_t)u * H + k];
        f += dg[(int64_t)u * H + k];
    }
    rows[(int64_t)n_u * H + k] = f;
}
__global__ void gmlp_in_bwd_kernel(const double* dz, int R, const double* phi, int H, float* dw_in, float* db_in) {
    const int64_t total = (int64_t)H * 32;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / 32;
        const int k = static_cast<int>(e % 32);
        double acc = 0.0, b = 0.0;
        for (int r = 0; r < R; ++r) {
            acc += dz[(int64_t)r * H + j] * phi[r * 32 + k];
            b += dz[(int64_t)r * H + j];
        }
        dw_in[e] += static_cast<float>(acc);
        if (k == 0) db_in[j] += static_cast<float>(b);
    }
}
void global_embed_bwd(const double* dg, int n_u, const double* phi, const double* z_in, const double* h_in,
                      const float* w_out, int H, float* dw_in, float* db_in, float* dw_out, float* db_out,
                      cudaStream_t s) {
    // scratch dz lives after h_in's rows? keep it simple: allocate per call (tiny, (n_u+1) x H doubles)
    double *dz = nullptr, *rows = nullptr;
    MGV_CUDA(cudaMallocAsync(&dz, sizeof(double) * (size_t)(n_u + 1) * H, s));
    MGV_CUDA(cudaMallocAsync(&rows, sizeof(double) * (size_t)(n_u + 1) * H, s));
    gmlp_out_bwd_kernel<<<grid_for((int64_t)H * H), 256, 0, s>>>(dg, n_u, h_in, H, dw_out, db_out); ::mgv::note_launch();
    gmlp_rows_kernel<<<(H + 255) / 256, 256, 0, s>>>(dg, n_u, H, rows); ::mgv::note_launch();
    vecmat<double>(rows, H, n_u + 1, w_out, H, H, z_in, dz, s);  // dz = (rows W_out) * silu'(z_in)
    gmlp_in_bwd_kernel<<<grid_for((int64_t)H * 32), 256, 0, s>>>(dz, n_u + 1, phi, H, dw_in, db_in); ::mgv::note_launch();
    MGV_CUDA(cudaFreeAsync(rows, s));
    MGV_CUDA(cudaFreeAsync(dz, s));
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ misc
__global__ void sumsq_kernel(const float* x, int64_t n, double* part) {
    __shared__ double red[RT / 32];
    double acc = 0.0;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += RT) acc += static_cast<double>(x[i]) * x[i];
    acc = block_sum_d(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
void sumsq(const float* x, int64_t n, double* part, double* out, cudaStream_t s) {
    sumsq_kernel<<<1024, RT, 0, s>>>(x, n, part); ::mgv::note_launch();
    sum_double_kernel<<<1, 1, 0, s>>>(part, 1024, out); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
__global__ void fill_kernel(float* p, int64_t n, float v) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}
__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) p[e] = v;
}
void fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t s) {
    fill_i32_kernel<<<grid_for(n), 256, 0, s>>>(p, n, v); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
void fill_f32(float* p, int64_t n, float v, cudaStream_t s) {
    fill_kernel<<<grid_for(n), 256, 0, s>>>(p, n, v); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

// ============================================================ instantiations
// ============================================================ tensor-parallel glue
template <class T>
__global__ void bias_gate_resid_kernel(const float* part, const float* bias, const float* table, int64_t tld,
                                       int gate_off, const int32_t* mod_id, const float* Xin, float* Xout, T* y_out,
                                       int N, int H) {
    const int64_t n = (int64_t)N * H;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = e / H;
        const int j = static_cast<int>(e - m * H);
        const float y = part[e] + bias[j];
        const float g = table[(int64_t)mod_id[m] * tld + gate_off + j];
        Xout[e] = Xin[e] + y * g;  // same expression as EpiGateResid
        y_out[e] = to_t<T>(y);
    }
}
template <class T>
void bias_gate_resid(const float* part, const float* bias, const float* table, int64_t tld, int gate_off,
                     const int32_t* mod_id, const float* Xin, float* Xout, T* y_out, int N, int H, cudaStream_t s) {
    bias_gate_resid_kernel<T><<<grid_for((int64_t)N * H), 256, 0, s>>>(part, bias, table, tld, gate_off, mod_id, Xin,
                                                                         Xout, y_out, N, H);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
template <class T>
__global__ void bias_to_kernel(const float* part, const float* bias, T* out, int N, int H) {
    const int64_t n = (int64_t)N * H;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = to_t<T>(part[e] + (bias ? bias[e % H] : 0.0f));
}
template <class T>
void bias_to(const float* part, const float* bias, T* out, int N, int H, cudaStream_t s) {
    bias_to_kernel<T><<<grid_for((int64_t)N * H), 256, 0, s>>>(part, bias, out, N, H);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
// dst row (v, c, j) <- src row (c, v, j) for C chunks of R = P * Rs rows (inverse swaps the roles)
template <class E>
__global__ void permute_shard_rows_kernel(const E* src, E* dst, int C, int R, int P, int64_t cols, int inverse) {
    const int Rs = R / P;
    const int64_t n = (int64_t)C * R * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / cols, col = e - row * cols;
        const int c = static_cast<int>(row / R), rr = static_cast<int>(row % R);
        const int v = rr / Rs, j = rr % Rs;
        const int64_t rank_major = ((int64_t)v * C + c) * Rs + j;  // row index in the rank-major layout
        if (inverse)
            dst[row * cols + col] = src[rank_major * cols + col];
        else
            dst[rank_major * cols + col] = src[row * cols + col];
    }
}
// column-parallel shard layout: (rows x cols) row-major <-> P rank-major blocks, block v = columns
// [v cols/P, (v+1) cols/P) stored compact (rows x cols/P)
template <class E>
__global__ void permute_shard_cols_kernel(const E* src, E* dst, int64_t rows, int64_t cols, int P, int inverse) {
    const int64_t cs = cols / P, n = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / cols, c = e - i * cols, v = c / cs, j = c - v * cs;
        const int64_t rm = (v * rows + i) * cs + j;
        if (inverse)
            dst[e] = src[rm];
        else
            dst[rm] = src[e];
    }
}
void permute_shard_cols(const float* src, float* dst, int64_t rows, int64_t cols, int P, int inverse, cudaStream_t s) {
    permute_shard_cols_kernel<float><<<grid_for(rows * cols), 256, 0, s>>>(src, dst, rows, cols, P, inverse);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
void permute_shard_cols(const double* src, double* dst, int64_t rows, int64_t cols, int P, int inverse,
                        cudaStream_t s) {
    permute_shard_cols_kernel<double><<<grid_for(rows * cols), 256, 0, s>>>(src, dst, rows, cols, P, inverse);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
void permute_shard_rows(const float* src, float* dst, int C, int R, int P, int64_t cols, int inverse, cudaStream_t s) {
    permute_shard_rows_kernel<float><<<grid_for((int64_t)C * R * cols), 256, 0, s>>>(src, dst, C, R, P, cols, inverse);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
void permute_shard_rows(const double* src, double* dst, int C, int R, int P, int64_t cols, int inverse,
                        cudaStream_t s) {
    permute_shard_rows_kernel<double><<<grid_for((int64_t)C * R * cols), 256, 0, s>>>(src, dst, C, R, P, cols, inverse);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

#define INST(T)                                                                                                       \
    template void prep_flow_sample<T>(const double*, const double*, const uint8_t*, const double*, int, int, double, \
                                      T*, float*, uint8_t*, int32_t*, cudaStream_t, int, int);                        \
    template void convert_rows<T>(const double*, int64_t, T*, cudaStream_t);                                          \
    template void convert_f32<T>(const float*, int64_t, T*, cudaStream_t);                                            \
    template void rms_mod<T>(const float*, int, int, const float*, int64_t, int, int, const int32_t*, T*, float*,     \
                             cudaStream_t);                                                                           \
    template void rms_gain<T>(const float*, int, int, const float*, T*, float*, cudaStream_t);                        \
    template void postnorm_resid<T>(const float*, const T*, int, int, const float*, float*, float*, cudaStream_t);    \
    template bool postnorm_resid_mod<T>(const float*, const T*, int, int, const float*, float*, float*, const float*, \
                                        int64_t, int, int, const int32_t*, T*, float*, cudaStream_t);                \
    template void qk_norm_rope<T>(const T*, const QKLayout&, int, int, int, const float*, const float2*, T*, float*,  \
                                  float*, cudaStream_t);                                                              \
    template void bias_gate_resid<T>(const float*, const float*, const float*, int64_t, int, const int32_t*,          \
                                     const float*, float*, T*, int, int, cudaStream_t);                               \
    template void bias_to<T>(const float*, const float*, T*, int, int, cudaStream_t);                                 \
    template void flow_loss_fwd<T>(const float*, const float*, const uint8_t*, int, int, double*, cudaStream_t);      \
    template void flow_loss_bwd<T>(const float*, const float*, const uint8_t*, int, int, float, const int*, T*,       \
                                   cudaStream_t);                                                                    \
    template void gate_bwd<T>(const float*, const T*, const float*, int64_t, int, const int32_t*, int, int, int, T*,  \
                              float*, float*, cudaStream_t);                                                          \
    template void rms_mod_bwd<T>(const T*, const float*, const float*, const float*, int64_t, int, int,               \
                                 const int32_t*, int, int, int, float*, float*, float*, cudaStream_t);                \
    template void rms_gain_bwd<T>(const T*, const float*, const float*, const float*, int, int, float*, int, float*,  \
                                  cudaStream_t);                                                                      \
    template void postnorm_bwd<T>(const float*, const T*, const float*, const float*, int, int, T*, float*,           \
                                  cudaStream_t);                                                                      \
    template void qk_norm_rope_bwd<T>(T*, const T*, const QKLayout&, int, int, int, const float*, const float2*,      \
                                      const float*, const float*, float*, cudaStream_t);                              \
    template void colsum<T>(const T*, int64_t, int, int, float*, cudaStream_t);
INST(float)
INST(__nv_bfloat16)
#undef INST

}  // namespace mgv

namespace mgv {
// 64 x 64 tiles through shared memory: coalesced 16-byte reads along columns and writes along rows.
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const __nv_bfloat16* __restrict__ in, int64_t ld_in,
                                                             int rows, int cols, __nv_bfloat16* __restrict__ out,
                                                             int64_t ld_out) {
    __shared__ __nv_bfloat16 t[64][66];
    const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
    const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;  // 8 x 32
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = ty + 32 * k;
        const int gr = r0 + r, gc = c0 + tx * 8;
        __nv_bfloat16 v[8];
        if (gr < rows && gc + 8 <= cols && (((uintptr_t)(in + (int64_t)gr * ld_in + gc)) & 15) == 0) {
            *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(in + (int64_t)gr * ld_in + gc);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                v[e] = (gr < rows && gc + e < cols) ? in[(int64_t)gr * ld_in + gc + e] : __float2bfloat16_rn(0.0f);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) t[r][tx * 8 + e] = v[e];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int c = ty + 32 * k;  // output row = input column
        const int gc = c0 + c, gr = r0 + tx * 8;
        if (gc >= cols) continue;
        __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = t[tx * 8 + e][c];
        __nv_bfloat16* dst = out + (int64_t)gc * ld_out + gr;
        if (gr + 8 <= rows && (((uintptr_t)dst) & 15) == 0) {
            *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<uint4*>(v);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (gr + e < rows) dst[e] = v[e];
        }
    }
}
void transpose_bf16(const __nv_bfloat16* in, int64_t ld_in, int rows, int cols, __nv_bfloat16* out, int64_t ld_out,
                    cudaStream_t s) {
    dim3 grid((cols + 63) / 64, (rows + 63) / 64);
    transpose_bf16_kernel<<<grid, 256, 0, s>>>(in, ld_in, rows, cols, out, ld_out); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
}  // namespace mgv

// ======================================================================================
// Vectorised bf16 row kernels (H % 8 == 0, H <= 4096): 16-byte accesses, 2 rows per block
// reduction.  Dispatched from the launchers above when T = bf16.
#include "kernels_vec.cuh"

namespace mgv {
namespace vec {

using bf = __nv_bfloat16;

template <int MODE>  // 0: out = n (1 + sc) + sh ; 1: out = n * g
__global__ void __launch_bounds__(RT) rms_fwd_vec(const float* X, int N, int H, const float* table, int64_t tld,
                                                  int sh_off, int sc_off, const int32_t* mod_id, const float* g,
                                                  bf* out, float* rs) {
    __shared__ float red[R][RT / 32];
    const int G = H / 8;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    for (int i = r0; i < r1; i += R) {
        float v[R][VG][8], ss[R];
        // the next row group: start its rows into L2 while this group reduces (block barrier below)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int nrow = i + R + rr;
            if (nrow >= r1) break;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(X + (int64_t)nrow * H + grp * 8));
            }
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            ss[rr] = 0.0f;
            const int row = i + rr;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (row < r1 && grp < G) {
                    ld8(X + (int64_t)row * H + grp * 8, v[rr][k]);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) v[rr][k][e] = 0.0f;
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) ss[rr] = fmaf(v[rr][k][e], v[rr][k][e], ss[rr]);
            }
        }
        block_sum_r(ss, red);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int row = i + rr;
            if (row >= r1) continue;
            const float rstd = 1.0f / sqrtf(ss[rr] / static_cast<float>(H) + 1e-6f);
            if (threadIdx.x == 0) rs[row] = rstd;
            const float* tb = MODE == 0 ? table + (int64_t)mod_id[row] * tld : nullptr;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                float o[8], a[8], b[8];
                if (MODE == 0) {
                    ld8(tb + sc_off + grp * 8, a);
                    ld8(tb + sh_off + grp * 8, b);
#pragma unroll
                    for (int e = 0; e < 8; ++e) o[e] = v[rr][k][e] * rstd * (1.0f + a[e]) + b[e];
                } else {
                    ld8(g + grp * 8, a);
#pragma unroll
                    for (int e = 0; e < 8; ++e) o[e] = v[rr][k][e] * rstd * a[e];
                }
                st8(out + (int64_t)row * H + grp * 8, o);
            }
        }
    }
}

// X2 = X1 + rms(co) * g (dit.cpp:305); MOD: the FFN's modulated RMSNorm of the new rows in the same pass
// (dit.cpp:308, f = rms(X2)(1 + sc2) + sh2 and its 1/rms r2), with rms_fwd_vec<0>'s per-thread order and block
// reduction, so f and r2 are bit-identical to running it on X2 afterwards
template <bool MOD>
__global__ void __launch_bounds__(RT) postnorm_resid_vec(const float* X1, const bf* co, int N, int H, const float* g,
                                                         float* X2, float* rc, const float* table, int64_t tld,
                                                         int sh_off, int sc_off, const int32_t* mod_id, bf* f,
                                                         float* r2) {
    __shared__ float red[R][RT / 32];
    const int G = H / 8;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    for (int i = r0; i < r1; i += R) {
        float v[R][VG][8], ss[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            ss[rr] = 0.0f;
            const int row = i + rr;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (row < r1 && grp < G) {
                    ld8(co + (int64_t)row * H + grp * 8, v[rr][k]);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) v[rr][k][e] = 0.0f;
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) ss[rr] = fmaf(v[rr][k][e], v[rr][k][e], ss[rr]);
            }
        }
        block_sum_r(ss, red);
        float ss2[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int row = i + rr;
            ss2[rr] = 0.0f;
            if (row >= r1) continue;
            const float rstd = 1.0f / sqrtf(ss[rr] / static_cast<float>(H) + 1e-6f);
            if (threadIdx.x == 0) rc[row] = rstd;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                float x[8], gg[8];
                ld8(X1 + (int64_t)row * H + grp * 8, x);
                ld8(g + grp * 8, gg);
#pragma unroll
                for (int e = 0; e < 8; ++e) x[e] += v[rr][k][e] * rstd * gg[e];
                st8(X2 + (int64_t)row * H + grp * 8, x);
                if (MOD) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        v[rr][k][e] = x[e];  // co is consumed: keep the new residual row
                        ss2[rr] = fmaf(x[e], x[e], ss2[rr]);
                    }
                }
            }
        }
        if (!MOD) continue;
        block_sum_r(ss2, red);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int row = i + rr;
            if (row >= r1) continue;
            const float rstd = 1.0f / sqrtf(ss2[rr] / static_cast<float>(H) + 1e-6f);
            if (threadIdx.x == 0) r2[row] = rstd;
            const float* tb = table + (int64_t)mod_id[row] * tld;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                float o[8], a[8], b[8];
                ld8(tb + sc_off + grp * 8, a);
                ld8(tb + sh_off + grp * 8, b);
#pragma unroll
                for (int e = 0; e < 8; ++e) o[e] = v[rr][k][e] * rstd * (1.0f + a[e]) + b[e];
                st8(f + (int64_t)row * H + grp * 8, o);
            }
        }
    }
}

// dY = dX * gate[u] ; partials: grouped sum dX*y, sum dY
__global__ void __launch_bounds__(RT) gate_bwd_vec(const float* __restrict__ dX, const bf* __restrict__ y,
                                                   const float* __restrict__ table, int64_t tld, int gate_off,
                                                   const int32_t* __restrict__ mod_id, int n_u, int N, int H,
                                                   bf* __restrict__ dY, float* part_dgate, float* part_db) {
    const int G = H / 8;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float pg[2][VG][8], pb[VG][8];
#pragma unroll
    for (int k = 0; k < VG; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) pg[0][k][e] = pg[1][k][e] = pb[k][e] = 0.0f;
    int ua, ub;
    chunk_rows(mod_id, r0, r1, ua, ub);
#pragma unroll 2  // restrict + two rows in flight: the next row's loads issue before this row's stores
    for (int i = r0; i < r1; ++i) {
        const int u = mod_id[i];
        const float* gt = table + (int64_t)u * tld + gate_off;
#pragma unroll
        for (int k = 0; k < VG; ++k) {
            const int grp = threadIdx.x + k * RT;
            if (grp >= G) continue;
            float dx[8], yy[8], gg[8], d[8];
            ld8(dX + (int64_t)i * H + grp * 8, dx);
            ld8(y + (int64_t)i * H + grp * 8, yy);
            ld8(gt + grp * 8, gg);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                d[e] = dx[e] * gg[e];
                pb[k][e] += d[e];
                const float t = dx[e] * yy[e];
                if (u == ua) pg[0][k][e] += t; else pg[1][k][e] += t;
            }
            st8(dY + (int64_t)i * H + grp * 8, d);
        }
    }
#pragma unroll
    for (int k = 0; k < VG; ++k) {
        const int grp = threadIdx.x + k * RT;
        if (grp >= G) continue;
        st8(part_db + (int64_t)blockIdx.x * H + grp * 8, pb[k]);
        float zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int u = 0; u < n_u; ++u)
            st8(part_dgate + ((int64_t)blockIdx.x * n_u + u) * H + grp * 8,
                u == ua ? pg[0][k] : (u == ub ? pg[1][k] : zero));
    }
}

// rms backward; MODE 0: dn = dA (1 + sc[u]), partials d shift / d scale (grouped); MODE 1: dn = dA g, partial d gain
template <int MODE>
__global__ void __launch_bounds__(RT, 2) rms_bwd_vec(const bf* dA, const float* X, const float* rs, const float* table,
                                                  int64_t tld, int sc_off, const int32_t* mod_id, int n_u,
                                                  const float* g, int N, int H, float* dX, int accumulate,
                                                  float* part_a, float* part_b) {
    __shared__ float red[R][RT / 32];
    const int G = H / 8;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float pa[2][VG][8], pb[2][VG][8];
#pragma unroll
    for (int k = 0; k < VG; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) pa[0][k][e] = pa[1][k][e] = pb[0][k][e] = pb[1][k][e] = 0.0f;
    int ua = 0, ub = 0;
    if (MODE == 0) chunk_rows(mod_id, r0, r1, ua, ub);
    for (int i = r0; i < r1; i += R) {
        float xv[R][VG][8], dn[R][VG][8], dot[R];
        // the next row group: start its rows into L2 while this group reduces (block barrier below)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int nrow = i + R + rr;
            if (nrow >= r1) break;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(dA + (int64_t)nrow * H + grp * 8));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(X + (int64_t)nrow * H + grp * 8));
            }
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            dot[rr] = 0.0f;
            const int row = i + rr;
            const bool ok = row < r1;
            const int u = (MODE == 0 && ok) ? mod_id[row] : 0;
            const float rstd = ok ? rs[row] : 0.0f;
            const float* tb = MODE == 0 ? table + (int64_t)u * tld + sc_off : g;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (ok && grp < G) {
                    // the dX accumulate read comes after the row reduction: start it now, into L2
                    if (accumulate) asm volatile("prefetch.global.L2 [%0];" ::"l"(dX + (int64_t)row * H + grp * 8));
                    float da[8], t[8];
                    ld8(dA + (int64_t)row * H + grp * 8, da);
                    ld8(X + (int64_t)row * H + grp * 8, xv[rr][k]);
                    ld8(tb + grp * 8, t);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float n = xv[rr][k][e] * rstd;
                        if (MODE == 0) {
                            dn[rr][k][e] = da[e] * (1.0f + t[e]);
                            if (u == ua) {
                                pa[0][k][e] += da[e];
                                pb[0][k][e] += da[e] * n;
                            } else {
                                pa[1][k][e] += da[e];
                                pb[1][k][e] += da[e] * n;
                            }
                        } else {
                            dn[rr][k][e] = da[e] * t[e];
                            pa[0][k][e] += da[e] * n;
                        }
                        dot[rr] = fmaf(dn[rr][k][e], xv[rr][k][e], dot[rr]);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) xv[rr][k][e] = dn[rr][k][e] = 0.0f;
                }
            }
        }
        block_sum_r(dot, red);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int row = i + rr;
            if (row >= r1) continue;
            const float rstd = rs[row];
            const float kk = dot[rr] * rstd * rstd * rstd / static_cast<float>(H);
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                float o[8];
                if (accumulate) ld8(dX + (int64_t)row * H + grp * 8, o);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float d = dn[rr][k][e] * rstd - xv[rr][k][e] * kk;
                    o[e] = accumulate ? o[e] + d : d;
                }
                st8(dX + (int64_t)row * H + grp * 8, o);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < VG; ++k) {
        const int grp = threadIdx.x + k * RT;
        if (grp >= G) continue;
        if (MODE == 0) {
            float zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int u = 0; u < n_u; ++u) {
                st8(part_a + ((int64_t)blockIdx.x * n_u + u) * H + grp * 8,
                    u == ua ? pa[0][k] : (u == ub ? pa[1][k] : zero));
                st8(part_b + ((int64_t)blockIdx.x * n_u + u) * H + grp * 8,
                    u == ua ? pb[0][k] : (u == ub ? pb[1][k] : zero));
            }
        } else {
            st8(part_a + (int64_t)blockIdx.x * H + grp * 8, pa[0][k]);
        }
    }
}

__global__ void __launch_bounds__(RT) postnorm_bwd_vec(const float* dX, const bf* co, const float* rc, const float* g,
                                                       int N, int H, bf* dco, float* part_dg) {
    __shared__ float red[R][RT / 32];
    const int G = H / 8;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float pg[VG][8];
#pragma unroll
    for (int k = 0; k < VG; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) pg[k][e] = 0.0f;
    for (int i = r0; i < r1; i += R) {
        float xv[R][VG][8], dn[R][VG][8], dot[R];
        // the next row group: start its rows into L2 while this group reduces (block barrier below)
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int nrow = i + R + rr;
            if (nrow >= r1) break;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(dX + (int64_t)nrow * H + grp * 8));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(co + (int64_t)nrow * H + grp * 8));
            }
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            dot[rr] = 0.0f;
            const int row = i + rr;
            const bool ok = row < r1;
            const float rr_s = ok ? rc[row] : 0.0f;
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (ok && grp < G) {
                    float dx[8], gg[8];
                    ld8(dX + (int64_t)row * H + grp * 8, dx);
                    ld8(co + (int64_t)row * H + grp * 8, xv[rr][k]);
                    ld8(g + grp * 8, gg);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        pg[k][e] += dx[e] * xv[rr][k][e] * rr_s;
                        dn[rr][k][e] = dx[e] * gg[e];
                        dot[rr] = fmaf(dn[rr][k][e], xv[rr][k][e], dot[rr]);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) xv[rr][k][e] = dn[rr][k][e] = 0.0f;
                }
            }
        }
        block_sum_r(dot, red);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
            const int row = i + rr;
            if (row >= r1) continue;
            const float rstd = rc[row];
            const float kk = dot[rr] * rstd * rstd * rstd / static_cast<float>(H);
#pragma unroll
            for (int k = 0; k < VG; ++k) {
                const int grp = threadIdx.x + k * RT;
                if (grp >= G) continue;
                float o[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) o[e] = dn[rr][k][e] * rstd - xv[rr][k][e] * kk;
                st8(dco + (int64_t)row * H + grp * 8, o);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < VG; ++k) {
        const int grp = threadIdx.x + k * RT;
        if (grp < G) st8(part_dg + (int64_t)blockIdx.x * H + grp * 8, pg[k]);
    }
}

// column sums of a bf16 matrix: thread = 8 columns, CTA = (row chunk, 2048-column block)
__global__ void __launch_bounds__(RT) colsum_vec(const bf* Y, int64_t ld, int N, int C, float* part) {
    const int grp = blockIdx.y * RT + threadIdx.x;
    if (grp * 8 >= C) return;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = r0; i < r1; ++i) {
        float v[8];
        ld8(Y + (int64_t)i * ld + grp * 8, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += v[e];
    }
    st8(part + (int64_t)blockIdx.x * C + grp * 8, acc);
}


// ---- QK-norm + temperature + RoPE (dit.cpp:289-294), bf16, head_dim % 8 == 0: lane l < hd/8 owns the
// 8 consecutive elements [8l, 8l+8) = rotation pairs [4l, 4l+4) of one (token, q|k, head) vector, so
// each vector is one 16-byte load / store per lane instead of hd/2 4-byte ones.
__device__ __forceinline__ float warp_sum_v(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}
__device__ __forceinline__ void ld_cs4(const float2* cs, float* c, float* sn) {  // 4 (cos, sin) pairs
    const float4 a = reinterpret_cast<const float4*>(cs)[0], b = reinterpret_cast<const float4*>(cs)[1];
    c[0] = a.x; sn[0] = a.y; c[1] = a.z; sn[1] = a.w; c[2] = b.x; sn[2] = b.y; c[3] = b.z; sn[3] = b.w;
}
constexpr int QKV = 4;  // vectors (heads) per warp in flight
__global__ void __launch_bounds__(256) qk_norm_rope_vec(const bf* qkv, QKLayout Lq, int N, int hd, int heads,
                                                        const float* temp, const float2* cs, bf* qk, float* iq,
                                                        float* ik) {
    const int hg = (heads + QKV - 1) / QKV;  // head groups
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (gw >= (int64_t)N * 2 * hg) return;
    const int h0 = static_cast<int>(gw % hg) * QKV;
    const int which = static_cast<int>((gw / hg) % 2);
    const int64_t n = gw / (2 * hg);
    const bool act = lane < hd / 8;
    float v[QKV][8];
#pragma unroll
    for (int u = 0; u < QKV; ++u) {  // all loads first (independent, in flight together)
#pragma unroll
        for (int e = 0; e < 8; ++e) v[u][e] = 0.0f;
        if (act && h0 + u < heads) ld8(qkv + n * Lq.in_ld + which * Lq.in_koff + (h0 + u) * hd + 8 * lane, v[u]);
    }
    float c[4] = {0, 0, 0, 0}, sn[4] = {0, 0, 0, 0};
    if (act) ld_cs4(cs + n * (hd / 2) + 4 * lane, c, sn);
    float ss[QKV];
#pragma unroll
    for (int u = 0; u < QKV; ++u) {
        ss[u] = 0.0f;
#pragma unroll
        for (int e = 0; e < 8; ++e) ss[u] = fmaf(v[u][e], v[u][e], ss[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < QKV; ++u) ss[u] += __shfl_xor_sync(0xffffffff, ss[u], o);
#pragma unroll
    for (int u = 0; u < QKV; ++u) {
        const int h = h0 + u;
        if (h >= heads) break;
        const float iv = 1.0f / sqrtf(ss[u] + 1e-6f);  // autodiff.cpp:727
        if (lane == 0) (which == 0 ? iq : ik)[n * Lq.i_ld + h] = iv;
        if (!act) continue;
        const float sc = which == 0 ? iv * temp[h] : iv;  // dit.cpp:292
        float o[8];
#pragma unroll
        for (int k = 0; k < 4; ++k)  // autodiff.cpp:864-865, the roundings of the fused QKV epilogue
            rope_pair(__fmul_rn(v[u][2 * k], sc), __fmul_rn(v[u][2 * k + 1], sc), c[k], sn[k], o[2 * k], o[2 * k + 1]);
        st8(qk + n * Lq.out_ld + which * Lq.out_koff + h * hd + 8 * lane, o);
    }
}

// backward: CTA = (chunk of kRowsPerChunk rows, 8 heads), warp = one head over the chunk (fixed-order dtemp
// partials); two rows x (q, k) are processed per iteration so four vectors' loads are in flight
constexpr int QRU = 1;  // rows per iteration of the backward (x (q, k) vectors in flight)
__global__ void __launch_bounds__(256) qk_norm_rope_bwd_vec(bf* dqkv, const bf* qkv, QKLayout Lq, int N, int hd,
                                                            int heads, const float* temp, const float2* cs,
                                                            const float* iq, const float* ik, float* part_dtemp) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const bool act = lane < hd / 8;
    const int r0 = blockIdx.x * kRowsPerChunk, r1 = min(N, r0 + kRowsPerChunk);
    for (int h = blockIdx.y * 8 + warp; h < heads; h += 8 * gridDim.y) {  // one head per warp
        const float tq = temp[h];
        float dtemp = 0.0f;
        for (int n0 = r0; n0 < r1; n0 += QRU) {
            // vectors u = 2 * (row - n0) + which: QRU rows x (q, k), loads all in flight
            float c[QRU][4], sn[QRU][4], d[2 * QRU][8], x[2 * QRU][8], iv[2 * QRU];
            int64_t off[2 * QRU];
            bool ok[2 * QRU];
            if (act)  // the next row group's q / k slices of dqkv and qkv: start them into L2 now
#pragma unroll
                for (int rr = 0; rr < QRU; ++rr) {
                    const int nn = n0 + QRU + rr;
                    if (nn >= r1) break;
#pragma unroll
                    for (int which = 0; which < 2; ++which) {
                        const int64_t o = (int64_t)nn * Lq.in_ld + which * Lq.in_koff + h * hd + 8 * lane;
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(dqkv + o));
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(qkv + o));
                    }
                }
#pragma unroll
            for (int rr = 0; rr < QRU; ++rr) {
                const int n = n0 + rr;
#pragma unroll
                for (int k = 0; k < 4; ++k) c[rr][k] = sn[rr][k] = 0.0f;
                if (act && n < r1) ld_cs4(cs + (int64_t)n * (hd / 2) + 4 * lane, c[rr], sn[rr]);
#pragma unroll
                for (int which = 0; which < 2; ++which) {
                    const int u = 2 * rr + which;
                    ok[u] = n < r1;
                    off[u] = (int64_t)n * Lq.in_ld + which * Lq.in_koff + h * hd + 8 * lane;
                    iv[u] = ok[u] ? (which == 0 ? iq : ik)[(int64_t)n * Lq.i_ld + h] : 0.0f;
#pragma unroll
                    for (int e = 0; e < 8; ++e) d[u][e] = x[u][e] = 0.0f;
                    if (act && ok[u]) {
                        ld8(dqkv + off[u], d[u]);
                        ld8(qkv + off[u], x[u]);
                    }
                }
            }
            float ga[2 * QRU][4], gb[2 * QRU][4], tdot[2 * QRU], dot[2 * QRU];
#pragma unroll
            for (int u = 0; u < 2 * QRU; ++u) {
                const int rr = u >> 1, which = u & 1;
                const float sc = which == 0 ? tq : 1.0f;
                tdot[u] = dot[u] = 0.0f;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // inverse rotation (autodiff.cpp:888-898)
                    ga[u][k] = d[u][2 * k] * c[rr][k] + d[u][2 * k + 1] * sn[rr][k];
                    gb[u][k] = -d[u][2 * k] * sn[rr][k] + d[u][2 * k + 1] * c[rr][k];
                    tdot[u] += (ga[u][k] * x[u][2 * k] + gb[u][k] * x[u][2 * k + 1]) * iv[u];  // d temp
                    ga[u][k] *= sc;
                    gb[u][k] *= sc;
                    dot[u] += ga[u][k] * x[u][2 * k] + gb[u][k] * x[u][2 * k + 1];
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int u = 0; u < 2 * QRU; ++u) {
                    dot[u] += __shfl_xor_sync(0xffffffff, dot[u], o);
                    tdot[u] += __shfl_xor_sync(0xffffffff, tdot[u], o);
                }
#pragma unroll
            for (int rr = 0; rr < QRU; ++rr)  // q of row n0, n0 + 1, ...: the sequential order
                if (ok[2 * rr]) dtemp += tdot[2 * rr];
#pragma unroll
            for (int u = 0; u < 2 * QRU; ++u) {
                if (!act || !ok[u]) continue;
                const float kk = dot[u] * iv[u] * iv[u] * iv[u];  // autodiff.cpp:746-748
                float o8[8];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    o8[2 * k] = ga[u][k] * iv[u] - x[u][2 * k] * kk;
                    o8[2 * k + 1] = gb[u][k] * iv[u] - x[u][2 * k + 1] * kk;
                }
                st8(dqkv + off[u], o8);
            }
        }
        if (lane == 0) part_dtemp[(int64_t)blockIdx.x * heads + h] = dtemp;
    }
}
}  // namespace vec
void qk_norm_rope_bwd_vec_launch(__nv_bfloat16* dqkv, const __nv_bfloat16* qkv, const QKLayout& L, int N, int hd, int heads,
                                 const float* temp, const float2* cs, const float* iq, const float* ik,
                                 float* part_dtemp, cudaStream_t s) {
    vec::qk_norm_rope_bwd_vec<<<dim3(row_chunks(N), (heads + 7) / 8), 256, 0, s>>>(dqkv, qkv, L, N, hd, heads, temp, cs, iq, ik, part_dtemp);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}
void qk_norm_rope_vec_launch(const __nv_bfloat16* qkv, const QKLayout& L, int N, int hd, int heads, const float* temp,
                             const float2* cs, __nv_bfloat16* qk, float* iq, float* ik, cudaStream_t s) {
    const int64_t threads = (int64_t)N * 2 * ((heads + vec::QKV - 1) / vec::QKV) * 32;
    vec::qk_norm_rope_vec<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(qkv, L, N, hd, heads, temp, cs, qk,
                                                                                 iq, ik);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

bool use_vec(int H) { return H % 8 == 0 && H <= vec::RT * vec::VG * 8; }

void rms_fwd_vec_launch(const float* X, int N, int H, const float* table, int64_t tld, int sh_off, int sc_off,
                        const int32_t* mod_id, const float* g, __nv_bfloat16* out, float* r, cudaStream_t s) {
    if (g)
        vec::rms_fwd_vec<1><<<row_chunks(N), vec::RT, 0, s>>>(X, N, H, table, tld, sh_off, sc_off, mod_id, g, out, r);
    else
        vec::rms_fwd_vec<0><<<row_chunks(N), vec::RT, 0, s>>>(X, N, H, table, tld, sh_off, sc_off, mod_id, g, out, r);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}
void postnorm_resid_vec_launch(const float* X1, const __nv_bfloat16* co, int N, int H, const float* g, float* X2,
                               float* rc, cudaStream_t s) {
    vec::postnorm_resid_vec<false><<<row_chunks(N), vec::RT, 0, s>>>(X1, co, N, H, g, X2, rc, nullptr, 0, 0, 0,
                                                                     nullptr, nullptr, nullptr);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}
void postnorm_resid_mod_vec_launch(const float* X1, const __nv_bfloat16* co, int N, int H, const float* g, float* X2,
                                   float* rc, const float* table, int64_t tld, int sh_off, int sc_off,
                                   const int32_t* mod_id, __nv_bfloat16* f, float* r2, cudaStream_t s) {
    vec::postnorm_resid_vec<true><<<row_chunks(N), vec::RT, 0, s>>>(X1, co, N, H, g, X2, rc, table, tld, sh_off, sc_off,
                                                                    mod_id, f, r2);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}
void gate_bwd_vec_launch(const float* dX, const __nv_bfloat16* y, const float* table, int64_t tld, int gate_off,
                         const int32_t* mod_id, int n_u, int N, int H, __nv_bfloat16* dY, float* part_dgate,
                         float* part_db, cudaStream_t s) {
    vec::gate_bwd_vec<<<row_chunks(N), vec::RT, 0, s>>>(dX, y, table, tld, gate_off, mod_id, n_u, N, H, dY, part_dgate,
                                                       part_db);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}
void rms_bwd_vec_launch(int mode, const __nv_bfloat16* dA, const float* X, const float* r, const float* table,
                        int64_t tld, int sc_off, const int32_t* mod_id, int n_u, const float* g, int N, int H, float* dX,
                        int accumulate, float* part_a, float* part_b, cudaStream_t s) {
    if (mode == 0)
        vec::rms_bwd_vec<0><<<row_chunks(N), vec::RT, 0, s>>>(dA, X, r, table, tld, sc_off, mod_id, n_u, g, N, H, dX,
                                                            accumulate, part_a, part_b);
    else
        vec::rms_bwd_vec<1><<<row_chunks(N), vec::RT, 0, s>>>(dA, X, r, table, tld, sc_off, mod_id, n_u, g, N, H, dX,
                                                            accumulate, part_a, part_b);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}
void postnorm_bwd_vec_launch(const float* dX, const __nv_bfloat16* co, const float* rc, const float* g, int N, int H,
                             __nv_bfloat16* dco, float* part_dg, cudaStream_t s) {
    vec::postnorm_bwd_vec<<<row_chunks(N), vec::RT, 0, s>>>(dX, co, rc, g, N, H, dco, part_dg);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}
void colsum_vec_launch(const __nv_bfloat16* Y, int64_t ld, int N, int C, float* part, cudaStream_t s) {
    dim3 grid(row_chunks(N), (C / 8 + vec::RT - 1) / vec::RT);
    vec::colsum_vec<<<grid, vec::RT, 0, s>>>(Y, ld, N, C, part);
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

}  // namespace mgv

namespace mgv {
// 16-byte vector path: head_dim % 8 == 0 (<= 256), 16-byte aligned bases, row strides / k offsets multiple of 8
bool qk_vec_ok(const void* a, const void* b, const QKLayout& L, int hd) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return hd % 8 == 0 && hd <= 256 && al(a) && al(b) && L.in_ld % 8 == 0 && L.in_koff % 8 == 0 && L.out_ld % 8 == 0 &&
           L.out_koff % 8 == 0;
}
}  // namespace mgv
