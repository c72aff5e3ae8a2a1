// Launchers for the memory-bound kernels of the DiT block (everything that is
// not a GEMM or an attention).  T is the activation storage type:
// float (fp32 parity mode) or __nv_bfloat16 (performance mode).  Residual
// stream, norms, reductions and statistics are always fp32 (loss in fp64).
//
// Reductions over tokens (bias / gain / gate / temperature gradients) are
// deterministic: each CTA owns a fixed chunk of kRowsPerChunk rows and writes
// one partial row; reduce_chunks() sums the partials in chunk order.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mgv {

#ifndef MGV_ROWS_PER_CHUNK
#define MGV_ROWS_PER_CHUNK 64
#endif
// rows per CTA of the row kernels; also the chunking of every fixed-order column reduction (bias / gain / gate grads)
constexpr int kRowsPerChunk = MGV_ROWS_PER_CHUNK;
inline int row_chunks(int N) { return (N + kRowsPerChunk - 1) / kRowsPerChunk; }

// ---- K1: interpolate + unit-aligned condition mask (flowtrain.cpp:9-20, 83-100); cond = N device flags or null,
// cond_lat = N x D device condition latents (read only at conditioned rows) or null (= clean)
template <class T>
void prep_flow_sample(const double* clean, const double* noise, const uint8_t* cond, const double* cond_lat, int N,
                      int D, double t, T* rows, float* v_target, uint8_t* loss_mask, int32_t* mod_id, cudaStream_t s,
                      int id_t = 0, int id_0 = 1);
// rows (fp64, host layout) -> T, plus mod ids given on device
template <class T>
void convert_rows(const double* src, int64_t n, T* dst, cudaStream_t s);
template <class T>
void convert_f32(const float* src, int64_t n, T* dst, cudaStream_t s);

// ---- 2x2 patchify gather / scatter (dit.cpp:92-141), bit-exact index math
void latent_rows_gather(const double* grid, int U, int h, int w, int C, double* rows, int32_t* coords, cudaStream_t s);
// returns through *status: 0 ok, 1 coord out of range, 2 duplicate coord
void rows_to_grid_scatter(const double* rows, const int32_t* coords, int N, int U, int Hp, int Wp, int C, double* grid,
                          int32_t* seen, int32_t* status, cudaStream_t s);

// ---- RoPE table: per (token, rotation pair) cos/sin from int coords, fp64 math (autodiff.cpp:851-870)
void rope_table(const int32_t* coords, int N, int s0, int s1, int s2, float2* cs, cudaStream_t s);

// ---- global embedding + modulation table, fp64 (dit.cpp:27-34, 236-255, 280-283)
// taus (n_u) ; gmlp weights fp32 -> g (n_u x H) fp64; caches for backward
void global_embed(const double* taus, int n_u, double fps, const float* w_in, const float* b_in, const float* w_out,
                  const float* b_out, int H, double* phi /*(n_u+1) x 32*/, double* z_in /*(n_u+1) x H*/,
                  double* h_in /*(n_u+1) x H*/, double* g /*n_u x H*/, cudaStream_t s);
// gb = g * gscale (n_u x H, fp64) ; m = gb W_mod^T + b_mod -> table (n_u x 6H, fp32)
void modulation_table(const double* g, const float* gscale, const float* w_mod, const float* b_mod, int n_u, int H,
                      double* gb, float* table, cudaStream_t s);

// ---- forward row kernels
// out = rms(X) * (1 + table[u, sc_off:]) + table[u, sh_off:]   (dit.cpp:287, 308)
template <class T>
void rms_mod(const float* X, int N, int H, const float* table, int64_t tld, int sh_off, int sc_off,
             const int32_t* mod_id, T* out, float* r, cudaStream_t s);
// out = rms(X) * g   (dit.cpp:300, 314)
template <class T>
void rms_gain(const float* X, int N, int H, const float* g, T* out, float* r, cudaStream_t s);
// X2 = X1 + rms(co) * g   (dit.cpp:305)
template <class T>
void postnorm_resid(const float* X1, const T* co, int N, int H, const float* g, float* X2, float* rc, cudaStream_t s);
// postnorm_resid followed by rms_mod of X2 (dit.cpp:305 + :308) in one pass, bit-identical to the two kernels;
// false (nothing launched) where only the two-kernel path exists (fp32 mode, H % 8 != 0 or H > 4096)
template <class T>
bool postnorm_resid_mod(const float* X1, const T* co, int N, int H, const float* g, float* X2, float* rc,
                        const float* table, int64_t tld, int sh_off, int sc_off, const int32_t* mod_id, T* f, float* r2,
                        cudaStream_t s);
// Row strides of the q/k views the QK-norm kernels read and write (a tensor-parallel rank sees a
// column slice of the full buffers): q at column 0 and k at column *_koff of rows with stride *_ld;
// the inverse norms iq/ik at [n * i_ld + h].
struct QKLayout {
    int64_t in_ld, in_koff, out_ld, out_koff, i_ld;
};
inline QKLayout qk_layout_full(int64_t H, int heads) { return QKLayout{3 * H, H, 2 * H, H, heads}; }
// per head: q <- rope(temp_h * q / |q|), k <- rope(k / |k|)   (dit.cpp:289-294)
// qkv: raw projection; qk_out: rotated q | k; iq/ik inverse norms.  Hl = heads * hd (this view's width)
template <class T>
void qk_norm_rope(const T* qkv, const QKLayout& L, int N, int Hl, int heads, const float* temp, const float2* cs,
                  T* qk_out, float* iq, float* ik, cudaStream_t s);

// ---- flow loss (flowtrain.cpp:22-42, autodiff.cpp:466-491)
// part (row_chunks(N)) double partial sums of squared error over unmasked rows; dV = coef * (V - vt) on unmasked rows
template <class T>
void flow_loss_fwd(const float* V, const float* vt, const uint8_t* mask, int N, int D, double* part, cudaStream_t s);
// dV = base / (count * D) * (V - vt) on unmasked rows (0 everywhere when count == 0)
template <class T>
void flow_loss_bwd(const float* V, const float* vt, const uint8_t* mask, int N, int D, float base, const int* count,
                   T* dV, cudaStream_t s);
// acc[0] += sum(part[0..n)) / (count * D)   (0 when count == 0), one thread, fixed order
void flow_loss_accumulate(const double* part, int n, const int* count, int D, double* acc, cudaStream_t s);
void count_mask(const uint8_t* mask, int N, int* count, cudaStream_t s);
void sum_double(const double* part, int n, double* out, cudaStream_t s);  // fixed-order sum, one thread

// ---- backward row kernels (partials: [row_chunks(N)][...])
// dY = dX * gate[u] ; part_dgate[c][u][j] = sum dX*y ; part_db[c][j] = sum dY
template <class T>
void gate_bwd(const float* dX, const T* y, const float* table, int64_t tld, int gate_off, const int32_t* mod_id,
              int n_u, int N, int H, T* dY, float* part_dgate, float* part_db, cudaStream_t s);
// dX += rms_bwd(X, r, dA * (1 + sc[u])) ; part_dsh[c][u][j] = sum dA ; part_dsc[c][u][j] = sum dA * n
template <class T>
void rms_mod_bwd(const T* dA, const float* X, const float* r, const float* table, int64_t tld, int sh_off, int sc_off,
                 const int32_t* mod_id, int n_u, int N, int H, float* dX, float* part_dsh, float* part_dsc,
                 cudaStream_t s);
// dX (+)= rms_bwd(X, r, dA * g) ; part_dg[c][j] = sum dA * n
template <class T>
void rms_gain_bwd(const T* dA, const float* X, const float* r, const float* g, int N, int H, float* dX, int accumulate,
                  float* part_dg, cudaStream_t s);
// dco = rms_bwd(co, rc, dX * g) ; part_dg[c][j] = sum dX * n(co)
template <class T>
void postnorm_bwd(const float* dX, const T* co, const float* rc, const float* g, int N, int H, T* dco, float* part_dg,
                  cudaStream_t s);
// dqkv (same layout as qkv: L.in_ld / L.in_koff) holds d(rotated q | k) on entry, raw-projection grads on
// exit; part_dtemp[c][h]
template <class T>
void qk_norm_rope_bwd(T* dqkv, const T* qkv, const QKLayout& L, int N, int Hl, int heads, const float* temp,
                      const float2* cs, const float* iq, const float* ik, float* part_dtemp, cudaStream_t s);
// ---- tensor-parallel glue (partial sums arrive in fp32 after the all-reduce)
// y = part + bias ; Xout = Xin + y * gate[mod_id] ; y_out (T) kept for the gate gradient   (dit.cpp:297, 311)
template <class T>
void bias_gate_resid(const float* part, const float* bias, const float* table, int64_t tld, int gate_off,
                     const int32_t* mod_id, const float* Xin, float* Xout, T* y_out, int N, int H, cudaStream_t s);
// out = part + bias (bias may be null), as T
template <class T>
void bias_to(const float* part, const float* bias, T* out, int N, int H, cudaStream_t s);
// rank-major row permutation of chunked weights: dst row (vr, c, j) <- src row (c, vr, j)
// (C chunks of R rows, each split into P shards); inverse = 1 maps back
void permute_shard_rows(const float* src, float* dst, int C, int R, int P, int64_t cols, int inverse, cudaStream_t s);
void permute_shard_rows(const double* src, double* dst, int C, int R, int P, int64_t cols, int inverse, cudaStream_t s);
// column-parallel weights: (rows x cols) <-> P compact rank-major (rows x cols/P) blocks
void permute_shard_cols(const float* src, float* dst, int64_t rows, int64_t cols, int P, int inverse, cudaStream_t s);
void permute_shard_cols(const double* src, double* dst, int64_t rows, int64_t cols, int P, int inverse,
                        cudaStream_t s);
// part[c][j] = sum over chunk rows of Y[i, j]   (bias gradients)
template <class T>
void colsum(const T* Y, int64_t ld, int N, int C, float* part, cudaStream_t s);
// out[j] (+)= alpha * sum_c part[c][j]   in chunk order
void reduce_chunks(const float* part, int chunks, int C, float* out, float alpha, int accumulate, cudaStream_t s);
// grouped: part[c][g][j] (j < C) -> out[g*out_stride + j]
void reduce_chunks_grouped(const float* part, int chunks, int groups, int C, float* out, int64_t out_stride,
                           float alpha, int accumulate, cudaStream_t s);

// ---- modulation / global-embedding backward (fp64 where the forward is fp64)
// dm (n_u x 6H fp32) -> dW_mod += dm^T gb ; db_mod += sum_u dm ; dgb = dm W_mod (n_u x H fp64)
void modulation_bwd(const float* dm, const double* gb, const float* w_mod, int n_u, int H, float* dw_mod,
                    float* db_mod, double* dgb, cudaStream_t s);
// dgscale += sum_u dgb*g ; dg += dgb * gscale
void gscale_bwd(const double* dgb, const double* g, const float* gscale, int n_u, int H, float* dgscale, double* dg,
                cudaStream_t s);
// MLP backward for the n_u timestep rows and the fps row (dg_f = sum_u dg_u)
void global_embed_bwd(const double* dg, int n_u, const double* phi, const double* z_in, const double* h_in,
                      const float* w_out, int H, float* dw_in, float* db_in, float* dw_out, float* db_out,
                      cudaStream_t s);
// sum of squares of a fp32 buffer into out (double), fixed order
void sumsq(const float* x, int64_t n, double* part /*>= 1024*/, double* out, cudaStream_t s);
void fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t s);
void fill_f32(float* p, int64_t n, float v, cudaStream_t s);
// out[c * ld_out + r] = in[r * ld_in + c] for r < rows, c < cols (bf16; attention operand transposes)
void transpose_bf16(const __nv_bfloat16* in, int64_t ld_in, int rows, int cols, __nv_bfloat16* out, int64_t ld_out,
                    cudaStream_t s);

// SPEC-only operators (spec_ops.cu): fused_modulate on host fp64 buffers (bias / scale / shift
// of 1, cols or rows*cols elements) and on device fp32 buffers (per-channel vectors); apply_rope3d
// (SPEC.md:168-176 = Tape::rope3d, autodiff.cpp:849-898) on host fp64 buffers, inverse != 0 rotates by -theta
void fused_modulate_host(const double* x, const double* bias, int64_t nb, const double* scale, int64_t ns,
                         const double* shift, int64_t nh, const double* residual, int64_t rows, int64_t cols,
                         double* out, cudaStream_t s);
void fused_modulate_dev_f32(const float* x, const float* bias, const float* scale, const float* shift,
                            const float* residual, int64_t rows, int64_t cols, float* out, cudaStream_t s);
void apply_rope3d_host(const double* x, int64_t N, int64_t heads, const int64_t split[3], const int32_t* coords,
                       double base, int inverse, double* out, cudaStream_t s);

}  // namespace mgv
