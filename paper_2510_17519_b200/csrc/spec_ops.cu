// The two SPEC-only operators of the DiT path that have no code in proj/ (SURVEY 8(b)):
//   fused_modulate(x, bias, scale, shift, residual)
//     out = residual + ((x + bias) * (1 + scale) + shift), one pass over x / residual, bit-exact against the
//     composed three-step reference evaluated in the same precision and order (no FMA contraction).
//   apply_rope3d(q_or_k, coords, split)              SPEC.md:168-176 = Tape::rope3d (autodiff.cpp:849-898)
//     per head, per axis slice (offset o, size d): pair (o+2i, o+2i+1) rotated by th = (pos * base^(-2i/d)) * dir.
//     The angle table is built on the host with the same libm calls the reference makes (std::pow, std::cos,
//     std::sin in rope_apply_vec, autodiff.cpp:856-858); the device applies a*c - b*s, a*s + b*c in fp64
//     with explicit round-to-nearest operations, so the output is bit-identical to the reference's.
#include <algorithm>
#include <array>
#include <cmath>
#include <string>
#include <vector>

#include "gemm.cuh"
#include "kernels.h"
#include "model.h"

namespace mgv {
namespace {

// n == 1: scalar, n == cols: per channel, otherwise full (rows x cols)
__device__ __forceinline__ double bcast(const double* p, int64_t n, int64_t cols, int64_t i) {
    return n == 1 ? p[0] : (n == cols ? p[i % cols] : p[i]);
}

__global__ void fused_modulate_f64_kernel(const double* x, const double* bias, int64_t nb, const double* scale,
                                          int64_t ns, const double* shift, int64_t nh, const double* res,
                                          int64_t n, int64_t cols, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double t = __dadd_rn(x[i], bcast(bias, nb, cols, i));                      // (i) bias
        const double m = __dadd_rn(__dmul_rn(t, __dadd_rn(1.0, bcast(scale, ns, cols, i))),  // (ii) modulation
                                   bcast(shift, nh, cols, i));
        out[i] = __dadd_rn(res[i], m);                                                      // (iii) residual
    }
}

// fp32 device form: per-channel bias / scale / shift (cols % 4 == 0), 16-byte accesses; one read of x and
// residual, one write of out (12 bytes per element of HBM traffic)
__global__ void fused_modulate_f32_kernel(const float4* x, const float* bias, const float* scale, const float* shift,
                                          const float4* res, int64_t n4, int64_t cols, float4* out) {
    const int64_t c4 = cols / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = (i % c4) * 4;
        const float4 xv = x[i], rv = res[i];
        const float4 b = *reinterpret_cast<const float4*>(bias + c);
        const float4 s = *reinterpret_cast<const float4*>(scale + c);
        const float4 h = *reinterpret_cast<const float4*>(shift + c);
        float4 o;
        o.x = __fadd_rn(rv.x, __fadd_rn(__fmul_rn(__fadd_rn(xv.x, b.x), __fadd_rn(1.0f, s.x)), h.x));
        o.y = __fadd_rn(rv.y, __fadd_rn(__fmul_rn(__fadd_rn(xv.y, b.y), __fadd_rn(1.0f, s.y)), h.y));
        o.z = __fadd_rn(rv.z, __fadd_rn(__fmul_rn(__fadd_rn(xv.z, b.z), __fadd_rn(1.0f, s.z)), h.z));
        o.w = __fadd_rn(rv.w, __fadd_rn(__fmul_rn(__fadd_rn(xv.w, b.w), __fadd_rn(1.0f, s.w)), h.w));
        out[i] = o;
    }
}

// one thread per (token, head, pair); tab holds (cos, sin) per (axis, pos - pos_min[axis], i)
struct RopeGeom {
    int split[3], off[3], pmin[3], span[3];
    int64_t tab_off[3];
    int hd, pairs;
};
__global__ void rope3d_f64_kernel(const double* x, int64_t N, int heads, const int32_t* coords, RopeGeom g,
                                  const double2* tab, double* out) {
    const int64_t total = N * heads * g.pairs;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int p = static_cast<int>(e % g.pairs);
        const int64_t th = e / g.pairs;  // token * heads + head
        const int64_t tok = th / heads;
        const int axis = p < g.split[0] / 2 ? 0 : (p < (g.split[0] + g.split[1]) / 2 ? 1 : 2);
        const int i = p - g.off[axis] / 2;
        const int pos = coords[tok * 3 + axis];
        const double2 cs = tab[g.tab_off[axis] + (int64_t)(pos - g.pmin[axis]) * (g.split[axis] / 2) + i];
        const int64_t j = th * g.hd + g.off[axis] + 2 * i;
        const double a = x[j], b = x[j + 1];
        out[j] = __dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(b, cs.y));  // autodiff.cpp:860-861
        out[j + 1] = __dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(b, cs.x));
    }
}

int grid_for(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }

}  // namespace

void fused_modulate_host(const double* x, const double* bias, int64_t nb, const double* scale, int64_t ns,
                         const double* shift, int64_t nh, const double* residual, int64_t rows, int64_t cols,
                         double* out, cudaStream_t s) {
    if (rows < 0 || cols < 1 || !x || !bias || !scale || !shift || !residual || !out)
        throw InputError("fused_modulate: bad arguments");
    const int64_t n = rows * cols;
    for (int64_t k : {nb, ns, nh})
        if (k != 1 && k != cols && k != n)
            throw DimensionError("fused_modulate: bias/scale/shift of " + std::to_string(k) +
                                 " elements do not broadcast to (" + std::to_string(rows) + ", " +
                                 std::to_string(cols) + ")");
    if (n == 0) return;
    double *d = nullptr;
    const int64_t tot = 3 * n + nb + ns + nh;
    MGV_CUDA(cudaMallocAsync(&d, sizeof(double) * tot, s));
    double *dx = d, *dr = dx + n, *db = dr + n, *dsc = db + nb, *dsh = dsc + ns, *dout = dsh + nh;
    MGV_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(dr, residual, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(db, bias, sizeof(double) * nb, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(dsc, scale, sizeof(double) * ns, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(dsh, shift, sizeof(double) * nh, cudaMemcpyHostToDevice, s));
    fused_modulate_f64_kernel<<<grid_for(n), 256, 0, s>>>(dx, db, nb, dsc, ns, dsh, nh, dr, n, cols, dout);
    note_launch();
    MGV_CUDA(cudaGetLastError());
    MGV_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    MGV_CUDA(cudaFreeAsync(d, s));
    MGV_CUDA(cudaStreamSynchronize(s));
}

void fused_modulate_dev_f32(const float* x, const float* bias, const float* scale, const float* shift,
                            const float* residual, int64_t rows, int64_t cols, float* out, cudaStream_t s) {
    if (rows < 0 || cols < 1 || cols % 4)
        throw DimensionError("fused_modulate (device fp32): cols must be a positive multiple of 4");
    const uintptr_t al = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(residual) |
                         reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(bias) |
                         reinterpret_cast<uintptr_t>(scale) | reinterpret_cast<uintptr_t>(shift);
    if (al % 16) throw InputError("fused_modulate (device fp32): pointers must be 16-byte aligned");
    const int64_t n4 = rows * cols / 4;
    if (n4 == 0) return;
    fused_modulate_f32_kernel<<<grid_for(n4), 256, 0, s>>>(reinterpret_cast<const float4*>(x), bias, scale, shift,
                                                            reinterpret_cast<const float4*>(residual), n4, cols,
                                                            reinterpret_cast<float4*>(out));
    note_launch();
    MGV_CUDA(cudaGetLastError());
}

void apply_rope3d_host(const double* x, int64_t N, int64_t heads, const int64_t split[3], const int32_t* coords,
                       double base, int inverse, double* out, cudaStream_t s) {
    if (N < 0 || heads < 1 || !split || (N > 0 && (!x || !coords || !out)))
        throw InputError("apply_rope3d: bad arguments");
    for (int a = 0; a < 3; ++a)
        if (split[a] < 0 || split[a] % 2)  // autodiff.cpp:874-876
            throw ConfigError("rope3d: slice sizes must be even, got (" + std::to_string(split[0]) + ", " +
                              std::to_string(split[1]) + ", " + std::to_string(split[2]) + ")");
    if (N == 0) return;
    RopeGeom g{};
    g.hd = static_cast<int>(split[0] + split[1] + split[2]);
    g.pairs = g.hd / 2;
    if (g.pairs == 0) {
        std::copy(x, x + N * heads * g.hd, out);
        return;
    }
    const double dir = inverse ? -1.0 : 1.0;
    std::vector<double2> tab;
    int off = 0;
    for (int a = 0; a < 3; ++a) {
        g.split[a] = static_cast<int>(split[a]);
        g.off[a] = off;
        off += g.split[a];
        int lo = 0, hi = 0;
        for (int64_t t = 0; t < N; ++t) {
            const int p = coords[t * 3 + a];
            if (t == 0 || p < lo) lo = p;
            if (t == 0 || p > hi) hi = p;
        }
        g.pmin[a] = lo;
        g.span[a] = hi - lo + 1;
        g.tab_off[a] = static_cast<int64_t>(tab.size());
        const int d = g.split[a], half = d / 2;
        // the reference's expressions, term for term (rope_apply_vec, autodiff.cpp:852-859)
        for (int p = lo; p <= hi; ++p)
            for (int i = 0; i < half; ++i) {
                const double freq = std::pow(base, -2.0 * static_cast<double>(i) / static_cast<double>(d));
                const double th = static_cast<double>(p) * freq * dir;
                tab.push_back(make_double2(std::cos(th), std::sin(th)));
            }
    }
    const int64_t n = N * heads * g.hd;
    double *dx = nullptr, *dout = nullptr;
    double2* dtab = nullptr;
    int32_t* dc = nullptr;
    MGV_CUDA(cudaMallocAsync(&dx, sizeof(double) * n, s));
    MGV_CUDA(cudaMallocAsync(&dout, sizeof(double) * n, s));
    MGV_CUDA(cudaMallocAsync(&dtab, sizeof(double2) * std::max<size_t>(tab.size(), 1), s));
    MGV_CUDA(cudaMallocAsync(&dc, sizeof(int32_t) * 3 * N, s));
    MGV_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(dtab, tab.data(), sizeof(double2) * tab.size(), cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(dc, coords, sizeof(int32_t) * 3 * N, cudaMemcpyHostToDevice, s));
    rope3d_f64_kernel<<<grid_for(N * heads * g.pairs), 256, 0, s>>>(dx, N, static_cast<int>(heads), dc, g, dtab, dout);
    note_launch();
    MGV_CUDA(cudaGetLastError());
    MGV_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    for (void* p : {static_cast<void*>(dx), static_cast<void*>(dout), static_cast<void*>(dtab), static_cast<void*>(dc)})
        MGV_CUDA(cudaFreeAsync(p, s));
    MGV_CUDA(cudaStreamSynchronize(s));
}

}  // namespace mgv
