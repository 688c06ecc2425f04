// kth.cu — SURVEY.md §8(f) rows f2 and f3: the three-stage k-th eigenpair
// driver (Alg. 4) around the nu_sigma engine.
//
//   stage 1  Alg. 2: generalized Lanczos, Eq. (2.1)
//            A V_j = B V_j T_j + B v_{j+1} beta_j e_j^T, B-orthonormal V_j,
//            one fused A/B SpMV and one B-solve per step; Ritz values
//            theta_1^(j) / theta_j^(j) as shifts until two consecutive shifts
//            bracket lambda_k.
//   stage 2  Alg. 1' generalised to P shifts per round
//            (multisection, R12) until nu_u - nu_l <= m_max.
//   stage 3  Alg. 3: SI Lanczos at the interval midpoint on
//            the companions w = B^-1 v~ (B-orthonormal), one solve with the
//            retained factor and one B-product per step, x_{i,2} (Eq. 2.7)
//            without extra solves, error bounds Eq. (3.1), tests (3.3)-(3.5).
//
// Device kernels: fused SpMV y_A = A x, y_B = B x over one full symmetric CSR
// index array (20 B per stored nonzero: int32 column + two fp64 values), dot
// products, the skinny GEMVs of the reorthogonalisation and the Ritz-vector
// assembly.  The tridiagonal eigenproblems (j <= a few hundred) run on the
// host (symmetric QL with implicit shifts).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "device.cuh"

namespace kep {

namespace {

constexpr int VT = 256;
constexpr int kRitzMax = 32;     // Ritz vectors assembled per pass (m_max <= 32)

// y_a = A x, y_b = B x; one warp per row of the full symmetric CSR
__global__ void __launch_bounds__(VT) k_spmv2(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                              const double* __restrict__ va, const double* __restrict__ vb,
                                              const double* __restrict__ x, double* __restrict__ ya,
                                              double* __restrict__ yb, int64_t n) {
    const int64_t row = (int64_t)blockIdx.x * (VT / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    double sa = 0.0, sb = 0.0;
    for (int64_t q = rp[row] + lane; q < rp[row + 1]; q += 32) {
        const double xv = x[ci[q]];
        sa = fma(va[q], xv, sa);
        sb = fma(vb[q], xv, sb);
    }
    for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
        if (ya) ya[row] = sa;
        if (yb) yb[row] = sb;
    }
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[VT / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
#pragma unroll
    for (int q = 0; q < VT / 32; ++q) r += red[q];
    return r;
}

// out[t] += sum_i V[i + t ldv] r[i], t < j   (grid.y = t)
__global__ void __launch_bounds__(VT) k_gemv_t(const double* __restrict__ V, int64_t ldv, const double* __restrict__ r,
                                               int64_t n, double* __restrict__ out) {
    const int t = blockIdx.y;
    const double* v = V + (size_t)t * ldv;
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * VT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VT) s = fma(v[i], r[i], s);
    s = block_sum(s);
    if (threadIdx.x == 0) atomicAdd(&out[t], s);
}

// y[i] = beta_y * y[i] + sum_t V[i + t ldv] c[t] + a1 * x1[i] + a2 * x2[i]
__global__ void __launch_bounds__(VT) k_combine(const double* __restrict__ V, int64_t ldv, int j,
                                                const double* __restrict__ c, double cv, double beta_y, double* __restrict__ y,
                                                double a1, const double* __restrict__ x1, double a2,
                                                const double* __restrict__ x2, int64_t n) {
    extern __shared__ double cs[];
    for (int t = threadIdx.x; t < j; t += VT) cs[t] = cv * c[t];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * VT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VT) {
        double s = beta_y == 0.0 ? 0.0 : beta_y * y[i];
        for (int t = 0; t < j; ++t) s = fma(V[i + (size_t)t * ldv], cs[t], s);
        if (x1) s = fma(a1, x1[i], s);
        if (x2) s = fma(a2, x2[i], s);
        y[i] = s;
    }
}

// X[:, q] = sum_t W[:, t] C[t + q j] + r * g[q]   (Ritz vectors x_{i,2}, m columns)
__global__ void __launch_bounds__(VT) k_ritz(const double* __restrict__ W, int64_t ldw, int j, const double* __restrict__ C,
                                             const double* __restrict__ r, const double* __restrict__ g, int m,
                                             double* __restrict__ X, int64_t ldx, int64_t n) {
    extern __shared__ double cs[];            // j * m + m
    for (int t = threadIdx.x; t < j * m; t += VT) cs[t] = C[t];
    for (int q = threadIdx.x; q < m; q += VT) cs[j * m + q] = g[q];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * VT + threadIdx.x; i < n; i += (int64_t)gridDim.x * VT) {
        const double ri = r[i];
        double acc[kRitzMax];
#pragma unroll
        for (int q = 0; q < kRitzMax; ++q) acc[q] = q < m ? ri * cs[j * m + q] : 0.0;
        for (int t = 0; t < j; ++t) {                 // W read once per row
            const double w = W[i + (size_t)t * ldw];
#pragma unroll
            for (int q = 0; q < kRitzMax; ++q)
                if (q < m) acc[q] = fma(w, cs[t + q * j], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < kRitzMax; ++q)
            if (q < m) X[i + (size_t)q * ldx] = acc[q];
    }
}

int grid_for(int64_t n) { return (int)std::min<int64_t>((n + VT - 1) / VT, 148 * 8); }

}  // namespace

void launch_spmv2(const int64_t* rp, const int32_t* ci, const double* va, const double* vb, const double* x, double* ya,
                  double* yb, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_spmv2<<<(unsigned)((n + VT / 32 - 1) / (VT / 32)), VT, 0, st>>>(rp, ci, va, vb, x, ya, yb, n);
}

// out[0..j) = V^T r  (out is overwritten)
void launch_gemv_t(const double* V, int64_t ldv, int j, const double* r, int64_t n, double* out, cudaStream_t st) {
    if (j <= 0) return;
    cudaMemsetAsync(out, 0, sizeof(double) * j, st);
    const int gx = std::min(grid_for(n), 148);
    k_gemv_t<<<dim3(gx, j), VT, 0, st>>>(V, ldv, r, n, out);
}

void launch_combine(const double* V, int64_t ldv, int j, const double* c, double cv, double beta_y, double* y,
                    double a1, const double* x1, double a2, const double* x2, int64_t n, cudaStream_t st) {
    k_combine<<<grid_for(n), VT, sizeof(double) * std::max(j, 1), st>>>(V, ldv, j, c, cv, beta_y, y, a1, x1, a2, x2, n);
}

void launch_ritz(const double* W, int64_t ldw, int j, const double* C, const double* r, const double* g, int m,
                 double* X, int64_t ldx, int64_t n, cudaStream_t st) {
    const size_t smem = sizeof(double) * ((size_t)j * m + m);
    static unsigned long long attr = 0;
    if (first_on_device(attr)) { cudaFuncSetAttribute(k_ritz, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);  }
    k_ritz<<<grid_for(n), VT, smem, st>>>(W, ldw, j, C, r, g, m, X, ldx, n);
}

}  // namespace kep
