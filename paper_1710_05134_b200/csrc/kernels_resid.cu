// kernels_resid.cu — front-local bound of the factor residual (SURVEY.md §8(c)
// item 13; the P8 pin "residual <= 1e-10" of BASELINE north_star at sizes where
// the dense residual cannot be formed).
//
// Multifrontal identity: with F_s the assembled front of s (original entries of
// its pivot columns plus the children's trailing blocks T_c, extend-added), its
// eliminated columns L_s, D_s and its own trailing block T_s (what the parent
// extend-adds: delayed columns + contribution block), the front residual
//     E_s = P_s F_s P_s^T - L_s D_s L_s^T - (0 (+) T_s)
// telescopes over the tree: sum_s scatter(E_s) = P (A - sigma B) P^T - L D L^T,
// because every T_c enters exactly one parent.  Hence
//     || P (A - sigma B) P^T - L D L^T ||_F  <=  sum_s || E_s ||_F.
// Everything here is read-only diagnostics run by kep_factor_residual: F_s is
// captured right after the level's assembly (k_capture), and E_s is evaluated
// after the level's Schur update from the factor store (L, D exactly as the
// solves use them), the pivot permutation and the trailing block in the arena
// (read exactly as the parent's extend-add reads it, kernels.cu).
#include <cstdint>

#include "device.cuh"

namespace kep {

namespace {

constexpr int RT = 256;      // threads: 16 x 16, 4 x 4 outputs each
constexpr int RB = 64;       // output tile
constexpr int RK = 16;       // K chunk

__global__ void __launch_bounds__(256) k_capture(DevPlan P, const int32_t* __restrict__ fronts, double* __restrict__ F0) {
    const int s = fronts[blockIdx.x];
    const int nd = P.nd_in[s];
    if (nd < 0) return;
    const int f = P.forder[s] + nd, ld = ldpad(P.cap[s]);
    const double* src = P.arena + P.arena_off[s];
    double* dst = F0 + P.arena_off[s];
    for (int j = blockIdx.y; j < f; j += gridDim.y)
        for (int i = j + threadIdx.x; i < f; i += blockDim.x) dst[i + (size_t)j * ld] = src[i + (size_t)j * ld];
}

// L[i, t] of the stored panel (unit lower; 0 at the in-pair entry of a 2x2 block)
__device__ __forceinline__ double lval(const double* L, int f, int i, int t) {
    return i == t ? 1.0 : (i > t ? L[(size_t)t * f + i] : 0.0);
}

__global__ void __launch_bounds__(RT) k_resid(DevPlan P, StorePlan T, const int4* __restrict__ items,
                                              const double* __restrict__ F0, double* __restrict__ out) {
    __shared__ double As[RK][RB + 1];
    __shared__ double Ws[RK][RB + 1];
    __shared__ double red[RT / 32];
    const int4 it = items[blockIdx.x];
    const int s = it.x, I = it.y, J = it.z;
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y, q = h.z, flag = h.w;
    const int i0 = RB * I, j0 = RB * J;
    if (i0 >= f) return;
    const double* L = T.panel + T.poff[s];
    const int64_t qo = T.qoff[s];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    const int kend = min(e, j0 + RB + 1);              // W[j, t] = 0 for t > j + 1 (2x2 pair straddling)
    for (int t0 = 0; t0 < kend; t0 += RK) {
        for (int x = tid; x < RK * RB; x += RT) {
            const int tt = x / RB, r = x % RB, t = t0 + tt;
            double a = 0.0, w = 0.0;
            if (t < kend) {
                const int i = i0 + r, j = j0 + r;
                if (i < f) a = lval(L, f, i, t);
                if (j < f) {
                    const int kd = T.kind[qo + t];
                    if (kd == PK_1X1) w = lval(L, f, j, t) * T.d[qo + t];
                    else if (kd == PK_2X2A) w = lval(L, f, j, t) * T.d[qo + t] + lval(L, f, j, t + 1) * T.ds[qo + t];
                    else if (kd == PK_2X2B) w = lval(L, f, j, t - 1) * T.ds[qo + t - 1] + lval(L, f, j, t) * T.d[qo + t];
                }
            }
            As[tt][r] = a;
            Ws[tt][r] = w;
        }
        __syncthreads();
#pragma unroll
        for (int tt = 0; tt < RK; ++tt) {
            double a[4], w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { a[u] = As[tt][ty * 4 + u]; w[u] = Ws[tt][tx * 4 + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], w[v], acc[u][v]);
        }
        __syncthreads();
    }
    const int c = P.ncb[s];
    const AuxRec A = aux_rec(P, 0, s, P.cap[s] - c);
    const int ld = ldpad(P.cap[s]);
    const double* F = P.arena + P.arena_off[s];
    const double* G = F0 + P.arena_off[s];
    const int ndo = q - e;
    const bool wup = flag == FL_OK && ndo > 0;
    double sum = 0.0, sreg[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int i = i0 + ty * 4 + u, j = j0 + tx * 4 + v;
            if (i >= f || j >= f || i < j) continue;
            const int pi = i < q ? A.perm[i] : i, pj = j < q ? A.perm[j] : j;
            const double f0 = pi >= pj ? G[pi + (size_t)pj * ld] : G[pj + (size_t)pi * ld];
            double tv = 0.0;
            if (i >= e && j >= e) {
                const int x = i - e, y = j - e;
                tv = (wup && y < ndo && x >= ndo) ? F[(e + y) + (size_t)(e + x) * ld] : F[i + (size_t)j * ld];
            }
            const double r = f0 - acc[u][v] - tv;
            const double w = (i == j ? 1.0 : 2.0) * r * r;
            sum += w;
            sreg[j >= e ? 2 : (i < q ? 0 : 1)] += w;
        }
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((tid & 31) == 0) red[tid >> 5] = sum;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < RT / 32; ++w) t += red[w];
        atomicAdd(&out[(size_t)4 * s], t);
    }
#pragma unroll
    for (int x = 0; x < 3; ++x) {                        // diagnostics: FS x eliminated, CB x eliminated, trailing
        double v = sreg[x];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((tid & 31) == 0 && v != 0.0) atomicAdd(&out[(size_t)4 * s + 1 + x], v);
    }
}

}  // namespace

int resid_tile() { return RB; }

void launch_capture(const DevPlan& P, const int32_t* fronts, int nfronts, double* F0, cudaStream_t st) {
    if (nfronts <= 0) return;
    k_capture<<<dim3(nfronts, 32), 256, 0, st>>>(P, fronts, F0);
}

void launch_resid(const DevPlan& P, const StorePlan& T, const int4* items, int nitems, const double* F0, double* out,
                  cudaStream_t st) {
    if (nitems <= 0) return;
    k_resid<<<nitems, RT, 0, st>>>(P, T, items, F0, out);
}

}  // namespace kep
