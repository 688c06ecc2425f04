// kernels_solve.cu — SURVEY.md §8(f) row f1: retained factors and the
// supernodal (multifrontal) triangular solves with them.
//
// kep_factor keeps, per front s, the panel of its eliminated columns
// (f_s x e_s, column-major, ld = f_s; unit lower L, zero at the in-pair entry
// of a 2x2 block), the labels of its rows (elimination positions of the
// variables: FS positions after pivoting, then the CB rows), the local pivot
// permutation and D.  With S = P Q (A - sigma B) Q^T P^T = L D L^T (Alg. 1'
// line 3), a solve S y = b is
//   forward  (postorder levels): the front vector is b on the front's own
//            pivots plus its children's update vectors, extend-added in child
//            order (the vector analogue of the assembly: deterministic, no
//            atomics); y_e = L11^-1 y_e, the delayed and CB rows get -L21 y_e
//            and become this front's update vector; z_e = D^-1 y_e;
//   backward (reverse levels):   x_e = L11^-T (z_e - L21^T x_rest).
// Fronts larger than shared memory allows keep their vector in global scratch.
// These are the shift-and-invert solves of stage 3 (Alg. 3)
// and of the stage-1 B-solves.
#include <algorithm>
#include <cstdint>

#include "device.cuh"

namespace kep {

namespace {

constexpr int ST_T = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double r = 0.0;
#pragma unroll
    for (int q = 0; q < ST_T / 32; ++q) r += red[q];
    return r;
}

// Copy the factor panel of each front of a level (shift 0 of the batch) into
// the factor store.  Fast-path fronts keep G = L21 Q |Lambda|^1/2 in the upper part
// (k_l21); unblocked fronts keep L in the lower part in position order.
__global__ void __launch_bounds__(ST_T) k_store(DevPlan P, StorePlan T, const int32_t* __restrict__ fronts) {
    const int s = fronts[blockIdx.x];
    const int nd = P.nd_in[s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ldf = ldpad(P.cap[s]), ld = f;     // ldf: front, ld: stored panel
    const int e = q - P.nd_out[s];
    const int flag = P.flag[s];
    const double* F = P.arena + P.arena_off[s];
    const AuxRec A = aux_rec(P, 0, s, P.cap[s] - c);
    double* panel = T.panel + T.poff[s];
    int* lab = T.lab + T.loff[s];
    const int64_t qo = T.qoff[s];
    if (threadIdx.x == 0) T.hdr[s] = make_int4(e, f, q, flag);
    for (int i = threadIdx.x; i < f; i += ST_T)
        lab[i] = i < q ? A.label[A.perm[i]] : P.cb_rows[P.cb_ptr[s] + (i - q)];
    for (int i = threadIdx.x; i < q; i += ST_T) T.perm[qo + i] = A.perm[i];
    for (int t = threadIdx.x; t < e; t += ST_T) {
        T.d[qo + t] = A.d[t];
        T.ds[qo + t] = A.ds[t];
        T.kind[qo + t] = A.kind[t];
    }
    for (int t = 0; t < e; ++t) {
        const int kd = A.kind[t];
        // fast path, CB rows: L21 = G M^-1 (G = L21 Q |Lambda|^1/2 in the upper part, k_l21)
        double ca = 0.0, cb = 0.0;
        int o = 0;
        if (kd == PK_1X1) ca = 1.0 / sqrt(fabs(A.d[t]));
        else if (kd == PK_2X2A || kd == PK_2X2B) {
            const int a = kd == PK_2X2A ? t : t - 1;
            double cs, sn, l1, l2;
            pair_eig(A.d[a], A.ds[a], A.d[a + 1], cs, sn, l1, l2);
            const double r1 = 1.0 / sqrt(fabs(l1)), r2 = 1.0 / sqrt(fabs(l2));
            if (kd == PK_2X2A) { ca = cs * r1; cb = -sn * r2; o = 1; }    // L_t = cs G_t/r1' - sn G_t+1/r2'
            else { ca = cs * r2; cb = sn * r1; o = -1; }                  // L_t+1 = sn G_t/r1' + cs G_t+1/r2'
        }
        double* col = panel + (size_t)t * ld;
        for (int i = threadIdx.x; i < f; i += ST_T) {
            double v = 0.0;
            if (i > t && !(kd == PK_2X2A && i == t + 1)) {
                if (flag == FL_REF) v = F[i + (size_t)t * ldf];
                else if (i < q) {      // fast path FS rows hold G11 = L11 M (k_fsp): B' = G11 S, L11 = B' (D M^-T)^-1
                    const double bt = F[i + (size_t)t * ldf] * A.sgn[t];
                    if (kd == PK_2X2A) v = bt * A.gca[t] + F[i + (size_t)(t + 1) * ldf] * A.sgn[t + 1] * A.gcb[t + 1];
                    else if (kd == PK_2X2B) v = bt * A.gca[t] + F[i + (size_t)(t - 1) * ldf] * A.sgn[t - 1] * A.gcb[t - 1];
                    else v = bt * A.gca[t];
                } else v = F[t + (size_t)i * ldf] * ca + (o ? F[(t + o) + (size_t)i * ldf] * cb : 0.0);
            }
            if (kd == PK_ZERO) v = 0.0;
            col[i] = v;
        }
    }
}

// forward elimination and D^-1 for the fronts of one level; x in elimination positions (b on
// entry for every variable, z = D^-1 L^-1 P b for the eliminated ones on exit)
__global__ void __launch_bounds__(ST_T) k_fwd(DevPlan P, StorePlan T, const int32_t* __restrict__ fronts,
                                              double* __restrict__ x) {
    extern __shared__ double ysm[];
    const int s = fronts[blockIdx.x];
    if (T.yoff[s] >= 0) return;                                          // large front: the blocked kernels
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y, q = h.z;
    const int p = P.npiv[s], nd = q - p;
    const double* L = T.panel + T.poff[s];
    const int* lab = T.lab + T.loff[s];
    const int64_t qo = T.qoff[s];
    double* yo = ysm;                                                    // front vector, original local order
    double* y = yo + f;                                                  // pivoted order
    for (int i = threadIdx.x; i < f; i += ST_T) yo[i] = i < p ? x[P.piv_first[s] + i] : 0.0;
    __syncthreads();
    // extend-add of the children's update vectors (children in order; rows of one child are distinct)
    int dof = 0;
    for (int k = P.child_ptr[s]; k < P.child_ptr[s + 1]; ++k) {
        const int c = P.child_list[k];
        const int4 hc = T.hdr[c];
        const int ndo = hc.z - hc.x, mc = hc.y - hc.x;
        const double* uc = T.upd + T.loff[c];
        const int32_t* rm = P.rmap + P.rmap_ptr[c];
        for (int xx = threadIdx.x; xx < mc; xx += ST_T) {
            int pos;
            if (xx < ndo) pos = p + dof + xx;
            else { const int r = rm[xx - ndo]; pos = r < p ? r : r + nd; }
            yo[pos] += uc[xx];
        }
        dof += ndo;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < f; i += ST_T) y[i] = i < q ? yo[T.perm[qo + i]] : yo[i];
    __syncthreads();
    for (int t = 0; t < e; ++t) {
        const double yt = y[t];
        const double* col = L + (size_t)t * f;
        for (int i = t + 1 + threadIdx.x; i < f; i += ST_T) y[i] = fma(-col[i], yt, y[i]);
        __syncthreads();
    }
    for (int t = threadIdx.x; t < e; t += ST_T) {
        const int kd = T.kind[qo + t];
        double z = 0.0;
        if (kd == PK_1X1) z = y[t] / T.d[qo + t];
        else if (kd == PK_2X2A || kd == PK_2X2B) {
            const int a = kd == PK_2X2A ? t : t - 1;
            const double d11 = T.d[qo + a], d21 = T.ds[qo + a], d22 = T.d[qo + a + 1];
            const double det = d11 * d22 - d21 * d21;
            z = kd == PK_2X2A ? (d22 * y[a] - d21 * y[a + 1]) / det : (d11 * y[a + 1] - d21 * y[a]) / det;
        }
        x[lab[t]] = z;
    }
    double* us = T.upd + T.loff[s];                                      // update vector: rows e..f
    for (int i = e + threadIdx.x; i < f; i += ST_T) us[i - e] = y[i];
}

// back substitution for the fronts of one level (levels top-down)
__global__ void __launch_bounds__(ST_T) k_bwd(StorePlan T, const int32_t* __restrict__ fronts, double* __restrict__ x) {
    extern __shared__ double xsm[];
    __shared__ double red[ST_T / 32];
    const int s = fronts[blockIdx.x];
    if (T.yoff[s] >= 0) return;                                          // large front: the blocked kernels
    double* xs = xsm;
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y;
    const double* L = T.panel + T.poff[s];
    const int* lab = T.lab + T.loff[s];
    for (int i = threadIdx.x; i < f; i += ST_T) xs[i] = x[lab[i]];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = warp; t < e; t += ST_T / 32) {            // z_t - L21[:, t] . x_rest
        const double* col = L + (size_t)t * f;
        double a = 0.0;
        for (int i = e + lane; i < f; i += 32) a = fma(col[i], xs[i], a);
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) xs[t] -= a;
    }
    __syncthreads();
    for (int t = e - 1; t >= 0; --t) {                      // L11^-T
        const double* col = L + (size_t)t * f;
        double a = 0.0;
        for (int i = t + 1 + threadIdx.x; i < e; i += ST_T) a = fma(col[i], xs[i], a);
        a = block_sum(a, red);
        if (threadIdx.x == 0) xs[t] -= a;
        __syncthreads();
    }
    for (int t = threadIdx.x; t < e; t += ST_T) x[lab[t]] = xs[t];
}

// ---------------------------------------------------------------- large fronts: blocked solves
// A front of order f > solve_big_front() solves with all SMs: its vectors live in global scratch
// (ybuf at yoff: original order [0, f), pivoted order [f, 2f)); the unit lower L11 is processed in
// 64-column blocks -- the 64 x 64 diagonal block by one CTA, the rows below by a grid of CTAs
// (forward), or the block's columns against the rows below by one CTA per column (backward, fixed
// reduction order: deterministic).
constexpr int SBK = 64;

// forward: extend-add of the children's update vectors into the front vector, then pivot order
__global__ void __launch_bounds__(ST_T) k_fwdb_prep(DevPlan P, StorePlan T, const int32_t* __restrict__ fronts,
                                                    const double* __restrict__ x) {
    const int s = fronts[blockIdx.x];
    const int4 h = T.hdr[s];
    const int f = h.y, q = h.z;
    const int p = P.npiv[s], nd = q - p;
    const int64_t qo = T.qoff[s];
    double* yo = T.ybuf + T.yoff[s];
    double* y = yo + f;
    for (int i = threadIdx.x; i < f; i += ST_T) yo[i] = i < p ? x[P.piv_first[s] + i] : 0.0;
    __syncthreads();
    int dof = 0;
    for (int k = P.child_ptr[s]; k < P.child_ptr[s + 1]; ++k) {
        const int c = P.child_list[k];
        const int4 hc = T.hdr[c];
        const int ndo = hc.z - hc.x, mc = hc.y - hc.x;
        const double* uc = T.upd + T.loff[c];
        const int32_t* rm = P.rmap + P.rmap_ptr[c];
        for (int xx = threadIdx.x; xx < mc; xx += ST_T) {
            int pos;
            if (xx < ndo) pos = p + dof + xx;
            else { const int r = rm[xx - ndo]; pos = r < p ? r : r + nd; }
            yo[pos] += uc[xx];
        }
        dof += ndo;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < f; i += ST_T) y[i] = i < q ? yo[T.perm[qo + i]] : yo[i];
}

// forward, block b: y_b = L_bb^-1 y_b (one warp, the block's L in shared memory)
__global__ void __launch_bounds__(32) k_fwdb_diag(StorePlan T, const int32_t* __restrict__ fronts, int b) {
    __shared__ double Lb[SBK][SBK + 1];
    const int s = fronts[blockIdx.x];
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y;
    const int t0 = b * SBK;
    if (t0 >= e) return;
    const int nb = min(SBK, e - t0);
    const double* L = T.panel + T.poff[s];
    double* y = T.ybuf + T.yoff[s] + f;
    for (int t = 0; t < nb; ++t)
        for (int i = threadIdx.x; i < nb; i += 32) Lb[i][t] = L[(size_t)(t0 + t) * f + t0 + i];
    __syncwarp();
    double v0 = threadIdx.x < nb ? y[t0 + threadIdx.x] : 0.0;
    double v1 = threadIdx.x + 32 < nb ? y[t0 + 32 + threadIdx.x] : 0.0;
    for (int t = 0; t < nb; ++t) {
        const double yt = __shfl_sync(0xffffffffu, t < 32 ? v0 : v1, t & 31);
        const int i0 = threadIdx.x, i1 = threadIdx.x + 32;
        if (i0 > t && i0 < nb) v0 = fma(-Lb[i0][t], yt, v0);
        if (i1 > t && i1 < nb) v1 = fma(-Lb[i1][t], yt, v1);
    }
    if (threadIdx.x < nb) y[t0 + threadIdx.x] = v0;
    if (threadIdx.x + 32 < nb) y[t0 + 32 + threadIdx.x] = v1;
}

// forward, block b: rows below the block, y[i] -= L[i, block] y_block (grid: front x row chunks)
__global__ void __launch_bounds__(ST_T) k_fwdb_panel(StorePlan T, const int32_t* __restrict__ fronts, int b) {
    __shared__ double yb[SBK];
    const int s = fronts[blockIdx.y];
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y;
    const int t0 = b * SBK;
    if (t0 >= e) return;
    const int nb = min(SBK, e - t0);
    const int i = t0 + nb + blockIdx.x * ST_T + threadIdx.x;
    if (t0 + nb + blockIdx.x * ST_T >= f) return;
    const double* L = T.panel + T.poff[s];
    double* y = T.ybuf + T.yoff[s] + f;
    if (threadIdx.x < nb) yb[threadIdx.x] = y[t0 + threadIdx.x];
    __syncthreads();
    if (i >= f) return;
    double acc = 0.0;
    for (int t = 0; t < nb; ++t) acc = fma(L[(size_t)(t0 + t) * f + i], yb[t], acc);
    y[i] -= acc;
}

// forward: D^-1, the eliminated variables' values, the update vector
__global__ void __launch_bounds__(ST_T) k_fwdb_fin(StorePlan T, const int32_t* __restrict__ fronts, double* __restrict__ x) {
    const int s = fronts[blockIdx.x];
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y;
    const int* lab = T.lab + T.loff[s];
    const int64_t qo = T.qoff[s];
    const double* y = T.ybuf + T.yoff[s] + f;
    for (int t = threadIdx.x; t < e; t += ST_T) {
        const int kd = T.kind[qo + t];
        double z = 0.0;
        if (kd == PK_1X1) z = y[t] / T.d[qo + t];
        else if (kd == PK_2X2A || kd == PK_2X2B) {
            const int a = kd == PK_2X2A ? t : t - 1;
            const double d11 = T.d[qo + a], d21 = T.ds[qo + a], d22 = T.d[qo + a + 1];
            const double det = d11 * d22 - d21 * d21;
            z = kd == PK_2X2A ? (d22 * y[a] - d21 * y[a + 1]) / det : (d11 * y[a + 1] - d21 * y[a]) / det;
        }
        x[lab[t]] = z;
    }
    double* us = T.upd + T.loff[s];
    for (int i = e + threadIdx.x; i < f; i += ST_T) us[i - e] = y[i];
}

// backward: gather x over the front's rows
__global__ void __launch_bounds__(ST_T) k_bwdb_prep(StorePlan T, const int32_t* __restrict__ fronts,
                                                    const double* __restrict__ x) {
    const int s = fronts[blockIdx.x];
    const int f = T.hdr[s].y;
    const int* lab = T.lab + T.loff[s];
    double* xs = T.ybuf + T.yoff[s];
    for (int i = threadIdx.x; i < f; i += ST_T) xs[i] = x[lab[i]];
}

// backward: x[t] -= sum_{i in [r0, r1)} L[i, t] x[i] for the columns t of [c0, c1) (one CTA per column,
// grid: front x column): rows [r0, r1) = [e, f) (the L21 part) or the L11 rows below a block
__global__ void __launch_bounds__(ST_T) k_bwdb_cols(StorePlan T, const int32_t* __restrict__ fronts, int b, int l21) {
    __shared__ double red[ST_T / 32];
    const int s = fronts[blockIdx.y];
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y;
    int t, r0, r1;
    if (l21) { t = blockIdx.x; r0 = e; r1 = f; if (t >= e) return; }
    else {
        const int t0 = b * SBK;
        if (t0 >= e) return;
        const int nb = min(SBK, e - t0);
        if ((int)blockIdx.x >= nb) return;
        t = t0 + blockIdx.x; r0 = t0 + nb; r1 = e;
    }
    if (r0 >= r1) return;
    const double* col = T.panel + T.poff[s] + (size_t)t * f;
    double* xs = T.ybuf + T.yoff[s];
    double a = 0.0;
    for (int i = r0 + threadIdx.x; i < r1; i += ST_T) a = fma(col[i], xs[i], a);
    a = block_sum(a, red);
    if (threadIdx.x == 0) xs[t] -= a;
}

// backward, block b: x_b = L_bb^-T x_b (one warp)
__global__ void __launch_bounds__(32) k_bwdb_diag(StorePlan T, const int32_t* __restrict__ fronts, int b) {
    __shared__ double Lb[SBK][SBK + 1];
    const int s = fronts[blockIdx.x];
    const int4 h = T.hdr[s];
    const int e = h.x, f = h.y;
    const int t0 = b * SBK;
    if (t0 >= e) return;
    const int nb = min(SBK, e - t0);
    const double* L = T.panel + T.poff[s];
    double* xs = T.ybuf + T.yoff[s];
    for (int t = 0; t < nb; ++t)
        for (int i = threadIdx.x; i < nb; i += 32) Lb[i][t] = L[(size_t)(t0 + t) * f + t0 + i];
    __syncwarp();
    double v0 = threadIdx.x < nb ? xs[t0 + threadIdx.x] : 0.0;
    double v1 = threadIdx.x + 32 < nb ? xs[t0 + 32 + threadIdx.x] : 0.0;
    for (int t = nb - 1; t >= 0; --t) {                      // x_t is final; remove it from rows < t
        const double xt = __shfl_sync(0xffffffffu, t < 32 ? v0 : v1, t & 31);
        const int i0 = threadIdx.x, i1 = threadIdx.x + 32;
        if (i0 < t) v0 = fma(-Lb[t][i0], xt, v0);
        if (i1 < t) v1 = fma(-Lb[t][i1], xt, v1);
    }
    if (threadIdx.x < nb) xs[t0 + threadIdx.x] = v0;
    if (threadIdx.x + 32 < nb) xs[t0 + 32 + threadIdx.x] = v1;
}

__global__ void __launch_bounds__(ST_T) k_bwdb_fin(StorePlan T, const int32_t* __restrict__ fronts, double* __restrict__ x) {
    const int s = fronts[blockIdx.x];
    const int e = T.hdr[s].x;
    const int* lab = T.lab + T.loff[s];
    const double* xs = T.ybuf + T.yoff[s];
    for (int t = threadIdx.x; t < e; t += ST_T) x[lab[t]] = xs[t];
}

}  // namespace

void launch_store(const DevPlan& P, const StorePlan& T, const int32_t* fronts, int nfronts, cudaStream_t st) {
    if (nfronts <= 0) return;
    k_store<<<nfronts, ST_T, 0, st>>>(P, T, fronts);
}

static void set_smem_attr() {
    static unsigned long long done = 0;
    if (!first_on_device(done)) return;
    cudaFuncSetAttribute(k_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

int solve_max_front() { return 200 * 1024 / 16; }     // k_fwd keeps two vectors of f doubles
int solve_big_front() { return 2048; }                 // larger fronts: the blocked multi-CTA solves

void launch_fwd_big(const DevPlan& P, const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, int emax,
                    double* x, cudaStream_t st) {
    if (nfronts <= 0) return;
    k_fwdb_prep<<<nfronts, ST_T, 0, st>>>(P, T, fronts, x);
    const int nblk = (emax + SBK - 1) / SBK;
    for (int b = 0; b < nblk; ++b) {
        k_fwdb_diag<<<nfronts, 32, 0, st>>>(T, fronts, b);
        const int rows = fmax - b * SBK;
        if (rows > 0) k_fwdb_panel<<<dim3((rows + ST_T - 1) / ST_T, nfronts), ST_T, 0, st>>>(T, fronts, b);
    }
    k_fwdb_fin<<<nfronts, ST_T, 0, st>>>(T, fronts, x);
}

void launch_bwd_big(const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, int emax, double* x,
                    cudaStream_t st) {
    if (nfronts <= 0) return;
    (void)fmax;
    k_bwdb_prep<<<nfronts, ST_T, 0, st>>>(T, fronts, x);
    k_bwdb_cols<<<dim3(emax, nfronts), ST_T, 0, st>>>(T, fronts, 0, 1);
    const int nblk = (emax + SBK - 1) / SBK;
    for (int b = nblk - 1; b >= 0; --b) {
        k_bwdb_cols<<<dim3(SBK, nfronts), ST_T, 0, st>>>(T, fronts, b, 0);
        k_bwdb_diag<<<nfronts, 32, 0, st>>>(T, fronts, b);
    }
    k_bwdb_fin<<<nfronts, ST_T, 0, st>>>(T, fronts, x);
}

void launch_fwd(const DevPlan& P, const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, double* x,
                cudaStream_t st) {
    if (nfronts <= 0) return;
    set_smem_attr();
    const int fs = std::min(fmax, solve_max_front());
    k_fwd<<<nfronts, ST_T, (size_t)2 * fs * sizeof(double), st>>>(P, T, fronts, x);
}

void launch_bwd(const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, double* x, cudaStream_t st) {
    if (nfronts <= 0) return;
    set_smem_attr();
    const int fs = std::min(fmax, solve_max_front());
    k_bwd<<<nfronts, ST_T, (size_t)fs * sizeof(double), st>>>(T, fronts, x);
}

}  // namespace kep
