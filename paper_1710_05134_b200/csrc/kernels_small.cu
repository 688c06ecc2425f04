// kernels_small.cu — row a3 (+ a5) of SURVEY.md §8 for fronts whose whole
// fully-summed panel fits in shared memory (the many small fronts of the lower
// elimination-tree levels: at c4, levels 0-3 hold ~40 % of the fronts' time).
//
// One CTA per (front, shift).  The assembled FS columns of the front (all f
// rows: FS rows and CB rows; the FS x FS block kept full symmetric) are loaded
// into shared memory once; the partial LDL^T then runs right-looking on them
// with the rule of DESIGN.md reading R1 exactly as the oracle states it
// (oracle/sparse_mf.py _partial_fs_bk): Bunch-Kaufman (alpha = (1+sqrt17)/8,
// PAPER.md:86) among the FS candidates, each pivot accepted only if the
// threshold test against its WHOLE current column holds (u; 1x1: |d| >= u
// max_i |a_ij|; 2x2: Duff-Reid), otherwise delayed to the parent.  Because the
// whole column is in shared memory the test is exact at pivot time: no rerun
// passes, no separate W21 solve.  The result is written back in the fast-path
// layout (kernels_front.cu), so k_schur, the parent's extend-add, k_store and
// k_resid read it unchanged:
//   FS rows of eliminated columns: G11 = L11 M (M = Q |Lambda|^1/2 per pivot
//   block, R21), D on the diagonal, 0 at a 2x2 block's in-pair entry;
//   CB rows: G21 = L21 M in the upper part F[t + i ld] (k_schur's operand), and
//   for the delayed columns the updated CB part W21 there (what the parent reads);
//   delayed x delayed block: the updated values in the lower part;
//   aux records: D, kind, permutation, sign and G coefficients of every pivot.
// A front whose panel exceeds the launch's shared memory (more delayed columns
// than planned) is flagged FL_REF for the unblocked kernel (k_factor_ref).
#include <cfloat>
#include <climits>
#include <cstdint>

#include "device.cuh"

namespace kep {

namespace {

constexpr double kAlphaS = 0.6403882032022076;   // (1 + sqrt(17)) / 8

struct MI {
    double v;
    int i;
};

__device__ __forceinline__ MI mi_better(MI a, MI b) {
    return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}

// block-wide (max, argmax) of a and max of b, c, d
template <int TH>
__device__ __forceinline__ void reduce4(MI& a, double& b, double& c, double& d, MI (*sa2)[TH / 32 > 0 ? TH / 32 : 1],
                                        double (*sx2)[3][TH / 32 > 0 ? TH / 32 : 1], int& flip) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        MI y;
        y.v = __shfl_xor_sync(0xffffffffu, a.v, o);
        y.i = __shfl_xor_sync(0xffffffffu, a.i, o);
        a = mi_better(a, y);
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    if (TH > 32) {
        // two scratch records used alternately: a record is rewritten two reductions later,
        // after at least one more barrier, so one barrier per reduction suffices
        MI* sa = sa2[flip];
        double (*sx)[TH / 32 > 0 ? TH / 32 : 1] = sx2[flip];
        flip ^= 1;
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) { sa[w] = a; sx[0][w] = b; sx[1][w] = c; sx[2][w] = d; }
        __syncthreads();
        a = sa[0]; b = sx[0][0]; c = sx[1][0]; d = sx[2][0];
#pragma unroll
        for (int q = 1; q < TH / 32; ++q) {
            a = mi_better(a, sa[q]);
            b = fmax(b, sx[0][q]);
            c = fmax(c, sx[1][q]);
            d = fmax(d, sx[2][q]);
        }
    }
}

template <int TH>
__device__ __forceinline__ void bar() {
    if (TH > 32) __syncthreads(); else __syncwarp();
}

}  // namespace

// at least 2048 / TH / 2 CTAs per SM (half of the thread limit): caps the registers per thread at 64
template <int TH>
__global__ void __launch_bounds__(TH, 1024 / TH) k_small(DevPlan P, const int32_t* __restrict__ fronts, int cap_doubles) {
    extern __shared__ __align__(16) double Ps[];         // [q][LDS] column-major FS panel, all rows
    __shared__ MI s_a[2][TH / 32 > 0 ? TH / 32 : 1];
    __shared__ double s_x[2][3][TH / 32 > 0 ? TH / 32 : 1];
    int flip = 0;
    __shared__ int s_perm[64 + 64];                       // FS positions (q <= 128 on this path)
    const int s = fronts[blockIdx.x];
    const int sh = blockIdx.y;
    const int tid = threadIdx.x;
    const int32_t* nd_in = P.nd_in + (size_t)sh * P.nf;
    int32_t* nd_out = P.nd_out + (size_t)sh * P.nf;
    int32_t* flag = P.flag + (size_t)sh * P.nf + s;
    ShiftStat* st = P.stats + sh;
    const int nd = nd_in[s];
    if (nd < 0) {                                         // slack overflow: the batch is re-planned
        if (tid == 0) { nd_out[s] = -1; *flag = FL_OK; }
        return;
    }
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int LDS = f | 1;                                // odd stride: row-wise panel reads spread over banks
    if ((int64_t)q * LDS > cap_doubles || q > 128) {    // more delayed columns than planned: unblocked kernel
        if (tid == 0) *flag = FL_REF;
        return;
    }
    const bool root = c == 0;
    const double u = P.u;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    // ---- load the FS columns: FS x FS block full symmetric, CB rows from the lower part
    for (int x = tid; x < q * f; x += TH) {
        const int t = x / f, i = x - t * f;
        Ps[(size_t)t * LDS + i] = i >= t ? F[i + (size_t)t * ld] : F[t + (size_t)i * ld];
    }
    for (int i = tid; i < q; i += TH) s_perm[i] = i;
    __syncthreads();

    unsigned long long c_neg = 0, c_zero = 0, c_pos = 0, c_2x2 = 0;
    double minpiv = DBL_MAX;
    int e = 0, qe = q;
    auto col = [&](int j) -> double* { return Ps + (size_t)j * LDS; };
    // symmetric interchange of FS positions a < b in one pass (each element moved by one thread):
    // rows a, b of the other panel columns, rows i != a, b of columns a, b, and the 2 x 2 intersection
    auto swap_sym = [&](int a, int b) {
        if (a == b) return;
        double* ca = col(a);
        double* cb = col(b);
        for (int x = tid; x < q + f; x += TH) {
            if (x < q) {
                if (x == a || x == b) continue;
                double* cl = col(x);
                const double y = cl[a]; cl[a] = cl[b]; cl[b] = y;
            } else {
                const int i = x - q;
                if (i == a || i == b) continue;
                const double y = ca[i]; ca[i] = cb[i]; cb[i] = y;
            }
        }
        if (tid == 0) {
            const double y = ca[a]; ca[a] = cb[b]; cb[b] = y;      // (a,a) <-> (b,b); (b,a) = (a,b) stays
            const int z = s_perm[a]; s_perm[a] = s_perm[b]; s_perm[b] = z;
        }
        bar<TH>();
    };
    while (e < qe) {
        const int k = e;
        const double* ck = col(k);
        // column k: FS candidates (k, qe) -> (gC, r); all rows (k, f) -> gR
        MI mC{-1.0, INT_MAX};
        double gR = 0.0, z1 = 0.0, z2 = 0.0;
        for (int i = k + 1 + tid; i < f; i += TH) {
            const double a = fabs(ck[i]);
            if (i < qe) mC = mi_better(mC, MI{a, i});
            gR = fmax(gR, a);
        }
        reduce4<TH>(mC, gR, z1, z2, s_a, s_x, flip);
        const double gC = mC.v > 0.0 ? mC.v : 0.0;
        const int r = mC.v >= 0.0 ? mC.i : k;
        const double akk = fabs(ck[k]);
        if (akk == 0.0 && gR == 0.0) {                    // zero column: exact zero pivot, nothing to update
            if (tid == 0) {
                A.kind[k] = PK_ZERO; A.d[k] = 0.0; A.ds[k] = 0.0;
                A.sgn[k] = 1.0; A.gca[k] = 0.0; A.gcb[k] = 0.0;
            }
            c_zero++;
            minpiv = 0.0;
            e++;
            continue;
        }
        int kind = 1, j = k;
        double rall = 0.0, gk = 0.0;                     // column r rows not in {k, r}; column k rows not in {k, r}
        if (akk < kAlphaS * gC) {
            const double* cr = col(r);
            MI dm{-1.0, INT_MAX};
            double rho = 0.0, ra = 0.0;
            double gkk = 0.0;
            for (int i = k + tid; i < f; i += TH) {
                if (i == r) continue;
                const double a = fabs(cr[i]);
                if (i < qe) rho = fmax(rho, a);              // includes |a_kr| = gC
                if (i != k) { ra = fmax(ra, a); gkk = fmax(gkk, fabs(ck[i])); }
            }
            double rho2 = rho;
            reduce4<TH>(dm, rho2, ra, gkk, s_a, s_x, flip);
            rall = ra;
            gk = gkk;
            const double arr = fabs(cr[r]);
            if (akk * rho2 >= kAlphaS * gC * gC) { kind = 1; j = k; }
            else if (arr >= kAlphaS * rho2) { kind = 1; j = r; }
            else { kind = 2; j = r; }
        }
        bool ok = true;
        if (!root) {
            if (kind == 1) {
                const double fa = (j == k) ? gR : fmax(rall, gC);      // whole column j, rows != j
                ok = fabs(col(j)[j]) >= u * fa;
            } else {
                const double a11 = ck[k], a21 = ck[r], a22 = col(r)[r];
                const double det = a11 * a22 - a21 * a21;
                if (det == 0.0) ok = false;
                else {
                    const double ad = fabs(det);
                    ok = (fabs(a22) * gk + fabs(a21) * rall) / ad <= 1.0 / u &&
                         (fabs(a21) * gk + fabs(a11) * rall) / ad <= 1.0 / u;
                }
            }
        }
        bar<TH>();                                        // everyone has read the column values used above
        if (!ok) {                                        // delay column k to the parent (R1)
            swap_sym(k, qe - 1);
            qe--;
            continue;
        }
        if (kind == 1) {
            swap_sym(k, j);
            const double* w = col(k);
            const double d = w[k], dinv = 1.0 / d;
            // right-looking update of the remaining panel columns (all rows below k)
            for (int i = k + 1 + tid; i < f; i += TH) {       // thread per row, columns in turn
                const double li = w[i] * dinv;
                for (int jj = k + 1; jj < q; ++jj) col(jj)[i] -= li * w[jj];
            }
            bar<TH>();                                    // W = L d stays in column k (converted at write-back)
            if (tid == 0) {
                const double sg = d < 0.0 ? -1.0 : 1.0;
                A.kind[k] = PK_1X1; A.d[k] = d; A.ds[k] = 0.0;
                A.sgn[k] = sg; A.gca[k] = sg / sqrt(fabs(d)); A.gcb[k] = 0.0;
            }
            if (d < 0.0) c_neg++; else if (d > 0.0) c_pos++; else c_zero++;
            minpiv = fmin(minpiv, fabs(d));
            e += 1;
        } else {
            swap_sym(k + 1, r);
            const double* w1 = col(k);
            const double* w2 = col(k + 1);
            const double d11 = w1[k], d21 = w1[k + 1], d22 = w2[k + 1];
            const double det = d11 * d22 - d21 * d21;
            const double i11 = d22 / det, i21 = -d21 / det, i22 = d11 / det;
            for (int i = k + 2 + tid; i < f; i += TH) {       // thread per row: L[i, k:k+2] = W[i] D^-1
                const double a1 = w1[i], a2 = w2[i];
                const double l1 = a1 * i11 + a2 * i21, l2 = a1 * i21 + a2 * i22;
                for (int jj = k + 2; jj < q; ++jj) col(jj)[i] -= l1 * w1[jj] + l2 * w2[jj];
            }
            bar<TH>();                                    // W = L D stays in columns k, k+1
            if (tid == 0) {
                A.kind[k] = PK_2X2A; A.d[k] = d11; A.ds[k] = d21;
                A.kind[k + 1] = PK_2X2B; A.d[k + 1] = d22; A.ds[k + 1] = 0.0;
                double cs, sn, l1, l2;
                pair_eig(d11, d21, d22, cs, sn, l1, l2);
                const double s1 = l1 < 0.0 ? -1.0 : 1.0, s2 = l2 < 0.0 ? -1.0 : 1.0;
                const double k1 = s1 / sqrt(fabs(l1)), k2 = s2 / sqrt(fabs(l2));
                A.sgn[k] = s1; A.sgn[k + 1] = s2;
                A.gca[k] = cs * k1;     A.gcb[k] = sn * k1;
                A.gca[k + 1] = cs * k2; A.gcb[k + 1] = -sn * k2;
            }
            const double tt = (d11 / d21) * (d22 / d21) - 1.0;          // a5: sign(det), scaled (R2)
            if (tt < 0.0) { c_neg++; c_pos++; }
            else if (tt > 0.0) { if (d11 < 0.0) c_neg += 2; else c_pos += 2; }
            else { c_zero++; if (d11 + d22 < 0.0) c_neg++; else c_pos++; }
            const double tr = 0.5 * (d11 + d22);
            const double disc = sqrt(0.25 * (d11 - d22) * (d11 - d22) + d21 * d21);
            const double big = fabs(tr) + disc;
            minpiv = fmin(minpiv, big > 0.0 ? fabs(det) / big : 0.0);
            c_2x2++;
            e += 2;
        }
    }
    // ---- write back in the fast-path layout.  The panel holds W = L D; per column t the G
    // column is G[:, t] = W[:, a] g1[t] + W[:, a+1] g2[t] (a = t's pivot block start; G = L M).
    __shared__ double g1[128], g2[128];
    __shared__ int ga[128];
    for (int i = tid; i < q; i += TH) A.perm[i] = s_perm[i];
    for (int t = tid; t < q; t += TH) {
        double x1 = 0.0, x2 = 0.0;
        int a = t;
        if (t >= e) x1 = 1.0;                              // delayed column: W21 itself
        else {
            const int kd = A.kind[t];
            if (kd == PK_1X1) { const double d = A.d[t]; x1 = sqrt(fabs(d)) / d; }
            else if (kd == PK_2X2A || kd == PK_2X2B) {
                a = kd == PK_2X2A ? t : t - 1;
                const double d11 = A.d[a], d21 = A.ds[a], d22 = A.d[a + 1];
                const double det = d11 * d22 - d21 * d21;
                const double i11 = d22 / det, i21 = -d21 / det, i22 = d11 / det;
                double cs, sn, l1, l2;
                pair_eig(d11, d21, d22, cs, sn, l1, l2);
                const double r1 = sqrt(fabs(l1)), r2 = sqrt(fabs(l2));
                if (kd == PK_2X2A) { x1 = (i11 * cs + i21 * sn) * r1; x2 = (i21 * cs + i22 * sn) * r1; }
                else { x1 = (i21 * cs - i11 * sn) * r2; x2 = (i22 * cs - i21 * sn) * r2; }
            }
        }
        g1[t] = x1; g2[t] = x2; ga[t] = a;
    }
    __syncthreads();
    // FS rows (lower part, column by column): eliminated columns G11 with D on the diagonal and 0 at the
    // in-pair entry; delayed columns their updated values (trailing FS block)
    for (int x = tid; x < q * q; x += TH) {
        const int t = x / q, i = x - t * q;
        if (i < t) continue;
        double v;
        if (t < e && i == t) v = A.d[t];
        else if (t < e && A.kind[t] == PK_2X2A && i == t + 1) v = 0.0;
        else v = col(ga[t])[i] * g1[t] + (g2[t] != 0.0 ? col(ga[t] + 1)[i] * g2[t] : 0.0);
        F[i + (size_t)t * ld] = v;
    }
    // CB rows (upper part, row by row: coalesced): G21 for eliminated columns, W21 for delayed ones
    for (int x = tid; x < c * q; x += TH) {
        const int ii = x / q, t = x - ii * q, i = q + ii;
        const double v = col(ga[t])[i] * g1[t] + (g2[t] != 0.0 ? col(ga[t] + 1)[i] * g2[t] : 0.0);
        F[t + (size_t)i * ld] = v;
    }
    if (tid == 0) {
        nd_out[s] = q - e;
        *flag = FL_OK;
    }
    // inertia (a5), delays, smallest pivot
    __shared__ unsigned long long s_cnt[4];
    if (tid == 0) {
        if (c_neg) atomicAdd(&st->n_neg, c_neg);
        if (c_zero) atomicAdd(&st->n_zero, c_zero);
        if (c_pos) atomicAdd(&st->n_pos, c_pos);
        if (c_2x2) atomicAdd(&st->n_2x2, c_2x2);
        if (q - e) atomicAdd(&st->n_delayed, (unsigned long long)(q - e));
        if (minpiv < DBL_MAX) atomic_min_pos_double(&st->minpiv_bits, minpiv);
    }
    (void)s_cnt;
}

size_t small_smem_bytes(int cap_doubles) { return (size_t)cap_doubles * sizeof(double); }

void launch_small(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int cap_doubles, int threads,
                  cudaStream_t st) {
    if (nfronts <= 0) return;
    const size_t smem = small_smem_bytes(cap_doubles);
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(k_small<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_small<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_small<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_small<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    if (threads <= 32) k_small<32><<<dim3(nfronts, batch), 32, smem, st>>>(P, fronts, cap_doubles);
    else if (threads <= 64) k_small<64><<<dim3(nfronts, batch), 64, smem, st>>>(P, fronts, cap_doubles);
    else if (threads <= 128) k_small<128><<<dim3(nfronts, batch), 128, smem, st>>>(P, fronts, cap_doubles);
    else k_small<256><<<dim3(nfronts, batch), 256, smem, st>>>(P, fronts, cap_doubles);
}

}  // namespace kep
