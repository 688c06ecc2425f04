// kernels_fast.cu — blocked front factorisation (a3 + a5) and the DMMA Schur
// update of the contribution block (a4).
//
// a3 (k_panel): one CTA per (front, shift).  The fully-summed (FS) columns are
// factorised in panels of NB accepted pivots.  Inside a panel each candidate
// column is brought up to date on demand (left-looking over the panel's
// earlier pivots) into a shared-memory buffer; it is written back only when
// its pivot is accepted, so a rejected (delayed) column stays "stale" and is
// swapped to the end of the FS block untouched.  After a panel, the remaining
// FS columns (all rows) receive the rank-NB update  A -= L W^T  on the FP64
// tensor cores (mma.sync m8n8k4 f64 = SASS DMMA).  The contribution block
// (CB x CB) is NOT touched here.
//
// Storage per front (lower = L / trailing matrix, upper = W^T):
//   L[i, t]  at F[i + t*ld]   (i > t, unit lower factor, t eliminated)
//   W[i, t]  at F[t + i*ld]   (the unscaled pivot column, W = L D)
//   D        diagonal / sub-diagonal of the eliminated block
// so that every update is  A -= L W^T = L D L^T  (Alg. 1 l.3).
//
// a4 (k_schur): CB -= L_CB W_CB^T over all eliminated pivots, one CTA per
// 64x64 lower tile of each CB of a level, K = #eliminated; operands staged
// through shared memory with cp.async (double buffered), DMMA inner product.
#include <cfloat>
#include <climits>
#include <cstdint>

#include "device.cuh"

namespace kep {

namespace {

constexpr double kAlpha = 0.6403882032022076;   // (1 + sqrt(17)) / 8
constexpr int PT = 256;                         // panel CTA threads
constexpr int NB = 32;                          // panel width (accepted pivots)

struct MaxIdx {
    double v;
    int i;
};

__device__ __forceinline__ MaxIdx better(MaxIdx a, MaxIdx b) {
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}

__device__ __forceinline__ MaxIdx warp_max_idx(MaxIdx x) {
    for (int o = 16; o > 0; o >>= 1) {
        MaxIdx y;
        y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
        y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
        x = better(x, y);
    }
    return x;
}

__device__ __forceinline__ double warp_max(double x) {
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// block-wide: (max,argmax) of a and plain max of b, c in one pass of barriers
__device__ void block_reduce3(MaxIdx& a, double& b, double& c, MaxIdx* sa, double* sb, double* sc) {
    a = warp_max_idx(a);
    b = warp_max(b);
    c = warp_max(c);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { sa[w] = a; sb[w] = b; sc[w] = c; }
    __syncthreads();
    MaxIdx ra = sa[0];
    double rb = sb[0], rc = sc[0];
#pragma unroll
    for (int q = 1; q < PT / 32; ++q) {
        ra = better(ra, sa[q]);
        rb = fmax(rb, sb[q]);
        rc = fmax(rc, sc[q]);
    }
    a = ra;
    b = rb;
    c = rc;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// symmetric interchange of positions a < b of the active part, with L rows
// (columns t < a) and W rows (upper, t < kacc accepted pivots)
__device__ void sym_swap_lw(double* F, int ld, int f, int a, int b, int kacc) {
    if (a == b) return;
    for (int t = threadIdx.x; t < f; t += PT) {
        if (t < a) {
            double* x = F + a + (size_t)t * ld;
            double* y = F + b + (size_t)t * ld;
            double v = *x; *x = *y; *y = v;
            if (t < kacc) {
                double* xw = F + t + (size_t)a * ld;
                double* yw = F + t + (size_t)b * ld;
                double w = *xw; *xw = *yw; *yw = w;
            }
        } else if (t == a) {
            double* x = F + a + (size_t)a * ld;
            double* y = F + b + (size_t)b * ld;
            double v = *x; *x = *y; *y = v;
        } else if (t < b) {
            double* x = F + t + (size_t)a * ld;
            double* y = F + b + (size_t)t * ld;
            double v = *x; *x = *y; *y = v;
        } else if (t > b) {
            double* x = F + t + (size_t)a * ld;
            double* y = F + t + (size_t)b * ld;
            double v = *x; *x = *y; *y = v;
        }
    }
    __syncthreads();
}

// A[i, j] -= sum_{t in [kp, e)} L[i,t] W[j,t]   for j in [e, q), i in [j, f)
__device__ void trailing_update(double* F, int ld, int f, int q, int kp, int e) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int ncol = q - e;
    const int nct = (ncol + 15) >> 4;          // 16-wide column tiles
    // enumerate (column tile, row tile of 32) pairs with rows >= tile's first column
    int total = 0;
    for (int ct = 0; ct < nct; ++ct) {
        const int j0 = e + 16 * ct;
        total += (f - j0 + 31) >> 5;
    }
    for (int w = warp; w < total; w += PT / 32) {
        int ct = 0, rem = w, j0 = e;
        for (;; ++ct) {
            j0 = e + 16 * ct;
            const int nr = (f - j0 + 31) >> 5;
            if (rem < nr) break;
            rem -= nr;
        }
        const int i0 = j0 + 32 * rem;
        double acc[4][2][2];
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
#pragma unroll
            for (int nb = 0; nb < 2; ++nb) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
        for (int t0 = kp; t0 < e; t0 += 4) {
            const int t = t0 + tg;
            const bool tv = t < e;
            double a[4], b[2];
#pragma unroll
            for (int mb = 0; mb < 4; ++mb) {
                const int i = i0 + 8 * mb + g;
                a[mb] = (tv && i < f) ? F[i + (size_t)t * ld] : 0.0;
            }
#pragma unroll
            for (int nb = 0; nb < 2; ++nb) {
                const int j = j0 + 8 * nb + g;
                b[nb] = (tv && j < q) ? F[t + (size_t)j * ld] : 0.0;
            }
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 2; ++nb) dmma(acc[mb][nb], a[mb], b[nb]);
        }
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int i = i0 + 8 * mb + g;
                    const int j = j0 + 8 * nb + 2 * tg + h;
                    if (i < f && j < q && i >= j) F[i + (size_t)j * ld] -= acc[mb][nb][h];
                }
    }
}

__global__ void __launch_bounds__(PT) k_panel(DevPlan P, const int32_t* __restrict__ fronts) {
    extern __shared__ double dyn[];
    __shared__ double wrowk[NB + 4], wrowr[NB + 4];
    __shared__ MaxIdx s_mi[PT / 32];
    __shared__ double s_b[PT / 32], s_c[PT / 32];
    const int s = fronts[blockIdx.x];
    const int sh = blockIdx.y;
    ShiftStat* st = P.stats + sh;
    const int32_t* nd_in = P.nd_in + (size_t)sh * P.nf;
    int32_t* nd_out = P.nd_out + (size_t)sh * P.nf;
    const int nd = nd_in[s];
    if (nd < 0) {
        if (threadIdx.x == 0) nd_out[s] = -1;
        return;
    }
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = f;
    const bool root = (c == 0);
    const double u = P.u;
    double* wk = dyn;          // current column k, indexed by position
    double* wr = dyn + f;      // current column r
    const int tid = threadIdx.x;
    unsigned long long c_neg = 0, c_zero = 0, c_pos = 0, c_2x2 = 0, c_del = 0;
    double minpiv = DBL_MAX;
    int e = 0, qe = q;
    while (e < qe) {
        const int kp = e;
        while (e < qe && e - kp < NB) {
            const int k = e, np = k - kp;
            if (tid < np) wrowk[tid] = F[(kp + tid) + (size_t)k * ld];
            __syncthreads();
            MaxIdx mC{-1.0, INT_MAX};
            double mR = 0.0, dummy = 0.0;
            for (int i = k + tid; i < f; i += PT) {
                double v = F[i + (size_t)k * ld];
                for (int t = 0; t < np; ++t) v = fma(-F[i + (size_t)(kp + t) * ld], wrowk[t], v);
                wk[i] = v;
                if (i > k) {
                    const double x = fabs(v);
                    if (i < qe) mC = better(mC, MaxIdx{x, i});
                    mR = fmax(mR, x);
                }
            }
            block_reduce3(mC, mR, dummy, s_mi, s_b, s_c);
            const double gC = mC.v > 0.0 ? mC.v : 0.0;
            const int r = mC.v >= 0.0 ? mC.i : k;
            const double gR = mR;
            const double akk = fabs(wk[k]);
            if (akk == 0.0 && gR == 0.0) {                 // zero column: exact zero pivot
                for (int i = k + tid; i < f; i += PT) {
                    if (i > k) { F[k + (size_t)i * ld] = 0.0; F[i + (size_t)k * ld] = 0.0; }
                    else F[k + (size_t)k * ld] = 0.0;
                }
                __syncthreads();
                c_zero++;
                minpiv = 0.0;
                e++;
                continue;
            }
            int kind = 1, j = k;
            double rho = 0.0, rall = 0.0;
            if (akk < kAlpha * gC) {
                if (tid < np) wrowr[tid] = F[(kp + tid) + (size_t)r * ld];
                __syncthreads();
                double mc = 0.0, ma = 0.0;
                MaxIdx dm{-1.0, INT_MAX};
                for (int i = k + tid; i < f; i += PT) {
                    double v = i < r ? F[r + (size_t)i * ld] : F[i + (size_t)r * ld];
                    for (int t = 0; t < np; ++t) v = fma(-F[i + (size_t)(kp + t) * ld], wrowr[t], v);
                    wr[i] = v;
                    if (i != r) {
                        const double x = fabs(v);
                        if (i < qe) mc = fmax(mc, x);
                        if (i != k) ma = fmax(ma, x);
                    }
                }
                block_reduce3(dm, mc, ma, s_mi, s_b, s_c);
                rho = mc;                                   // includes |a_kr| = gC
                rall = ma;                                  // column r, rows not in {k, r}
                const double arr = fabs(wr[r]);
                if (akk * rho >= kAlpha * gC * gC) { kind = 1; j = k; }
                else if (arr >= kAlpha * rho) { kind = 1; j = r; }
                else { kind = 2; j = r; }
            }
            if (!root) {
                bool ok;
                if (kind == 1 && j == k) {
                    ok = akk >= u * gR;
                } else if (kind == 1) {
                    ok = fabs(wr[r]) >= u * fmax(rall, gC);
                } else {
                    // gk' = max |wk[i]|, i in (k, f), i != r
                    double m = 0.0, d1 = 0.0;
                    MaxIdx dm{-1.0, INT_MAX};
                    for (int i = k + 1 + tid; i < f; i += PT)
                        if (i != r) m = fmax(m, fabs(wk[i]));
                    block_reduce3(dm, m, d1, s_mi, s_b, s_c);
                    const double gk = m, gr = rall;
                    const double a11 = wk[k], a21 = wk[r], a22 = wr[r];
                    const double det = a11 * a22 - a21 * a21;
                    if (det == 0.0) ok = false;
                    else {
                        const double ad = fabs(det);
                        const double t1 = (fabs(a22) * gk + fabs(a21) * gr) / ad;
                        const double t2 = (fabs(a21) * gk + fabs(a11) * gr) / ad;
                        ok = t1 <= 1.0 / u && t2 <= 1.0 / u;
                    }
                }
                if (!ok) {
                    sym_swap_lw(F, ld, f, k, qe - 1, k);
                    qe--;
                    c_del++;
                    continue;
                }
            }
            if (kind == 1) {
                const double* w = wk;
                if (j != k) {
                    sym_swap_lw(F, ld, f, k, j, k);
                    if (tid == 0) { const double x = wr[k]; wr[k] = wr[j]; wr[j] = x; }
                    __syncthreads();
                    w = wr;
                }
                const double d = w[k];
                const double dinv = 1.0 / d;
                for (int i = k + tid; i < f; i += PT) {
                    const double v = w[i];
                    if (i == k) F[k + (size_t)k * ld] = d;
                    else {
                        F[k + (size_t)i * ld] = v;          // W (upper)
                        F[i + (size_t)k * ld] = v * dinv;   // L (lower)
                    }
                }
                __syncthreads();
                if (d < 0.0) c_neg++; else if (d > 0.0) c_pos++; else c_zero++;
                minpiv = fmin(minpiv, fabs(d));
                e += 1;
            } else {
                sym_swap_lw(F, ld, f, k + 1, r, k);
                if (tid == 0) {
                    double x = wk[k + 1]; wk[k + 1] = wk[r]; wk[r] = x;
                    x = wr[k + 1]; wr[k + 1] = wr[r]; wr[r] = x;
                }
                __syncthreads();
                const double d11 = wk[k], d21 = wk[k + 1], d22 = wr[k + 1];
                const double det = d11 * d22 - d21 * d21;
                const double i11 = d22 / det, i21 = -d21 / det, i22 = d11 / det;
                for (int i = k + tid; i < f; i += PT) {
                    if (i == k) {
                        F[k + (size_t)k * ld] = d11;
                        F[k + 1 + (size_t)k * ld] = d21;
                        F[k + (size_t)(k + 1) * ld] = d21;
                        F[k + 1 + (size_t)(k + 1) * ld] = d22;
                    } else if (i >= k + 2) {
                        const double w1 = wk[i], w2 = wr[i];
                        F[k + (size_t)i * ld] = w1;
                        F[k + 1 + (size_t)i * ld] = w2;
                        F[i + (size_t)k * ld] = w1 * i11 + w2 * i21;
                        F[i + (size_t)(k + 1) * ld] = w1 * i21 + w2 * i22;
                    }
                }
                __syncthreads();
                const double tt = (d11 / d21) * (d22 / d21) - 1.0;
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
        if (e > kp && e < q) {
            trailing_update(F, ld, f, q, kp, e);
            __syncthreads();
        }
    }
    if (tid == 0) {
        nd_out[s] = q - e;
        if (c_neg) atomicAdd(&st->n_neg, c_neg);
        if (c_zero) atomicAdd(&st->n_zero, c_zero);
        if (c_pos) atomicAdd(&st->n_pos, c_pos);
        if (c_2x2) atomicAdd(&st->n_2x2, c_2x2);
        if (c_del) atomicAdd(&st->n_delayed, c_del);
        if (minpiv < DBL_MAX) atomic_min_pos_double(&st->minpiv_bits, minpiv);
    }
}

// ---------------------------------------------------------------- a4 Schur update
constexpr int ST = 64;          // CTA tile (rows and cols)
constexpr int KC = 16;          // K chunk per pipeline stage
constexpr int APAD = 72;        // A smem row stride (doubles), conflict-free fragments
constexpr int BPAD = 20;        // B smem row stride (doubles)
constexpr int SCH_T = 128;      // 4 warps, 2 x 2 of 32 x 32

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__global__ void __launch_bounds__(SCH_T) k_schur(DevPlan P, const int4* __restrict__ items) {
    __shared__ __align__(16) double As[2][KC][APAD];
    __shared__ __align__(16) double Bs[2][ST][BPAD];
    const int4 it = items[blockIdx.x];          // (front, I, J, -)
    const int s = it.x, I = it.y, J = it.z;
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = f;
    const int e = q - ndo;                       // eliminated pivots = K
    if (e <= 0) return;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const int r0 = q + I * ST, c0 = q + J * ST;  // tile origin (front positions)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    auto load = [&](int buf, int t0) {
        // A: KC x 64 (t, row), 1024 doubles; B: 64 x KC (col, t)
        for (int x = tid; x < KC * ST; x += SCH_T) {
            const int t = x / ST, i = x % ST;
            const int gi = r0 + i, gt = t0 + t;
            const bool v = gi < f && gt < e;
            cp_async8(&As[buf][t][i], F + (v ? (gi + (size_t)gt * ld) : 0), v);
        }
        for (int x = tid; x < KC * ST; x += SCH_T) {
            const int jj = x / KC, t = x % KC;
            const int gj = c0 + jj, gt = t0 + t;
            const bool v = gj < f && gt < e;
            cp_async8(&Bs[buf][jj][t], F + (v ? (gt + (size_t)gj * ld) : 0), v);
        }
        cp_async_commit();
    };
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const int nk = (e + KC - 1) / KC;
    load(0, 0);
    for (int kc = 0; kc < nk; ++kc) {
        const int buf = kc & 1;
        if (kc + 1 < nk) {
            load(buf ^ 1, (kc + 1) * KC);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll
        for (int k4 = 0; k4 < KC; k4 += 4) {
            double a[4], b[4];
#pragma unroll
            for (int mb = 0; mb < 4; ++mb) a[mb] = As[buf][k4 + tg][wm + 8 * mb + g];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) b[nb] = Bs[buf][wn + 8 * nb + g][k4 + tg];
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb], a[mb], b[nb]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = r0 + wm + 8 * mb + g;
                const int j = c0 + wn + 8 * nb + 2 * tg + h;
                if (i < f && j < f && i >= j) F[i + (size_t)j * ld] -= acc[mb][nb][h];
            }
}

}  // namespace

int panel_max_front() { return 4096; }

void launch_panel(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int max_f, cudaStream_t st) {
    const size_t smem = (size_t)2 * max_f * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4096 * 8);
        attr = true;
    }
    k_panel<<<dim3(nfronts, batch), PT, smem, st>>>(P, fronts);
}

void launch_schur(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st) {
    if (nitems <= 0) return;
    k_schur<<<dim3(nitems, batch), SCH_T, 0, st>>>(P, items);
}

}  // namespace kep
