// kernels_front.cu — rows a3 + a5 of SURVEY.md §8 for the fast path: partial
// LDL^T of the fully-summed (FS) columns of every front of one level with
// Bunch–Kaufman pivoting, the threshold test and delayed pivots (DESIGN.md
// reading R1; PAPER.md:86 cites Bunch–Kaufman; Alg. 1' line 3, PAPER.md:419,
// factorises A - sigma B).
//
// Front  F = [A11 A21^T; A21 A22]  (A11: q x q FS block, A21: c x q CB rows).
// Partial factorisation  P A11 P^T = L11 D11 L11^T,  W21 = A21 P^T L11^-T,
// L21 = W21 D11^-1,  Schur complement A22 - W21 L21^T (row a4, k_schur).
//
// The threshold test of R1 compares a pivot with the maximum of its whole
// current column, FS rows AND CB rows.  Every such maximum is
// max(FS part, CB part), and the CB part of the column eliminated at
// position t is exactly max_i |W21[i, t]|.  So the rule is applied in three
// kernels per level:
//
//  k_fs    one CTA per (front, shift): the FS x FS block only.  Blocks of NB
//          pivots, raw block columns in shared memory, candidate columns
//          brought up to date on demand (left-looking inside the block), BK
//          choice (alpha = (1+sqrt17)/8) among the FS candidates, threshold
//          test with the FS maxima (a column failing there is delayed — the
//          full test fails too), rank-nb DMMA update of the FS trailing
//          block (k_fsu).  Records, per position, the pivot kind, D, the FS
//          maxima and the permutation.
//  k_l21   many CTAs per front: 64 CB rows each, the unit-triangular solve
//          W21 = A21 P^T L11^-T (DMMA for the off-block part), written to
//          the upper triangle of the CB columns, and the column maxima of
//          W21 (the CB parts of the tests).
//  k_check one CTA per front: re-evaluates every test in pivot order with
//          the full-column maxima.  All pass -> the pivot sequence is the
//          unblocked rule's; inertia is counted and L21 = W21 D^-1 written.
//          A failure -> the front is assembled again (its children's CBs are
//          still live during the level) and rerun with a forced delay at the
//          failing step; after FMAX forced delays, or once the level's kReruns = 2 rerun passes
//          (api.cu) are used up, it is handed to k_factor_ref.
//
// Storage per front (column-major, ld = f):  L[i,t] at F[i + t*ld] (i > t;
// 0 at the subdiagonal of a 2x2 block, whose D lives in the aux record),
// W21[i,t] at F[t + i*ld] for CB rows i.
#include <cfloat>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"

namespace kep {

namespace {

constexpr double kAlpha = 0.6403882032022076;   // (1 + sqrt(17)) / 8
constexpr int FT = 256;                         // k_fs / k_check threads
constexpr int LT = 256;                         // k_l21 threads (8 warps x 16 rows)
constexpr int LR = 128;                         // k_l21 CB rows per CTA
constexpr int LB = 32;                          // k_l21 column block
constexpr int LST = 3;                          // k_l21 cp.async pipeline depth
static_assert(LT == 8 * LB, "k_l21 column-max reduction maps 8 threads to a column");
constexpr int KC = 16;                          // K chunk of the k_l21 GEMM
constexpr int kXMin = 48;                       // k_l21<2> (GEMM in-block solve) from this FS capacity (c4 sweep 32/48/56/64)
constexpr int kXMaxBlocks = 256;                // ... up to this many column blocks
constexpr int XPW = 4;                          // k_l21x_prep warps per CTA
constexpr int APAD = LR + 4;                    // = 4 (mod 16): conflict-free f64 fragments
constexpr int BP = KC + 4;

struct MaxIdx {
    double v;
    int i;
};

__device__ __forceinline__ MaxIdx better(MaxIdx a, MaxIdx b) {
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}

struct Red {
    MaxIdx mi[8];
    double x[3][8];
};

// block-wide (max, argmax) of a and max of b, c, d.  R points at two scratch
// records used alternately (flip toggles), so one barrier per reduction suffices:
// a record is rewritten two reductions later, after another barrier.
template <int TH>
__device__ void block_reduce(MaxIdx& a, double& b, double& c, double& d, Red* R2, int& flip) {
    Red* R = R2 + flip;
    flip ^= 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        MaxIdx y;
        y.v = __shfl_xor_sync(0xffffffffu, a.v, o);
        y.i = __shfl_xor_sync(0xffffffffu, a.i, o);
        a = better(a, y);
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { R->mi[w] = a; R->x[0][w] = b; R->x[1][w] = c; R->x[2][w] = d; }
    __syncthreads();
    a = R->mi[0]; b = R->x[0][0]; c = R->x[1][0]; d = R->x[2][0];
#pragma unroll
    for (int q = 1; q < TH / 32; ++q) {
        a = better(a, R->mi[q]);
        b = fmax(b, R->x[0][q]);
        c = fmax(c, R->x[1][q]);
        d = fmax(d, R->x[2][q]);
    }
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src, int bytes) {   // bytes in {0, 8, 16}
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Symmetric interchange of FS positions a < b in the lower FS x FS block
// (rows/columns of the active part and L rows of the columns t < a).
template <int TH>
__device__ void sym_swap_fs(double* F, int ld, int q, int a, int b) {
    if (a == b) return;
    for (int t = threadIdx.x; t < q; t += TH) {
        if (t < a) {
            double* x = F + a + (size_t)t * ld;
            double* y = F + b + (size_t)t * ld;
            double v = *x; *x = *y; *y = v;
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
}

template <int NB>
struct Smem {
    double* Ls;            // [NB][RS] block columns by position row (i - kp); raw, then L
    double* wk;            // [RS] updated column k (FS rows)
    double* wr;            // [RS] updated column r
    double* cs;            // [NB] W = Ls[t]*cs + Ls[t+oo]*co  (W = L D)
    double* co;
    double* wrow;          // [NB]
    double* wrowr;         // [NB]
    double* d1;            // [NB] D diagonal / 2x2 entries, FS maxima of the tests
    double* d2;
    double* fa;
    double* fb;
    int* oo;               // [NB] 2x2 partner offset (0 / +1 / -1)
    int* tp;               // [NB] kind per block column
    int* st;               // [NB] S1 step index per block column
    Red* red;
};

// gls != NULL: the block columns and the two column buffers live in a global
// scratch area of the front (FS blocks too large for shared memory).
template <int NB>
__device__ Smem<NB> carve(double* base, int RS, double* gls) {
    Smem<NB> S;
    double* p = base;
    double* g = gls ? gls : base;
    S.Ls = g; g += (size_t)NB * RS;
    S.wk = g; g += RS;
    S.wr = g; g += RS;
    if (!gls) p = g;
    S.cs = p; p += NB;
    S.co = p; p += NB;
    S.wrow = p; p += NB;
    S.wrowr = p; p += NB;
    S.d1 = p; p += NB;
    S.d2 = p; p += NB;
    S.fa = p; p += NB;
    S.fb = p; p += NB;
    S.red = (Red*)p; p += (2 * sizeof(Red) + 7) / 8;
    S.oo = (int*)p; p += (NB + 1) / 2;
    S.tp = (int*)p; p += (NB + 1) / 2;
    S.st = (int*)p; p += (NB + 1) / 2;
    return S;
}

}  // namespace

size_t fs_smem_bytes(int nb, int RS, bool gls) {
    size_t d = (gls ? 0 : (size_t)nb * RS + 2 * (size_t)RS) + 8 * nb + (2 * sizeof(Red) + 7) / 8 + 3 * ((nb + 1) / 2);
    return d * sizeof(double);
}

size_t fs_gls_doubles(int nb, int RS) { return (size_t)(nb + 2) * RS; }

namespace {

template <int NB>
__device__ __forceinline__ double wform(const Smem<NB>& S, int RS, int t, int ii) {
    // W[position kp+ii, block column t]
    const double* L = S.Ls + (size_t)t * RS + ii;
    const int o = S.oo[t];
    return L[0] * S.cs[t] + (o ? L[(ptrdiff_t)o * RS] * S.co[t] : 0.0);
}

// After the global interchange of positions a < b: L rows a, b of all block
// columns (raw ones included), whole raw columns a, b reloaded, rows a, b of
// the other raw columns reloaded.  kfirst = first raw (not yet pivoted) column.
template <int NB, int TH>
__device__ void swap_block(const Smem<NB>& S, int RS, const double* F, int ld, int q, int kp, int kfirst, int a, int b,
                           int* perm) {
    const int tid = threadIdx.x;
    __syncthreads();                                   // global interchange complete
    for (int t = tid; t < NB; t += TH) {
        double* col = S.Ls + (size_t)t * RS;
        const double x = col[a - kp];
        col[a - kp] = col[b - kp];
        col[b - kp] = x;
    }
    if (tid == 0) { const int x = perm[a]; perm[a] = perm[b]; perm[b] = x; }
    __syncthreads();
    const int hi = min(kp + NB, q);
    for (int j = kfirst + tid; j < hi; j += TH) {
        if (j == a || j == b) continue;
        double* col = S.Ls + (size_t)(j - kp) * RS;
        if (a >= j) col[a - kp] = F[a + (size_t)j * ld];
        if (b >= j) col[b - kp] = F[b + (size_t)j * ld];
    }
    const int cols[2] = {a, b};
    for (int x = 0; x < 2; ++x) {
        const int j = cols[x];
        if (j < kfirst || j >= hi) continue;
        double* col = S.Ls + (size_t)(j - kp) * RS;
        for (int i = j + tid; i < q; i += TH) col[i - kp] = F[i + (size_t)j * ld];
    }
    __syncthreads();
}

template <int NB, int TH>
__device__ void do_swap(const Smem<NB>& S, int RS, double* F, int ld, int q, int kp, int kfirst, int a, int b, int* perm) {
    if (a == b) return;
    sym_swap_fs<TH>(F, ld, q, a, b);
    swap_block<NB, TH>(S, RS, F, ld, q, kp, kfirst, a, b, perm);
}

// One block of at most NB pivots per launch (mode 0: first block of pass 0;
// mode 1: first block of a rerun pass; mode 2: next block).  The state between
// launches (e, qe, S1 step, forced-delay cursor, block start) lives in fstate.
// TH threads per front (one warp for tiny FS blocks).
template <int NB, int TH, bool GLS>
__global__ void __launch_bounds__(TH) k_fsp(DevPlan P, const int32_t* __restrict__ fronts, int RS, int mode) {
    extern __shared__ __align__(16) double dyn[];
    const int s = fronts[blockIdx.x];
    const int sh = blockIdx.y;
    // compile-time choice: with GLS = false every block-column access is a shared-memory access
    const Smem<NB> S = carve<NB>(dyn, RS, GLS ? P.gscratch + (size_t)sh * P.gscratch_stride + P.goff[s] : nullptr);
    const int32_t* nd_in = P.nd_in + (size_t)sh * P.nf;
    int32_t* nd_out = P.nd_out + (size_t)sh * P.nf;
    const int nd = nd_in[s];
    int32_t* flag = P.flag + (size_t)sh * P.nf + s;
    int32_t* forced = P.forced + ((size_t)sh * P.nf + s) * (FMAX + 1);
    int32_t* fst = P.fstate + ((size_t)sh * P.nf + s) * FSTATE_W;
    if (mode == 2) {
        if (*flag != FL_ACTIVE) return;
        const bool done = fst[0] >= fst[1];
        __syncthreads();
        if (threadIdx.x == 0) fst[5] = 0;                // the previous block's update has been applied
        if (done) return;
    } else if (mode == 1) {
        if (*flag != FL_RERUN) return;
    } else if (threadIdx.x == 0) {
        forced[0] = 0;
    }
    if (nd < 0) {
        if (threadIdx.x == 0) { nd_out[s] = -1; *flag = FL_OK; }
        return;
    }
    __shared__ int s_forced[FMAX + 1];
    if (threadIdx.x <= FMAX) s_forced[threadIdx.x] = mode ? forced[threadIdx.x] : 0;
    __syncthreads();
    if (threadIdx.x == 0) *flag = FL_ACTIVE;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    (void)f;
    const bool root = (c == 0);
    const double u = P.u;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int Q = P.cap[s] - c;
    AuxRec A = aux_rec(P, sh, s, Q);

    int e = 0, qe = q;
    int step = 0, fnext = 0;                           // S1 actions so far; next forced delay
    int rflip = 0;                                     // block_reduce scratch toggle
    if (mode < 2) {
        for (int i = tid; i < q; i += TH) { A.perm[i] = i; A.cm[i] = 0ull; }
    } else {
        e = fst[0]; qe = fst[1]; step = fst[2]; fnext = fst[3];
    }
    __syncthreads();
    const int kp = e;
    {
        {   // raw block columns [kp, kp+NB), rows [j, q)
            const int npre = min(NB, q - kp), R = q - kp;
            for (int idx = tid; idx < npre * R; idx += TH) {
                const int x = idx / R, ii = idx - x * R;
                if (ii >= x) S.Ls[(size_t)x * RS + ii] = F[(kp + ii) + (size_t)(kp + x) * ld];
            }
            __syncthreads();
        }
        while (e < qe && e - kp < NB) {
            const int k = e, t = k - kp;
            if (fnext < s_forced[0] && step == s_forced[1 + fnext]) {
                // the full-column test failed here in an earlier pass: delay (R1)
                do_swap<NB, TH>(S, RS, F, ld, q, kp, k, k, qe - 1, A.perm);
                qe--;
                fnext++;
                step++;
                continue;
            }
            if (tid < t) S.wrow[tid] = wform<NB>(S, RS, tid, k - kp);
            __syncthreads();
            MaxIdx mC{-1.0, INT_MAX};
            double mR = 0.0, z1 = 0.0, z2 = 0.0;
            {
                const double* raw = S.Ls + (size_t)t * RS;
                for (int i = k + tid; i < q; i += TH) {
                    const int ii = i - kp;
                    double v = raw[ii];
                    for (int x = 0; x < t; ++x) v = fma(-S.Ls[(size_t)x * RS + ii], S.wrow[x], v);
                    S.wk[ii] = v;
                    if (i > k) {
                        const double a = fabs(v);
                        if (i < qe) mC = better(mC, MaxIdx{a, i});
                        mR = fmax(mR, a);
                    }
                }
            }
            block_reduce<TH>(mC, mR, z1, z2, S.red, rflip);
            const double gC = mC.v > 0.0 ? mC.v : 0.0;
            const int r = mC.v >= 0.0 ? mC.i : k;
            const double akk = fabs(S.wk[k - kp]);
            if (akk == 0.0 && mR == 0.0) {
                // FS part of column k is zero: a zero pivot if its CB part is
                // zero too (k_check), else the unblocked rule delays it there
                for (int i = k + tid; i < q; i += TH) S.Ls[(size_t)t * RS + (i - kp)] = 0.0;
                if (tid == 0) {
                    S.cs[t] = 0.0; S.co[t] = 0.0; S.oo[t] = 0; S.tp[t] = PK_ZERO;
                    S.d1[t] = 0.0; S.d2[t] = 0.0; S.fa[t] = 0.0; S.fb[t] = 0.0; S.st[t] = step;
                }
                __syncthreads();
                e++;
                step++;
                continue;
            }
            int kind = 1, j = k;
            double rall = 0.0, gk = 0.0;
            if (akk < kAlpha * gC) {
                if (tid < t) S.wrowr[tid] = wform<NB>(S, RS, tid, r - kp);
                __syncthreads();
                double mc = 0.0, ma = 0.0, m3 = 0.0;
                MaxIdx dm{-1.0, INT_MAX};
                for (int i = k + tid; i < q; i += TH) {
                    const int ii = i - kp;
                    double v = i >= r ? F[i + (size_t)r * ld] : F[r + (size_t)i * ld];
                    for (int x = 0; x < t; ++x) v = fma(-S.Ls[(size_t)x * RS + ii], S.wrowr[x], v);
                    S.wr[ii] = v;
                    if (i != r) {
                        const double a = fabs(v);
                        if (i < qe) mc = fmax(mc, a);
                        if (i != k) { ma = fmax(ma, a); m3 = fmax(m3, fabs(S.wk[ii])); }
                    }
                }
                block_reduce<TH>(dm, mc, ma, m3, S.red, rflip);
                const double rho = mc;                       // includes |a_kr| = gC
                rall = ma;                                   // column r, rows not in {k, r}
                gk = m3;                                     // column k, rows not in {k, r}
                const double arr = fabs(S.wr[r - kp]);
                if (akk * rho >= kAlpha * gC * gC) { kind = 1; j = k; }
                else if (arr >= kAlpha * rho) { kind = 1; j = r; }
                else { kind = 2; j = r; }
            }
            if (kind == 2 && t + 2 > NB) break;             // no room for the 2x2 in this block
            double fa = 0.0, fb = 0.0;
            bool ok = true;
            if (kind == 1 && j == k) fa = mR;
            else if (kind == 1) fa = fmax(rall, gC);
            else { fa = gk; fb = rall; }
            if (!root) {
                if (kind == 1) ok = fabs(j == k ? S.wk[k - kp] : S.wr[r - kp]) >= u * fa;
                else {
                    const double a11 = S.wk[k - kp], a21 = S.wk[r - kp], a22 = S.wr[r - kp];
                    const double det = a11 * a22 - a21 * a21;
                    if (det == 0.0) ok = false;
                    else {
                        const double ad = fabs(det);
                        ok = (fabs(a22) * fa + fabs(a21) * fb) / ad <= 1.0 / u &&
                             (fabs(a21) * fa + fabs(a11) * fb) / ad <= 1.0 / u;
                    }
                }
            }
            if (!ok) {                                      // fails on the FS rows already: delay
                do_swap<NB, TH>(S, RS, F, ld, q, kp, k, k, qe - 1, A.perm);
                qe--;
                step++;
                continue;
            }
            if (kind == 1) {
                double* w = S.wk;
                if (j != k) {
                    do_swap<NB, TH>(S, RS, F, ld, q, kp, k + 1, k, j, A.perm);
                    if (tid == 0) { const double x = S.wr[k - kp]; S.wr[k - kp] = S.wr[j - kp]; S.wr[j - kp] = x; }
                    __syncthreads();
                    w = S.wr;
                }
                const double d = w[k - kp];
                const double dinv = 1.0 / d;
                for (int i = k + 1 + tid; i < q; i += TH) S.Ls[(size_t)t * RS + (i - kp)] = w[i - kp] * dinv;
                if (tid == 0) {
                    S.cs[t] = d; S.co[t] = 0.0; S.oo[t] = 0; S.tp[t] = PK_1X1;
                    S.d1[t] = d; S.d2[t] = 0.0; S.fa[t] = fa; S.fb[t] = 0.0; S.st[t] = step;
                }
                __syncthreads();
                e += 1;
                step++;
            } else {
                do_swap<NB, TH>(S, RS, F, ld, q, kp, k + 2, k + 1, r, A.perm);
                if (tid == 0) {
                    double x = S.wk[k + 1 - kp]; S.wk[k + 1 - kp] = S.wk[r - kp]; S.wk[r - kp] = x;
                    x = S.wr[k + 1 - kp]; S.wr[k + 1 - kp] = S.wr[r - kp]; S.wr[r - kp] = x;
                }
                __syncthreads();
                const double d11 = S.wk[k - kp], d21 = S.wk[k + 1 - kp], d22 = S.wr[k + 1 - kp];
                const double det = d11 * d22 - d21 * d21;
                const double i11 = d22 / det, i21 = -d21 / det, i22 = d11 / det;
                for (int i = k + 2 + tid; i < q; i += TH) {
                    const double w1 = S.wk[i - kp], w2 = S.wr[i - kp];
                    S.Ls[(size_t)t * RS + (i - kp)] = w1 * i11 + w2 * i21;
                    S.Ls[(size_t)(t + 1) * RS + (i - kp)] = w1 * i21 + w2 * i22;
                }
                if (tid == 0) {
                    S.cs[t] = d11; S.co[t] = d21; S.oo[t] = 1; S.tp[t] = PK_2X2A;
                    S.cs[t + 1] = d22; S.co[t + 1] = d21; S.oo[t + 1] = -1; S.tp[t + 1] = PK_2X2B;
                    S.d1[t] = d11; S.d2[t] = d21; S.fa[t] = fa; S.fb[t] = fb;
                    S.d1[t + 1] = d22; S.d2[t + 1] = 0.0; S.fa[t + 1] = 0.0; S.fb[t + 1] = 0.0;
                    S.st[t] = step; S.st[t + 1] = step;
                }
                __syncthreads();
                e += 2;
                step++;
            }
        }
        // ---- commit the block: G11 = L11 M (FS rows), D and the test record (k_fsu: FS trailing update)
        const int nbn = e - kp;
        __syncthreads();                                     // the S1 loop is done with cs / co
        for (int t = warp; t < nbn; t += TH / 32) {
            const int cpos = kp + t;
            const int o = S.oo[t];
            if (lane == 0) {
                F[cpos + (size_t)cpos * ld] = S.d1[t];
                if (o == 1) F[cpos + 1 + (size_t)cpos * ld] = 0.0;      // unit L: D's 2x2 coupling is in the record
                A.d[cpos] = S.d1[t];
                A.ds[cpos] = S.d2[t];
                A.fa[cpos] = S.fa[t];
                A.fb[cpos] = S.fb[t];
                A.kind[cpos] = S.tp[t];
                A.step[cpos] = S.st[t];
                if (o == 0) {                                       // 1x1 (or zero): G = W sign(d) / sqrt|d|
                    const double dd = S.d1[t], sg = dd < 0.0 ? -1.0 : 1.0;
                    A.sgn[cpos] = sg;
                    A.gca[cpos] = S.tp[t] == PK_ZERO ? 0.0 : sg / sqrt(fabs(dd));
                    A.gcb[cpos] = 0.0;
                    S.cs[t] = S.tp[t] == PK_ZERO ? 0.0 : sqrt(fabs(dd));             // G = L sqrt|d|
                    S.co[t] = 0.0;
                } else if (o == 1) {                                // 2x2: G = W Q |Lambda|^-1/2 S
                    double cs, sn, l1, l2;
                    pair_eig(S.d1[t], S.d2[t], S.d1[t + 1], cs, sn, l1, l2);
                    const double s1 = l1 < 0.0 ? -1.0 : 1.0, s2 = l2 < 0.0 ? -1.0 : 1.0;
                    const double k1 = s1 / sqrt(fabs(l1)), k2 = s2 / sqrt(fabs(l2));
                    A.sgn[cpos] = s1;
                    A.sgn[cpos + 1] = s2;
                    A.gca[cpos] = cs * k1;      A.gcb[cpos] = sn * k1;        // G_t   = (W_t cs + W_t+1 sn) k1
                    A.gca[cpos + 1] = cs * k2;  A.gcb[cpos + 1] = -sn * k2;   // G_t+1 = (W_t+1 cs - W_t sn) k2
                    const double r1 = sqrt(fabs(l1)), r2 = sqrt(fabs(l2));   // G = L M, M = Q |Lambda|^1/2
                    S.cs[t] = cs * r1;          S.co[t] = sn * r1;
                    S.cs[t + 1] = cs * r2;      S.co[t + 1] = -sn * r2;
                }
            }
        }
        __syncthreads();
        for (int t = warp; t < nbn; t += TH / 32) {
            const int cpos = kp + t;
            const int o = S.oo[t];
            const int i1 = cpos + 1 + (o == 1 ? 1 : 0);
            const double* Lt = S.Ls + (size_t)t * RS - kp;
            const double* Lo = S.Ls + (size_t)(t + o) * RS - kp;
            const double ca = S.cs[t], cb = S.co[t];
            for (int i = i1 + lane; i < q; i += 32) F[i + (size_t)cpos * ld] = Lt[i] * ca + (o ? Lo[i] * cb : 0.0);
        }
        __syncthreads();
    }
    if (tid == 0) {
        fst[0] = e; fst[1] = qe; fst[2] = step; fst[3] = fnext; fst[4] = kp; fst[5] = 1;   // update pending
        if (e >= qe) nd_out[s] = q - e;
    }
}


// ------------------------------------------------------------------ k_fsu
// FS x FS trailing block [e, q)^2 (lower) -= L D L^T over the block [kp, e)
// committed by k_fsp = G S G^T with G = L M (stored), S = diag(+-1).
// One CTA per 64 x 64 tile (tiles anchored at the current e).
constexpr int UT = 128;
constexpr int UK = 32;          // >= any NB
constexpr int UPA = 64 + 4;     // = 4 (mod 16)

__global__ void __launch_bounds__(UT) k_fsu(DevPlan P, const int4* __restrict__ items) {
    __shared__ __align__(16) double As[UK][UPA];     // L[i, t]   (t-major)
    __shared__ __align__(16) double Bs[64][UK + 4];  // W[j, t] = (L D)[j, t]
    const int4 it = items[blockIdx.x];
    const int s = it.x, I = it.y, J = it.z;
    const int sh = blockIdx.y;
    if (P.flag[(size_t)sh * P.nf + s] != FL_ACTIVE) return;
    const int32_t* fst = P.fstate + ((size_t)sh * P.nf + s) * FSTATE_W;
    if (fst[5] != 1) return;                              // no block committed since the last update
    const int e = fst[0], kp = fst[4];
    const int K = e - kp;
    if (K <= 0) return;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int q = p + nd, ld = ldpad(P.cap[s]);
    const int i0 = e + 64 * I, j0 = e + 64 * J;
    if (i0 >= q) return;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    for (int x = tid; x < UK * 64; x += UT) {
        const int t = x >> 6, ii = x & 63;
        const bool vt = t < K;
        const int gi = i0 + ii, gj = j0 + ii;
        As[t][ii] = (vt && gi < q) ? F[gi + (size_t)(kp + t) * ld] : 0.0;
        double w = 0.0;
        if (vt && gj < q) w = F[gj + (size_t)(kp + t) * ld] * A.sgn[kp + t];    // (G S)[j, t]
        Bs[ii][t] = w;
    }
    __syncthreads();
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int k4 = 0; k4 < K; k4 += 4) {
        double a[4], b[4];
#pragma unroll
        for (int mb = 0; mb < 4; ++mb) a[mb] = As[k4 + tg][wm + 8 * mb + g];
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) b[nb] = Bs[wn + 8 * nb + g][k4 + tg];
#pragma unroll
        for (int mb = 0; mb < 4; ++mb)
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb], a[mb], b[nb]);
    }
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = i0 + wm + 8 * mb + g;
                const int j = j0 + wn + 8 * nb + 2 * tg + h;
                if (i < q && j < q && i >= j) atomicAdd(&F[i + (size_t)j * ld], -acc[mb][nb][h]);   // one writer: RED
            }
}

// ------------------------------------------------------------------ k_l21
// W21 = A21 P^T L11^-T for 64 CB rows of one front; column maxima of W21.
// L11[i,t] = 0 for t >= e (delayed columns have no pivot: their W21 column
// is the fully updated CB part of the delayed column).
// MODE 0: in-block solve by the paired-thread triangle (below).
// MODE 1 (SMALL): fronts with q < LB (one column block, no GEMM, compact shared memory).
// MODE 2 (XM): the in-block solve as a second DMMA GEMM with the block's precomputed
//   X = [L_bb^-T | L_bb^-T D^-1 M] (k_l21x_prep): [W | G] = R X with R = A21 P^T - G_prev B'_prev^T.
template <int MODE>
__global__ void __launch_bounds__(LT, 2) k_l21(DevPlan P, const int4* __restrict__ items) {
    constexpr bool SMALL = MODE == 1, XM = MODE == 2;
    extern __shared__ __align__(16) double l21_smem[];
    constexpr int OFF_S = SMALL ? 0 : LST * LR * BP + LST * LB * BP;
    double (*As)[LR][BP] = reinterpret_cast<double (*)[LR][BP]>(l21_smem);                       // [LST][LR][BP] rows x t
    double (*Bs)[LB][BP] = reinterpret_cast<double (*)[LB][BP]>(l21_smem + LST * LR * BP);        // [LST][LB][BP]
    double (*Sbase)[LB + 1] = reinterpret_cast<double (*)[LB + 1]>(l21_smem + OFF_S);
    static_assert(LR * (LB + 1) <= LST * LR * BP, "Sacc aliases As");
    static_assert(LB * (LB + 1) <= LST * LB * BP, "Lbb aliases Bs");
    double (*Sacc)[LB + 1] = reinterpret_cast<double (*)[LB + 1]>(l21_smem);
    double (*Lbb)[LB + 1] = reinterpret_cast<double (*)[LB + 1]>(l21_smem + (SMALL ? LR * (LB + 1) : LST * LR * BP));
    __shared__ int sperm[LB];
    __shared__ unsigned long long SgB[LST][KC];          // sign bits of B' = G11 S for the K chunks
    __shared__ int skind[LB];                             // pivot kind of the block columns (-1: delayed / none)
    __shared__ double sgca[LB], sgcb[LB];
    __shared__ double cmx[4][LB];                         // XM: column maxima of |W| per 32-row slice
    const int4 it = items[blockIdx.x];
    const int s = it.x, I = it.y;
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    if (P.flag[(size_t)sh * P.nf + s] != FL_ACTIVE) return;
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    if (ndo < 0) return;
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int e = q - ndo;
    const int r0 = q + I * LR;
    if (r0 >= f) return;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const int Q = P.cap[s] - c;
    AuxRec A = aux_rec(P, sh, s, Q);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int wm = warp * 16;
    const int row = tid >> 1, half = tid & 1;               // triangle: two threads per CB row
    const double* Xg = XM ? P.xscr + (size_t)sh * P.xstride + P.xoff[s] : nullptr;
    for (int b0 = 0, nbc = 0, blk = 0; b0 < q; b0 += nbc, ++blk) {
        nbc = min(LB, q - b0);
        if (nbc == LB && b0 + LB - 1 < e && A.kind[b0 + LB - 1] == PK_2X2A) nbc = LB - 1;   // keep 2x2 pairs whole
        const int K = SMALL ? 0 : min(b0, e);
        if (SMALL && b0 > 0) return;    // unreachable: the host routes only q < LB here (one block)
        if (tid < LB) {
            const int t = b0 + tid;
            sperm[tid] = tid < nbc ? A.perm[t] : 0;
            const bool el = tid < nbc && t < e;
            skind[tid] = el ? A.kind[t] : -1;
            sgca[tid] = el ? A.gca[t] : 0.0;
            sgcb[tid] = el ? A.gcb[t] : 0.0;
        }
        __syncthreads();
        // gathered A21 columns of the block (A21 P^T), fetched while the GEMM runs
        for (int x = tid; x < LB * LR; x += LT) {
            const int t = x / LR, ii = x - t * LR;
            const int gi = r0 + ii;
            const bool v = gi < f && t < nbc;
            cp_async8(&Sbase[ii][t], F + (v ? (gi + (size_t)sperm[t] * ld) : 0), v);
        }
        cp_async_commit();
        double acc[2][4][2];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) acc[mb][nb][0] = acc[mb][nb][1] = 0.0;
        if (!SMALL && K > 0) {
            // per-thread copy slots (fixed for the CTA): A: rows ii0 + 32 j (j < 4), columns 2 ta,
            // ta + 1 of the chunk; B: column jb of the block, chunk rows tb + 8 j (j < 2)
            static_assert((KC / 2) * LR == 4 * LT && KC * LB == 2 * LT, "k_l21 copy slots");
            const int ta = 2 * (tid % (KC / 2)), ii0 = tid / (KC / 2);
            const int jb = tid % LB, tb = tid / LB;
            auto load = [&](int buf, int t0) {
                const int gt = t0 + ta;
                const int nbt = gt + 1 < K ? 16 : (gt < K ? 8 : 0);
#pragma unroll
                for (int j = 0; j < 4; ++j) {                 // G rows: 16-byte pairs (even ld, t0 % 16 == 0)
                    const int ii = ii0 + 32 * j, gi = r0 + ii;
                    const int nb = gi < f ? nbt : 0;
                    cp_async16(&As[buf][ii][ta], F + (nb ? (gt + (size_t)gi * ld) : 0), nb);
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int tt = tb + 8 * j, gtb = t0 + tt;
                    const bool v = jb < nbc && gtb < K;
                    cp_async8(&Bs[buf][jb][tt], F + (v ? ((b0 + jb) + (size_t)gtb * ld) : 0), v);
                }
                if (tid < KC) SgB[buf][tid] = (t0 + tid < K && A.sgn[t0 + tid] < 0.0) ? 0x8000000000000000ull : 0ull;
                cp_async_commit();
            };
            const int nk = (K + KC - 1) / KC;
#pragma unroll
            for (int st0 = 0; st0 < LST - 1; ++st0) {
                if (st0 < nk) load(st0, st0 * KC);
                else cp_async_commit();
            }
            for (int kc = 0; kc < nk; ++kc) {
                const int buf = kc % LST;
                cp_async_wait<LST - 2>();
                __syncthreads();                    // chunk kc landed (and the gathered columns)
                {
                    const int nx = kc + LST - 1;
                    if (nx < nk) load(nx % LST, nx * KC);
                    else cp_async_commit();
                }
#pragma unroll
                for (int k4 = 0; k4 < KC; k4 += 4) {
                    double a[2], b[4];
#pragma unroll
                    for (int mb = 0; mb < 2; ++mb) a[mb] = As[buf][wm + 8 * mb + g][k4 + tg];
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb)
                        b[nb] = __longlong_as_double(__double_as_longlong(Bs[buf][8 * nb + g][k4 + tg]) ^ (long long)SgB[buf][k4 + tg]);
#pragma unroll
                    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                        for (int nb = 0; nb < 4; ++nb) dmma(acc[mb][nb], a[mb], b[nb]);
                }
            }
            cp_async_wait<0>();
            __syncthreads();                        // all chunks consumed before Sacc aliases As
        } else {
            cp_async_wait<0>();
            __syncthreads();
        }
        if (XM) {
            constexpr int XP = LB + 4;                          // = 4 (mod 16): conflict-free f64 fragments
            static_assert(LR * XP + 2 * LB * XP <= LST * LR * BP, "R and X alias As");
            double (*Rs)[XP] = reinterpret_cast<double (*)[XP]>(l21_smem);
            double (*Xs)[XP] = reinterpret_cast<double (*)[XP]>(l21_smem + LR * XP);
            const double* xb = Xg + (size_t)blk * (2 * LB * LB);
            for (int x = tid; x < 2 * LB * (LB / 2); x += LT) {    // X block [n][k], 64 x 32
                const int n = x / (LB / 2), k2 = 2 * (x - n * (LB / 2));
                cp_async16(&Xs[n][k2], xb + n * LB + k2, 16);
            }
            cp_async_commit();
#pragma unroll
            for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int rr = wm + 8 * mb + g, cc = 8 * nb + 2 * tg + h;
                        Rs[rr][cc] = Sbase[rr][cc] - acc[mb][nb][h];
                    }
            cp_async_wait<0>();
            __syncthreads();
            const int wm2 = (warp >> 1) * 32, wn2 = (warp & 1) * 32;     // 4 x 2 warps of 32 x 32
            double acc2[4][4][2];
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) acc2[mb][nb][0] = acc2[mb][nb][1] = 0.0;
#pragma unroll
            for (int k4 = 0; k4 < LB; k4 += 4) {
                double a[4], b[4];
#pragma unroll
                for (int mb = 0; mb < 4; ++mb) a[mb] = Rs[wm2 + 8 * mb + g][k4 + tg];
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) b[nb] = Xs[wn2 + 8 * nb + g][k4 + tg];
#pragma unroll
                for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) dmma(acc2[mb][nb], a[mb], b[nb]);
            }
            if (wn2 == 0) {                                     // W: column maxima (threshold tests, k_check)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        double m = 0.0;
#pragma unroll
                        for (int mb = 0; mb < 4; ++mb) m = fmax(m, fabs(acc2[mb][nb][h]));
                        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
                        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 8));
                        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 16));
                        if (g == 0) cmx[wm2 / 32][8 * nb + 2 * tg + h] = m;
                    }
            } else {                                            // G rows to the upper part
#pragma unroll
                for (int mb = 0; mb < 4; ++mb) {
                    const int i = r0 + wm2 + 8 * mb + g;
                    if (i >= f) continue;
                    double* __restrict__ Gi = F + (size_t)i * ld + b0;
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int t = 8 * nb + 2 * tg + h;
                            if (t < nbc) Gi[t] = acc2[mb][nb][h];
                        }
                }
            }
            __syncthreads();
            if (tid < LB) {
                const double m = fmax(fmax(cmx[0][tid], cmx[1][tid]), fmax(cmx[2][tid], cmx[3][tid]));
                if (tid < nbc && b0 + tid < e && m > 0.0)
                    atomicMax(&A.cm[b0 + tid], (unsigned long long)__double_as_longlong(m));
            }
            __syncthreads();                                    // Rs / Xs (As) and Sbase free for the next block
            continue;
        }
        if (!SMALL) {
#pragma unroll
            for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) Sacc[wm + 8 * mb + g][8 * nb + 2 * tg + h] = acc[mb][nb][h];
        }
        // diagonal block of B' = L11 D M^-T = G11 S (strict lower, columns < e only)
        for (int x = tid; x < LB * LB; x += LT) {           // consecutive threads walk a column (coalesced)
            const int b = x / LB, a = x - b * LB;
            double v = 0.0;
            if (a < nbc && b < a && b0 + b < e) v = F[(b0 + a) + (size_t)(b0 + b) * ld] * A.sgn[b0 + b];   // B' = G S
            Lbb[a][b] = v;
        }
        __syncthreads();
        {   // in-block solve in G space: x_t = A_t - sum_{t' < t} G_t' B'[t, t'] (G of the block's earlier
            // columns; a 2x2 pair's G is formed when its second column is known).  Thread pair
            // (row, parity) splits each dot product.
            const int i = r0 + row;
            const bool valid = i < f;
            double gh[LB / 2], ah[LB / 2];                   // own-parity columns: G (raw for delayed), |W21|
            double vprev = 0.0;
#pragma unroll
            for (int t = 0; t < LB; ++t) {
                if (t >= nbc) break;                         // (uniform)
                double p0 = 0.0, p1 = 0.0;
#pragma unroll
                for (int u = 0; 2 * u + half < t && u < LB / 2; u += 2) {
                    p0 = fma(gh[u], Lbb[t][2 * u + half], p0);
                    if (2 * (u + 1) + half < t) p1 = fma(gh[u + 1], Lbb[t][2 * (u + 1) + half], p1);
                }
                const double part = p0 + p1;
                const double tot = part + __shfl_xor_sync(0xffffffffu, part, 1);
                double v = SMALL ? Sbase[row][t] - tot : Sbase[row][t] - Sacc[row][t] - tot;
                v = (t < nbc && valid) ? v : 0.0;
                const int kd = skind[t];
                const bool own = (t & 1) == half;
                if (own) { ah[t >> 1] = fabs(v); gh[t >> 1] = v; }
                if (kd == PK_1X1 || kd == PK_ZERO) {
                    if (own) gh[t >> 1] = v * sgca[t];
                } else if (kd == PK_2X2B && t > 0) {
                    if (own) gh[t >> 1] = v * sgca[t] + vprev * sgcb[t];
                    else gh[(t - 1) >> 1] = vprev * sgca[t - 1] + v * sgcb[t - 1];
                }
                vprev = v;
            }
            if (valid) {
                double* __restrict__ Wi = F + (size_t)i * ld + b0;
#pragma unroll
                for (int u = 0; u < LB / 2; ++u)
                    if (2 * u + half < nbc) Wi[2 * u + half] = gh[u];
            }
            __syncwarp();                                    // both threads of the row are done with Sbase
#pragma unroll
            for (int u = 0; u < LB / 2; ++u) Sbase[row][2 * u + half] = valid ? ah[u] : 0.0;
        }
        __syncthreads();
        {   // CB column maxima of W21 (threshold tests, k_check): 8 threads per column, 16 rows each
            const int t = tid >> 3, part = tid & 7;
            double m = 0.0;
#pragma unroll
            for (int r = 0; r < LR / 8; ++r) m = fmax(m, Sbase[part * (LR / 8) + r][t]);
            m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
            m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
            m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
            if (part == 0 && t < nbc && b0 + t < e && m > 0.0)
                atomicMax(&A.cm[b0 + t], (unsigned long long)__double_as_longlong(m));
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ k_l21d
// G21 = W21 D^-1 M for the 128 CB rows i of one strip, by plain forward substitution
// along each row (fronts with FS capacity <= QMAX):
//   w_t = a_t - sum_{t' < min(t, e)} (g_t' s_t') G11[t, t'],   a_t = (A21 P^T)[i, t],
// i.e. W21 = A21 P^T L11^-T written in G space (B' = G11 S, R21), then
// g_t from w_t and its 2x2 partner (gca / gcb), |w_t| into the column maxima.
// One row per thread (TPR = 1) or per TPR adjacent threads (TPR = 4: the group splits
// the columns by t mod 4 and adds its partial sums with two shuffles).  The row's
// history g S stays in registers (QMAX / TPR of them); B' rows are streamed through
// shared memory in chunks of LDC rows (double-buffered cp.async, zero-filled for
// t' >= e and at a 2x2 block's in-pair entry) and read as 16-byte broadcasts.
// All arithmetic is fp64 FMA (on B200 the FMA pipe matches DMMA: 33.8 vs 35.5
// TFLOP/s measured), no explicit block inverses, no CTA barrier except per chunk.
template <int QMAX, int TPR>
struct L21d {
    static constexpr int NT = 128 * TPR, NW = NT / 32, NWS = NW < 8 ? NW : 8, LDC = 16, NH = QMAX / TPR;
    static constexpr int BW = NH + 2;                     // B' row (per class t' mod TPR) + pad, 16-byte aligned
    static_assert(QMAX % (2 * TPR) == 0 && LDC % 2 == 0 && QMAX % 64 == 0, "k_l21d shape");
    struct Smem {
        double Bs[2][LDC][TPR][BW];                       // B'[t0 + r][TPR k + h] at Bs[.][r][h][k]
        unsigned long long scm[NWS][QMAX];                // warp maxima of |w_t| (warps w, w + 8 share a row)
        double ssg[QMAX], sga[QMAX], sgb[QMAX];
        int sperm[QMAX], skind[QMAX];
    };
    Smem& S;
    const double* F;
    int q, e, ld, tid, lane, warp, h;
    bool valid;
    double vprev;

    // B' rows [t0, t0 + LDC), all QMAX columns (zeros outside the strict lower part below e, so the
    // unrolled dot products may read past their last term)
    __device__ __forceinline__ void stage(int buf, int t0) {
        for (int x = tid; x < LDC * QMAX; x += NT) {
            const int r = x % LDC, tp = x / LDC, t = t0 + r;   // consecutive threads walk a column of G11
            const bool v = t < q && tp < t && tp < e && !(tp == t - 1 && S.skind[tp] == PK_2X2A);
            cp_async8(&S.Bs[buf][r][tp % TPR][tp / TPR], F + (v ? (t + (size_t)tp * ld) : 0), v);
        }
        cp_async_commit();
    }

    // columns [T0, T0 + 64) of the substitution (64 per part keeps every loop fully unrolled,
    // so y[] stays in registers); false once t reaches q
    template <int T0>
    __device__ __forceinline__ bool part(double (&y)[NH]) {
        // Straight-line code per chunk of LDC columns (no data-dependent branches: the scheduler
        // overlaps the dot products of consecutive t, which share only their last terms); columns
        // t >= q inside the last chunk compute zeros (a_t = 0, B' = 0, kind -1) and are not stored.
#pragma unroll
        for (int t = T0; t < T0 + 64; ++t) {
            if (t % LDC == 0) {
                if (t >= q) return false;                  // uniform
                cp_async_wait<0>();
                __syncthreads();                           // chunk t / LDC landed; the other buffer is free
                if (t + LDC < q) stage((t / LDC + 1) & 1, t + LDC);
            }
            const double* b = &S.Bs[(t / LDC) & 1][t % LDC][h][0];
            double a[4] = {0.0, 0.0, 0.0, 0.0};
            const int kend = (t - h + TPR - 1) / TPR;      // own columns t' = TPR k + h < t
#pragma unroll
            for (int k = 0; k < NH; k += 2) {
                if (k >= (t + TPR - 1) / TPR) break;       // static bound (h = 0)
                const double2 bb = *reinterpret_cast<const double2*>(b + k);
                if (TPR == 1) {                            // kend = t: static
                    if (k < kend) a[(k >> 1) & 1] = fma(y[k], bb.x, a[(k >> 1) & 1]);
                    if (k + 1 < kend) a[2 + ((k >> 1) & 1)] = fma(y[k + 1], bb.y, a[2 + ((k >> 1) & 1)]);
                } else {
                    a[(k >> 1) & 1] = fma(k < kend ? y[k] : 0.0, bb.x, a[(k >> 1) & 1]);
                    a[2 + ((k >> 1) & 1)] = fma(k + 1 < kend ? y[k + 1] : 0.0, bb.y, a[2 + ((k >> 1) & 1)]);
                }
            }
            double tot = (a[0] + a[1]) + (a[2] + a[3]);
            if (TPR >= 2) tot += __shfl_xor_sync(0xffffffffu, tot, 1);
            if (TPR >= 4) tot += __shfl_xor_sync(0xffffffffu, tot, 2);
            double v = (t % TPR == h ? y[t / TPR] : 0.0) - tot;
            if (TPR >= 2) v = __shfl_sync(0xffffffffu, v, (lane & ~(TPR - 1)) | (t % TPR));
            const int kd = S.skind[t];
            {   // |w_t| into the column maxima (read back only for t < e)
                const double av = valid ? fabs(v) : 0.0;
                const unsigned hi = (unsigned)__double2hiint(av), lo = (unsigned)__double2loint(av);
                const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
                const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
                const unsigned long long mv = ((unsigned long long)mh << 32) | ml;
                if (NW <= 8) {
                    if (lane == 0) S.scm[warp][t] = mv;
                } else {
                    if (lane == 0 && warp < 8) S.scm[warp][t] = mv;
                    __syncwarp();
                    if (lane == 0 && warp >= 8) atomicMax(&S.scm[warp - 8][t], mv);
                }
            }
            const double ga = S.sga[t], gb = S.sgb[t], sg = S.ssg[t];
            const bool two = t > 0 && kd == PK_2X2B;
            // g_t s_t: 1x1 / zero pivot, second column of a 2x2 pair, or raw w_t (delayed; first of a pair)
            const double g = (kd == PK_1X1 || kd == PK_ZERO) ? v * ga * sg
                           : (two ? (v * ga + vprev * gb) * sg : v);
            if (t % TPR == h) y[t / TPR] = g;
            if (t > 0 && (t - 1) % TPR == h) {             // the pair's first column, now complete
                const int tm = t > 0 ? t - 1 : 0;
                const double g1 = (vprev * S.sga[tm] + v * S.sgb[tm]) * S.ssg[tm];
                y[tm / TPR] = two ? g1 : y[tm / TPR];
            }
            vprev = v;
        }
        return true;
    }
};

template <int QMAX, int TPR>
__global__ void __launch_bounds__(128 * TPR) k_l21d(DevPlan P, const int4* __restrict__ items) {
    using K = L21d<QMAX, TPR>;
    constexpr int NT = K::NT, NH = K::NH;
    __shared__ __align__(16) typename K::Smem S;
    const int4 it = items[blockIdx.x];
    const int s = it.x, I = it.y;
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    if (P.flag[(size_t)sh * P.nf + s] != FL_ACTIVE) return;
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    if (ndo < 0) return;
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int e = q - ndo;
    const int r0 = q + I * 128;
    if (r0 >= f || q > QMAX) return;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    const int tid = threadIdx.x;
    K k{S, F, q, e, ld, tid, tid & 31, tid >> 5, tid & (TPR - 1), r0 + tid / TPR < f, 0.0};
    const int i = r0 + tid / TPR;
    for (int t = tid; t < QMAX; t += NT) {
        const bool el = t < e;
        S.sperm[t] = t < q ? A.perm[t] : 0;
        S.skind[t] = el ? A.kind[t] : -1;
        S.ssg[t] = el ? A.sgn[t] : 0.0;
        S.sga[t] = el ? A.gca[t] : 0.0;
        S.sgb[t] = el ? A.gcb[t] : 0.0;
    }
    __syncthreads();
    k.stage(0, 0);
    double y[NH];                                          // a_t, then g_t s_t (raw w_t for delayed t)
#pragma unroll
    for (int x = 0; x < NH; ++x) {
        const int t = TPR * x + k.h;
        y[x] = (k.valid && t < q) ? F[i + (size_t)S.sperm[t] * ld] : 0.0;
    }
    if (k.template part<0>(y) && QMAX > 64) k.template part<(QMAX > 64 ? 64 : 0)>(y);
    if (k.valid) {                                         // G (W for delayed columns) to the upper part
        double* __restrict__ Gi = F + (size_t)i * ld;
#pragma unroll
        for (int x = 0; x < NH; ++x) {
            const int t = TPR * x + k.h;
            if (t < q) Gi[t] = S.skind[t] >= 0 ? y[x] * S.ssg[t] : y[x];
        }
    }
    __syncthreads();
    for (int t = tid; t < e; t += NT) {
        unsigned long long m = 0;
#pragma unroll
        for (int w = 0; w < K::NWS; ++w) m = max(m, S.scm[w][t]);
        if (m > 0) atomicMax(&A.cm[t], m);
    }
}

// ------------------------------------------------------------------ k_l21x_prep
// Per front and column block [b0, b0 + nbc) of k_l21 (the same block rule): the
// unit lower block L_bb of L11 (from the stored G11 = L11 M: L = G11 S (D M^-T)^-1,
// as in k_store), its inverse by forward substitution (one lane per column), and
//   X[n][k] = L_bb^-1[n][k]                               n < 32   (W = R L_bb^-T)
//   X[32 + t][k] = L_bb^-1[t][k] gca[t] + L_bb^-1[t'][k] gcb[t]     (G = W D^-1 M,
//                  t' the 2x2 partner; delayed columns: G = W)
// stored [n][k] (k contiguous) in the level's X scratch for k_l21<2>.
__global__ void __launch_bounds__(XPW * 32) k_l21x_prep(DevPlan P, const int32_t* __restrict__ fronts) {
    extern __shared__ double xp_smem[];                   // [XPW][LB][LB + 1]
    __shared__ int sb0[kXMaxBlocks], snb[kXMaxBlocks];
    __shared__ int s_nblk;
    const int s = fronts[blockIdx.x];
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    if (P.flag[(size_t)sh * P.nf + s] != FL_ACTIVE) return;
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    if (ndo < 0) return;
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int e = q - ndo;
    const double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    double* X = P.xscr + (size_t)sh * P.xstride + P.xoff[s];
    if (threadIdx.x == 0) {
        int nb = 0;
        for (int b0 = 0, nbc = 0; b0 < q && nb < kXMaxBlocks; b0 += nbc) {
            nbc = min(LB, q - b0);
            if (nbc == LB && b0 + LB - 1 < e && A.kind[b0 + LB - 1] == PK_2X2A) nbc = LB - 1;   // as k_l21
            sb0[nb] = b0; snb[nb] = nbc; ++nb;
        }
        s_nblk = nb;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double (*Lw)[LB + 1] = reinterpret_cast<double (*)[LB + 1]>(xp_smem + (size_t)warp * LB * (LB + 1));
    // L[i][t] for a pivot column t < e (rows i > t of the block): from B' = G11 S
    auto lval = [&](int i, int t) -> double {
        const int kd = A.kind[t];
        double v = F[i + (size_t)t * ld] * A.sgn[t] * A.gca[t];
        if (kd == PK_2X2A) v = (i == t + 1) ? 0.0 : v + F[i + (size_t)(t + 1) * ld] * A.sgn[t + 1] * A.gcb[t + 1];
        else if (kd == PK_2X2B) v += F[i + (size_t)(t - 1) * ld] * A.sgn[t - 1] * A.gcb[t - 1];
        else if (kd == PK_ZERO) v = 0.0;
        return v;
    };
    for (int bk = warp; bk < s_nblk; bk += XPW) {
        const int b0 = sb0[bk], nbc = snb[bk];
        for (int x = lane; x < LB * LB; x += 32) {         // strict lower L_bb (zero elsewhere)
            const int b = x / LB, a = x - b * LB;           // column b, row a (lanes walk a column)
            Lw[a][b] = (a < nbc && b < a && b0 + b < e) ? lval(b0 + a, b0 + b) : 0.0;
        }
        __syncwarp();
        // lane j: column j of L_bb^-1 (unit lower), kept transposed in the upper part: Y[t][j] -> Lw[j][t]
        {
            const int j = lane;
            for (int t = j + 1; t < nbc; ++t) {
                double acc = Lw[t][j];                      // Y[j][j] = 1
                for (int u = j + 1; u < t; ++u) acc = fma(Lw[t][u], Lw[j][u], acc);
                Lw[j][t] = -acc;
            }
        }
        __syncwarp();
        auto yinv = [&](int n, int k) -> double {           // L_bb^-1[n][k]
            if (n >= nbc || k >= nbc) return 0.0;
            return n == k ? 1.0 : (n > k ? Lw[k][n] : 0.0);
        };
        double* xb = X + (size_t)bk * (2 * LB * LB);
        for (int n = 0; n < 2 * LB; ++n) {
            const int k = lane;
            double v;
            if (n < LB) v = yinv(n, k);
            else {
                const int t = n - LB;
                if (t >= nbc) v = 0.0;
                else if (b0 + t >= e) v = yinv(t, k);       // delayed column: G = W
                else {
                    const int kd = A.kind[b0 + t];
                    v = yinv(t, k) * A.gca[b0 + t];
                    if (kd == PK_2X2A) v += yinv(t + 1, k) * A.gcb[b0 + t];
                    else if (kd == PK_2X2B) v += yinv(t - 1, k) * A.gcb[b0 + t];
                }
            }
            xb[n * LB + k] = v;
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ k_rerun_lists
// Between fast-path passes of a level (one CTA): the fronts flagged FL_RERUN in any
// shift of the batch and their tiles of every per-front list, so the rerun pass
// launches grids over those fronts only (≈1 % of a level) instead of the whole level.
__global__ void __launch_bounds__(1024) k_rerun_lists(DevPlan P, const int32_t* __restrict__ fl, int n, int batch,
                                                      RerunLists R) {
    __shared__ int cnt[8];
    if (threadIdx.x < 8) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int x = threadIdx.x; x < n; x += blockDim.x) {
        const int s = fl[x];
        bool fg = false, fa = false;                    // flagged for a rerun / for a rerun or the unblocked kernel
        for (int sh = 0; sh < batch; ++sh) {
            int32_t* fp = P.flag + (size_t)sh * P.nf + s;
            const int32_t v = *fp;
            fg |= v == FL_RERUN;
            fa |= v == FL_RERUN || v == FL_REFN;         // newly flagged by this pass only
            if (v == FL_REFN) *fp = FL_REF;
        }
        if (!fa) continue;
        const int4 a = R.d1[s], b = R.d2[s];           // (l21 mode, l21 off, l21 cnt, uitem off), (ucnt, aoff, acnt, -)
        int k;
        if (b.z > 0) {                                  // re-assembly (restore) of every flagged front
            k = atomicAdd(&cnt[5], b.z);
            for (int i = 0; i < b.z; ++i) R.a[k + i] = R.sa[b.y + i];
        }
        if (!fg) continue;
        k = atomicAdd(&cnt[0], 1);
        R.fr[k] = s;
        if (a.z > 0) {
            k = atomicAdd(&cnt[a.x < 3 ? 1 + a.x : 7], a.z);
            for (int i = 0; i < a.z; ++i) R.l[a.x][k + i] = R.sl[a.x][a.y + i];
        }
        if (b.x > 0) {
            k = atomicAdd(&cnt[4], b.x);
            for (int i = 0; i < b.x; ++i) R.u[k + i] = R.su[a.w + i];
        }
        if (a.x == 2) {
            k = atomicAdd(&cnt[6], 1);
            R.x[k] = s;
        }
    }
    __syncthreads();
    if (threadIdx.x < 8) R.cnt[threadIdx.x] = cnt[threadIdx.x];
}

// ------------------------------------------------------------------ k_check
__global__ void __launch_bounds__(FT) k_check(DevPlan P, const int32_t* __restrict__ fronts) {
    __shared__ int s_ok;
        const int s = fronts[blockIdx.x];
    const int sh = blockIdx.y;
    const int nd = P.nd_in[(size_t)sh * P.nf + s];
    if (nd < 0) return;
    int32_t* flag = P.flag + (size_t)sh * P.nf + s;
    if (*flag != FL_ACTIVE) return;
    __shared__ int s_fail;
    const int ndo = P.nd_out[(size_t)sh * P.nf + s];
    const int p = P.npiv[s], c = P.ncb[s];
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const int e = q - ndo;
    const bool root = c == 0;
    double* F = P.arena + (size_t)sh * P.arena_stride + P.arena_off[s];
    const int Q = P.cap[s] - c;
    AuxRec A = aux_rec(P, sh, s, Q);
    ShiftStat* st = P.stats + sh;
    const double u = P.u;
    const int tid = threadIdx.x;
    // every pivot's test in parallel (the tests are independent given the stored maxima);
    // the first failure in pivot order is a block-wide min, the inertia a block-wide sum
    __shared__ int s_first;
    __shared__ unsigned long long s_cnt[4];
    __shared__ unsigned long long s_minb;
    if (tid == 0) { s_first = INT_MAX; s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0ull; s_minb = ~0ull; }
    __syncthreads();
    unsigned long long c_neg = 0, c_zero = 0, c_pos = 0, c_2x2 = 0;
    double minpiv = DBL_MAX;
    int first = INT_MAX;
    for (int t = tid; t < e; t += FT) {
        const int kd = A.kind[t];
        if (kd == PK_2X2B) continue;                      // tested with its first column
        const double ca = root ? 0.0 : __longlong_as_double((long long)A.cm[t]);
        bool ok = true;
        if (kd == PK_ZERO) {
            ok = ca == 0.0;
            c_zero++;
            minpiv = 0.0;
        } else if (kd == PK_1X1) {
            const double d = A.d[t];
            ok = root || fabs(d) >= u * fmax(A.fa[t], ca);
            if (d < 0.0) c_neg++; else if (d > 0.0) c_pos++; else c_zero++;
            minpiv = fmin(minpiv, fabs(d));
        } else {
            const double d11 = A.d[t], d21 = A.ds[t], d22 = A.d[t + 1];
            const double det = d11 * d22 - d21 * d21;
            if (!root) {
                const double cb = __longlong_as_double((long long)A.cm[t + 1]);
                const double gk = fmax(A.fa[t], ca), gr = fmax(A.fb[t], cb);
                if (det == 0.0) ok = false;
                else {
                    const double ad = fabs(det);
                    ok = (fabs(d22) * gk + fabs(d21) * gr) / ad <= 1.0 / u &&
                         (fabs(d21) * gk + fabs(d11) * gr) / ad <= 1.0 / u;
                }
            }
            const double tt = (d11 / d21) * (d22 / d21) - 1.0;
            if (tt < 0.0) { c_neg++; c_pos++; }
            else if (tt > 0.0) { if (d11 < 0.0) c_neg += 2; else c_pos += 2; }
            else { c_zero++; if (d11 + d22 < 0.0) c_neg++; else c_pos++; }
            const double tr = 0.5 * (d11 + d22);
            const double disc = sqrt(0.25 * (d11 - d22) * (d11 - d22) + d21 * d21);
            const double big = fabs(tr) + disc;
            minpiv = fmin(minpiv, big > 0.0 ? fabs(det) / big : 0.0);
            c_2x2++;
        }
        if (!ok) {
            first = min(first, t);
            if (P.debug)
                printf("[kep] test fails: front %d shift %d pos %d kind %d d=%.3e ds=%.3e fa=%.3e fb=%.3e cm=%.3e\n",
                       s, sh, t, kd, A.d[t], A.ds[t], A.fa[t], A.fb[t], ca);
        }
    }
    if (first < INT_MAX) atomicMin(&s_first, first);
    if (c_neg) atomicAdd(&s_cnt[0], c_neg);
    if (c_zero) atomicAdd(&s_cnt[1], c_zero);
    if (c_pos) atomicAdd(&s_cnt[2], c_pos);
    if (c_2x2) atomicAdd(&s_cnt[3], c_2x2);
    if (minpiv < DBL_MAX) atomicMin(&s_minb, (unsigned long long)__double_as_longlong(minpiv));
    __syncthreads();
    if (tid == 0) {
        const bool ok = s_first == INT_MAX;
        s_ok = ok;
        s_fail = s_first;
        if (!ok && P.debug) printf("[kep] redo front %d shift %d: q=%d e=%d c=%d\n", s, sh, q, e, c);
        if (ok) {
            if (s_cnt[0]) atomicAdd(&st->n_neg, s_cnt[0]);
            if (s_cnt[1]) atomicAdd(&st->n_zero, s_cnt[1]);
            if (s_cnt[2]) atomicAdd(&st->n_pos, s_cnt[2]);
            if (s_cnt[3]) atomicAdd(&st->n_2x2, s_cnt[3]);
            if (ndo) atomicAdd(&st->n_delayed, (unsigned long long)ndo);
            if (s_minb != ~0ull) atomic_min_pos_double(&st->minpiv_bits, __longlong_as_double((long long)s_minb));
        }
    }
    __syncthreads();
    if (!s_ok) {
        // the front is assembled again next (k_assemble, flagged mode); then a rerun or the unblocked kernel
        if (tid == 0) {
            int32_t* forced = P.forced + ((size_t)sh * P.nf + s) * (FMAX + 1);
            const int nf_ = forced[0];
            if (nf_ < FMAX) {                                // rerun the fast path, delaying there
                forced[1 + nf_] = A.step[s_fail];
                forced[0] = nf_ + 1;
                *flag = FL_RERUN;
                atomicAdd(P.pending, 1);
                atomicMax(P.pending + 1, q);                 // largest FS block to rerun (iteration count)
            } else {
                *flag = FL_REFN;
            }
            atomicAdd(&st->n_redo, 1ull);
        }
        return;
    }
    if (tid == 0) *flag = FL_OK;
}

}  // namespace

constexpr size_t kFsSmemLimit = 200 * 1024;   // dynamic; + static shared stays under the 227 KB opt-in

int fs_rows_pad(int qmax) { return ((qmax + 15) / 16) * 16 + 4; }

// NB for a level whose fronts have at most qmax fully-summed columns (with
// slack): the widest block whose shared memory fits; 0 = too large.
bool fs_uses_gls(int qmax) { return fs_smem_bytes(8, fs_rows_pad(qmax), false) > kFsSmemLimit; }

int front_nb_for(int qmax, int64_t nblocks) {
    const int RS = fs_rows_pad(qmax);
    const size_t lim = kFsSmemLimit;
    if (fs_uses_gls(qmax)) return 16;                  // block columns in global scratch
    // NB = 32 halves the k_fsu passes but its Ls block (q x 32) halves the CTAs per SM: on full
    // levels only up to q = 256 (measured at c4: 256 > 384 > 512 > 640)
    const int q32 = nblocks < 4 * 148 ? 640 : 256;
    if (fs_smem_bytes(32, RS, false) <= lim && qmax <= q32) return 32;
    if (fs_smem_bytes(16, RS, false) <= lim) return 16;
    if (fs_smem_bytes(8, RS, false) <= lim) return 8;
    return 0;
}

int fs_iters(int qmax, int64_t nblocks) {
    const int nb = front_nb_for(qmax, nblocks);
    return nb > 1 ? (qmax + nb - 2) / (nb - 1) + 1 : 0;
}

template <int NB, int TH, bool GLS>
void launch_fsp_t(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int RS, size_t smem, int mode,
                  cudaStream_t st) {
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(k_fsp<NB, TH, GLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFsSmemLimit);
        
    }
    k_fsp<NB, TH, GLS><<<dim3(nfronts, batch), TH, smem, st>>>(P, fronts, RS, mode);
}

void launch_fsp(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int qmax, int mode, cudaStream_t st) {
    if (nfronts <= 0) return;
    const int nb = front_nb_for(qmax, (int64_t)nfronts * batch);
    const int RS = fs_rows_pad(qmax);
    const bool gls = fs_uses_gls(qmax);
    const size_t smem = fs_smem_bytes(nb, RS, gls);
    if (gls) return launch_fsp_t<16, 256, true>(P, fronts, nfronts, batch, RS, smem, mode, st);
    // threads per front: one warp for tiny FS blocks (no CTA-wide barriers), 4 or 8 warps above
    static const int q1 = [] { const char* x = getenv("KEP_FSP_Q1"); return x ? atoi(x) : 40; }();
    static const int q4 = [] { const char* x = getenv("KEP_FSP_Q4"); return x ? atoi(x) : 192; }();
    const int th = qmax <= q1 ? 32 : (qmax <= q4 ? 128 : 256);
#define KEP_FSP(NBV, THV) if (nb == NBV && th == THV) return launch_fsp_t<NBV, THV, false>(P, fronts, nfronts, batch, RS, smem, mode, st)
    KEP_FSP(32, 32); KEP_FSP(32, 128); KEP_FSP(32, 256);
    KEP_FSP(16, 32); KEP_FSP(16, 128); KEP_FSP(16, 256);
    KEP_FSP(8, 32); KEP_FSP(8, 128); KEP_FSP(8, 256);
#undef KEP_FSP
}

// Model of the k_fsp + k_fsu passes of one group of fronts (host planning of the
// per-level size buckets): launches x waves x block columns, + a launch overhead.
double fs_cost(int qmax, int64_t nblocks) {
    const int nb = front_nb_for(qmax, nblocks);
    if (nb <= 0) return 0.0;
    const int RS = fs_rows_pad(qmax);
    const bool gls = fs_uses_gls(qmax);
    const double smem = (double)fs_smem_bytes(nb, RS, gls) + 2048.0;
    const int th = gls ? 256 : (qmax <= 40 ? 32 : (qmax <= 192 ? 128 : 256));
    const int cps = std::max(1, std::min((int)(233472.0 / smem), 2048 / th));
    const double waves = std::ceil((double)nblocks / (148.0 * cps));
    const double iters = (double)fs_iters(qmax, nblocks);
    return iters * (waves * nb + 12.0);
}

void launch_fsu(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st) {
    if (nitems <= 0) return;
    k_fsu<<<dim3(nitems, batch), UT, 0, st>>>(P, items);
}

// FS capacity up to which k_l21d replaces k_l21 (KEP_L21D_MAX: 0 = off, 64 = default, 128: also
// k_l21d<128,4>, measured slower than k_l21<2> at c4)
int l21d_max() {
    static const int v = [] { const char* x = getenv("KEP_L21D_MAX"); return x ? atoi(x) : 64; }();
    return v;
}

void launch_l21(const DevPlan& P, const int4* items, int nitems, int batch, int mode, cudaStream_t st) {
    if (nitems <= 0) return;
    const size_t smem = sizeof(double) * (LST * LR * BP + LST * LB * BP + LR * (LB + 1));
    const size_t smem_s = sizeof(double) * (LR * (LB + 1) + LB * (LB + 1));
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(k_l21<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_l21<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s);
        cudaFuncSetAttribute(k_l21<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        
    }
    if (mode == 3) k_l21d<128, 4><<<dim3(nitems, batch), 512, 0, st>>>(P, items);
    else if (mode == 1 && l21d_max() >= 64) k_l21d<64, 1><<<dim3(nitems, batch), 128, 0, st>>>(P, items);
    else if (mode == 1) k_l21<1><<<dim3(nitems, batch), LT, smem_s, st>>>(P, items);
    else if (mode == 2) k_l21<2><<<dim3(nitems, batch), LT, smem, st>>>(P, items);
    else k_l21<0><<<dim3(nitems, batch), LT, smem, st>>>(P, items);
}

int l21_mode(int qcap) {
    const int dm = l21d_max();
    if (dm >= 64 && qcap <= 64) return 1;
    if (dm >= 128 && qcap <= 128) return 3;
    if (qcap < LB) return 1;
    if (qcap >= kXMin && qcap <= (LB - 1) * kXMaxBlocks) return 2;
    return 0;
}

int64_t l21_x_doubles(int qcap) { return (int64_t)2 * LB * LB * ((qcap + LB - 2) / (LB - 1)); }

void launch_l21x_prep(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, cudaStream_t st) {
    if (nfronts <= 0) return;
    const size_t smem = sizeof(double) * XPW * LB * (LB + 1);
    static unsigned long long attr = 0;
    if (first_on_device(attr)) { cudaFuncSetAttribute(k_l21x_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  }
    k_l21x_prep<<<dim3(nfronts, batch), XPW * 32, smem, st>>>(P, fronts);
}

void launch_rerun_lists(const DevPlan& P, const int32_t* fl, int n, int batch, const RerunLists& R, cudaStream_t st) {
    k_rerun_lists<<<1, 1024, 0, st>>>(P, fl, n, batch, R);
}

void launch_check(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, cudaStream_t st) {
    if (nfronts <= 0) return;
    k_check<<<dim3(nfronts, batch), FT, 0, st>>>(P, fronts);
}


}  // namespace kep
