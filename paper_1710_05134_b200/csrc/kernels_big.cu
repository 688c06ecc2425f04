// kernels_big.cu — row a3 (+ a5) of SURVEY.md §8 for the few large fronts of the
// top elimination-tree levels (c3 / c5 roots of 12k-30k fully-summed columns),
// where one CTA per front leaves almost every SM idle while the pivot loop runs.
//
// Each (front, shift) group gets ncta CTAs (all co-resident: cooperative launch);
// CTA j owns the rows [f j / ncta, f (j+1) / ncta) of the front.  The pivot rule
// is DESIGN.md reading R1 exactly as the oracle states it (oracle/sparse_mf.py,
// the blocked form _partial_fs_bk_blocked): Bunch-Kaufman among the
// FS candidates with the threshold test against the WHOLE current column, whose
// every row is formed here (no CB maxima to guess, no reruns); a root runs plain
// BK.  The FS columns are processed in blocks of BNB pivots:
//   k_bigp  (one launch per block) the current column k is formed on demand,
//           left-looking over the block's eliminated columns,
//               col_k[i] = F[i, k] - sum_t G[i, t] S_t G[k, t],   G = L M (R21),
//           group-wide (max, argmax) reductions through global partials and a
//           spin barrier, BK choice, threshold test, symmetric interchanges of
//           the front rows / columns, then the G column(s) of the pivot stored
//           in place (all rows) and D, kind, permutation, signs recorded;
//   k_bigu  the trailing update of the remaining FS columns (all rows) with the
//           block's G columns, F[i, j] -= sum_t G[i, t] S_t G[j, t] (DMMA tiles,
//           persistent over the level's groups);
//   k_bigfin the CB rows of G (eliminated columns) and of the updated delayed
//           columns (W21) are copied to the upper part F[t + i ld], the layout
//           k_schur and the parent's extend-add read (kernels_front.cu), and the
//           inertia counts are added to the shift's statistics.
// F holds, for the not-yet-eliminated columns, the values updated through the
// previous blocks ("raw" for the current block), so every interchange commutes
// with the pending update of the current block.
#include <cfloat>
#include <climits>
#include <cstdint>

#include "device.cuh"

namespace kep {

namespace {

constexpr double kAlphaB = 0.6403882032022076;   // (1 + sqrt(17)) / 8
constexpr int BT = 256;                           // k_bigp threads
constexpr int BNB = 128;                          // pivots per block (the trailing update's K)
constexpr int BST_W = 16;                         // state record (int) per group

// state record of a group (global, persists between launches)
enum { S_E = 0, S_QE, S_STEP, S_K0, S_NEG, S_ZERO, S_POS, S_2X2, S_INIT, S_BAR };

struct Part {               // one CTA's reduction partial
    double v0, v1, v2, v3;  // max candidates, max all, extra, owner value
    int i0, own;            // argmax of v0, owner flag of v3
    int pad0, pad1;
};

__device__ __forceinline__ void part_better(double& v, int& i, double v2, int i2) {
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// group-wide barrier: monotone counter, target = ncta x (barrier number)
__device__ __forceinline__ void gbar(unsigned* cnt, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(cnt) : "memory");
            if (v < target) __nanosleep(20);
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

// block reduce of (max, argmax) + 3 maxima
__device__ __forceinline__ void cta_reduce(double& a, int& ai, double& b, double& c, double& d, double* sv, int* si) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double a2 = __shfl_xor_sync(0xffffffffu, a, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, ai, o);
        part_better(a, ai, a2, i2);
        b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) { sv[4 * w] = a; sv[4 * w + 1] = b; sv[4 * w + 2] = c; sv[4 * w + 3] = d; si[w] = ai; }
    __syncthreads();
    a = sv[0]; b = sv[1]; c = sv[2]; d = sv[3]; ai = si[0];
    for (int q = 1; q < BT / 32; ++q) {
        part_better(a, ai, sv[4 * q], si[q]);
        b = fmax(b, sv[4 * q + 1]);
        c = fmax(c, sv[4 * q + 2]);
        d = fmax(d, sv[4 * q + 3]);
    }
}

struct GroupCtx {
    int s, sh, f, q, p, c, ld, root;
    double* F;
    AuxRec A;
    int* st;
    Part* part;
    double* colk;
    double* colr;
    unsigned* bar;
};

__device__ __forceinline__ GroupCtx group_ctx(const DevPlan& P, const int2* groups, const int64_t* scroff,
                                               double* scr, int* state, unsigned* bars, int gy) {
    GroupCtx G;
    const int2 gr = groups[gy];
    G.s = gr.x;
    G.sh = gr.y;
    const int nd = P.nd_in[(size_t)G.sh * P.nf + G.s];
    G.p = P.npiv[G.s];
    G.c = P.ncb[G.s];
    G.f = P.forder[G.s] + (nd > 0 ? nd : 0);
    G.q = G.p + (nd > 0 ? nd : 0);
    G.ld = ldpad(P.cap[G.s]);
    G.root = G.c == 0;
    G.F = P.arena + (size_t)G.sh * P.arena_stride + P.arena_off[G.s];
    G.A = aux_rec(P, G.sh, G.s, P.cap[G.s] - G.c);
    G.st = state + (size_t)gy * BST_W;
    double* base = scr + scroff[gy];
    const int cap = P.cap[G.s];
    G.colk = base;
    G.colr = base + cap;
    G.part = reinterpret_cast<Part*>(base + 2 * (size_t)cap);
    G.bar = bars + gy;
    return G;
}

}  // namespace

// ------------------------------------------------------------------ k_biginit
__global__ void k_biginit(DevPlan P, const int2* __restrict__ groups, const int64_t* __restrict__ scroff, double* scr,
                          int* state, unsigned* bars) {
    GroupCtx G = group_ctx(P, groups, scroff, scr, state, bars, blockIdx.x);
    const int nd = P.nd_in[(size_t)G.sh * P.nf + G.s];
    for (int i = threadIdx.x; i < G.q; i += blockDim.x) G.A.perm[i] = i;
    if (threadIdx.x == 0) {
        for (int k = 0; k < BST_W; ++k) G.st[k] = 0;
        G.st[S_E] = 0;
        G.st[S_QE] = nd < 0 ? 0 : G.q;           // slack overflow: nothing to do (the batch is re-planned)
        G.st[S_INIT] = nd < 0 ? -1 : 1;
        *G.bar = 0u;
    }
}

// ------------------------------------------------------------------ k_bigp
__global__ void __launch_bounds__(BT, 1) k_bigp(DevPlan P, const int2* __restrict__ groups,
                                                const int64_t* __restrict__ scroff, double* scr, int* state,
                                                unsigned* bars) {
    __shared__ double sG[BNB + 2];                  // G row of the pivot (row k or r) over the block's columns
    __shared__ double sv[4 * (BT / 32)];
    __shared__ int si[BT / 32];
    GroupCtx G = group_ctx(P, groups, scroff, scr, state, bars, blockIdx.y);
    const int ncta = gridDim.x, cj = blockIdx.x, tid = threadIdx.x;
    double* F = G.F;
    const int ld = G.ld, f = G.f, q = G.q;
    const double u = P.u;
    const AuxRec A = G.A;
    int e = G.st[S_E], qe = G.st[S_QE], step = G.st[S_STEP];
    unsigned nbar = (unsigned)G.st[S_BAR];
    if (e >= qe) {                                  // the group is done (all CTAs read the same state):
        if (cj == 0 && tid == 0) G.st[S_K0] = e;    // no block pending for k_bigu
        return;
    }
    const int k0 = e;
    const int ra = (int)((int64_t)f * cj / ncta), rb = (int)((int64_t)f * (cj + 1) / ncta);
    long long c_neg = 0, c_zero = 0, c_pos = 0, c_2x2 = 0;
    auto sync_all = [&]() { ++nbar; gbar(G.bar, nbar * (unsigned)ncta); };
    // symmetric interchange of positions a < b (both < q) in the lower-stored front; each CTA moves a
    // disjoint share: rows a, b of columns t < a (by t; column `skip` left out: it is rewritten right
    // after), columns a, b below b and the (a, b) band (by own row, the same thread-to-row map as the
    // G-column stores that follow, so a row's old values are moved before its G entry is written)
    auto swap_sym = [&](int a, int b, int skip) {
        for (int t = cj * BT + tid; t < a; t += ncta * BT) {
            if (t == skip) continue;
            double* x = F + a + (size_t)t * ld;
            double* y = F + b + (size_t)t * ld;
            const double vx = __ldcg(x), vy = __ldcg(y);            // rows owned by other CTAs: via L2
            *x = vy; *y = vx;
        }
        for (int i = max(ra, a + 1) + tid; i < rb; i += BT) {
            if (i == b) continue;
            double* x;
            double* y;
            if (i > b) { x = F + i + (size_t)a * ld; y = F + i + (size_t)b * ld; }
            else { x = F + i + (size_t)a * ld; y = F + b + (size_t)i * ld; }
            const double v = *x; *x = *y; *y = v;
        }
        if (cj == 0 && tid == 0) {
            double* x = F + a + (size_t)a * ld;
            double* y = F + b + (size_t)b * ld;
            const double v = *x; *x = *y; *y = v;
            const int z = A.perm[a]; A.perm[a] = A.perm[b]; A.perm[b] = z;
        }
    };
    // current column j over the own rows >= k (left-looking over the block's eliminated columns [k0, k))
    auto column = [&](int j, int k, double* out) {
        const int nt = k - k0;
        __syncthreads();
        // F is read through L2 (ld.global.cg): other CTAs of the group wrote it (G columns, interchanges)
        // before the last group barrier, and L1 lines cached earlier would be stale
        for (int t = tid; t < nt; t += BT) sG[t] = __ldcg(F + j + (size_t)(k0 + t) * ld) * __ldcg(A.sgn + k0 + t);
        __syncthreads();
        for (int i = max(ra, k) + tid; i < rb; i += BT) {
            double v = i >= j ? __ldcg(F + i + (size_t)j * ld) : __ldcg(F + j + (size_t)i * ld);
            const double* gi = F + i + (size_t)k0 * ld;
            for (int t = 0; t < nt; ++t) v = fma(-__ldcg(gi + (size_t)t * ld), sG[t], v);
            out[i] = v;
        }
        __syncthreads();                            // the column's own rows are read by other threads next
    };
    // group-wide reduction of the CTAs' partials: thread x < ncta loads CTA x's record from L2
    // (written by other SMs before the barrier), then one CTA reduction
    auto group_reduce = [&](int base, double& a, int& ai, double& b, double& c) {
        double va = -1.0, vb = 0.0, vc = 0.0, vd = 0.0;
        int vi = INT_MAX;
        if (tid < ncta) {
            const Part* pp = G.part + base + tid;
            va = __ldcg(&pp->v0); vb = __ldcg(&pp->v1); vc = __ldcg(&pp->v2); vi = __ldcg(&pp->i0);
        }
        cta_reduce(va, vi, vb, vc, vd, sv, si);
        a = va; ai = vi; b = vb; c = vc;
    };
    while (e < qe && e - k0 < BNB) {
        const int k = e;
        // ---- P1: column k, (max, argmax) over the FS candidates (k, qe), max over all rows > k, a_kk
        column(k, k, G.colk);
        double mC = -1.0, mR = 0.0, z1 = 0.0, z2 = 0.0;
        int iC = INT_MAX;
        for (int i = max(ra, k + 1) + tid; i < rb; i += BT) {
            const double a = fabs(G.colk[i]);
            if (i < qe) part_better(mC, iC, a, i);
            mR = fmax(mR, a);
        }
        cta_reduce(mC, iC, mR, z1, z2, sv, si);
        // partials: buffer 0 for column k, buffer 1 for column r (a buffer is rewritten only after
        // every CTA has passed a later barrier, i.e. after all reads of it)
        if (tid == 0) G.part[cj] = Part{mC, mR, 0.0, 0.0, iC, 0, 0, 0};
        sync_all();
        double gC = -1.0, gR = 0.0, akks = 0.0, zz = 0.0;
        int r = INT_MAX;
        group_reduce(0, gC, r, gR, zz);
        akks = __ldcg(G.colk + k);                                  // another CTA's row: visible after the barrier
        const double aakk = fabs(akks);
        if (gC < 0.0) { gC = 0.0; r = k; }
        if (aakk == 0.0 && gR == 0.0) {                             // zero column: exact zero pivot
            for (int i = max(ra, k + 1) + tid; i < rb; i += BT) F[i + (size_t)k * ld] = 0.0;
            if (cj == 0 && tid == 0) {
                F[k + (size_t)k * ld] = 0.0;
                A.kind[k] = PK_ZERO; A.d[k] = 0.0; A.ds[k] = 0.0; A.step[k] = step;
                A.sgn[k] = 1.0; A.gca[k] = 0.0; A.gcb[k] = 0.0;
            }
            c_zero++;
            e++;
            step++;
            sync_all();
            continue;
        }
        int kind = 1, j = k;
        double rall = 0.0, gk = 0.0, arr = 0.0;
        if (aakk < kAlphaB * gC) {
            // ---- P2: column r; rho over FS candidates [k, qe) \ {r}, rall / gk over all rows >= k \ {k, r}
            column(r, k, G.colr);
            double rho = 0.0, ra_ = 0.0, gk_ = 0.0, dummy = -1.0;
            int di = INT_MAX;
            for (int i = max(ra, k) + tid; i < rb; i += BT) {
                if (i == r) continue;
                const double a = fabs(G.colr[i]);
                if (i < qe) rho = fmax(rho, a);
                if (i != k) { ra_ = fmax(ra_, a); gk_ = fmax(gk_, fabs(G.colk[i])); }
            }
            cta_reduce(dummy, di, rho, ra_, gk_, sv, si);
            if (tid == 0) G.part[ncta + cj] = Part{rho, ra_, gk_, 0.0, 0, 0, 0, 0};
            sync_all();
            double rh = 0.0;
            int ri = 0;
            group_reduce(ncta, rh, ri, rall, gk);
            if (rh < 0.0) rh = 0.0;
            arr = fabs(__ldcg(G.colr + r));
            if (aakk * rh >= kAlphaB * gC * gC) { kind = 1; j = k; }
            else if (arr >= kAlphaB * rh) { kind = 1; j = r; }
            else { kind = 2; j = r; }
        }
        if (kind == 2 && e - k0 + 2 > BNB + 1) break;              // no room for the pair in this block
        bool ok = true;
        if (!G.root) {
            if (kind == 1) {
                const double fa = (j == k) ? gR : fmax(rall, gC);
                ok = (j == k ? aakk : arr) >= u * fa;
            } else {
                const double a11 = akks, a21 = __ldcg(G.colk + r), a22 = __ldcg(G.colr + r);
                const double det = a11 * a22 - a21 * a21;
                if (det == 0.0) ok = false;
                else {
                    const double ad = fabs(det);
                    ok = (fabs(a22) * gk + fabs(a21) * rall) / ad <= 1.0 / u &&
                         (fabs(a21) * gk + fabs(a11) * rall) / ad <= 1.0 / u;
                }
            }
        }
        if (!ok) {                                                   // delay column k (R1)
            if (qe - 1 != k) swap_sym(k, qe - 1, -1);
            qe--;
            step++;
            sync_all();
            continue;
        }
        if (kind == 1) {
            const bool fromr = j != k;
            if (fromr) swap_sym(k, r, -1);                           // no barrier: see swap_sym
            // pivot column after the interchange: column r's values with rows k and r exchanged
            const double* w = fromr ? G.colr : G.colk;
            const double d = fromr ? __ldcg(G.colr + r) : akks;
            const double wk = fromr ? __ldcg(G.colr + k) : 0.0;       // row r of the pivot column
            const double gsc = sqrt(fabs(d)) / d;                    // G = L sqrt|d| = W sqrt|d| / d
            for (int i = max(ra, k + 1) + tid; i < rb; i += BT) {
                const double wi = (fromr && i == r) ? wk : w[i];
                F[i + (size_t)k * ld] = wi * gsc;
            }
            if (cj == 0 && tid == 0) {
                F[k + (size_t)k * ld] = d;
                const double sg = d < 0.0 ? -1.0 : 1.0;
                A.kind[k] = PK_1X1; A.d[k] = d; A.ds[k] = 0.0; A.step[k] = step;
                A.sgn[k] = sg; A.gca[k] = sg / sqrt(fabs(d)); A.gcb[k] = 0.0;
            }
            if (d < 0.0) c_neg++; else if (d > 0.0) c_pos++; else c_zero++;
            e += 1;
            step++;
            sync_all();
        } else {
            if (r != k + 1) swap_sym(k + 1, r, k);                   // column k is rewritten below
            // columns k, k+1 after the interchange (k+1 <-> r): rows k+1 and r exchanged in both
            auto nk = [&](int i) { return __ldcg(G.colk + (i == k + 1 ? r : (i == r ? k + 1 : i))); };
            auto nr = [&](int i) { return __ldcg(G.colr + (i == k + 1 ? r : (i == r ? k + 1 : i))); };
            const double d11 = nk(k), d21 = nk(k + 1), d22 = nr(k + 1);
            const double det = d11 * d22 - d21 * d21;
            const double i11 = d22 / det, i21 = -d21 / det, i22 = d11 / det;
            double cs, sn, l1, l2;
            pair_eig(d11, d21, d22, cs, sn, l1, l2);
            const double r1 = sqrt(fabs(l1)), r2 = sqrt(fabs(l2));
            for (int i = max(ra, k + 2) + tid; i < rb; i += BT) {
                const double w1 = nk(i), w2 = nr(i);
                const double La = w1 * i11 + w2 * i21, Lb = w1 * i21 + w2 * i22;
                F[i + (size_t)k * ld] = (La * cs + Lb * sn) * r1;
                F[i + (size_t)(k + 1) * ld] = (Lb * cs - La * sn) * r2;
            }
            if (cj == 0 && tid == 0) {
                F[k + (size_t)k * ld] = d11;
                F[k + 1 + (size_t)k * ld] = 0.0;
                F[k + 1 + (size_t)(k + 1) * ld] = d22;
                A.kind[k] = PK_2X2A; A.d[k] = d11; A.ds[k] = d21; A.step[k] = step;
                A.kind[k + 1] = PK_2X2B; A.d[k + 1] = d22; A.ds[k + 1] = 0.0; A.step[k + 1] = step;
                const double s1 = l1 < 0.0 ? -1.0 : 1.0, s2 = l2 < 0.0 ? -1.0 : 1.0;
                const double k1 = s1 / r1, k2 = s2 / r2;
                A.sgn[k] = s1; A.sgn[k + 1] = s2;
                A.gca[k] = cs * k1;     A.gcb[k] = sn * k1;
                A.gca[k + 1] = cs * k2; A.gcb[k + 1] = -sn * k2;
            }
            const double tt = (d11 / d21) * (d22 / d21) - 1.0;       // a5: sign(det), scaled (R2)
            if (tt < 0.0) { c_neg++; c_pos++; }
            else if (tt > 0.0) { if (d11 < 0.0) c_neg += 2; else c_pos += 2; }
            else { c_zero++; if (d11 + d22 < 0.0) c_neg++; else c_pos++; }
            c_2x2++;
            e += 2;
            step++;
            sync_all();
        }
    }
    if (cj == 0 && tid == 0) {
        G.st[S_E] = e; G.st[S_QE] = qe; G.st[S_STEP] = step; G.st[S_K0] = k0;
        G.st[S_NEG] += (int)c_neg; G.st[S_ZERO] += (int)c_zero; G.st[S_POS] += (int)c_pos; G.st[S_2X2] += (int)c_2x2;
        G.st[S_BAR] = (int)nbar;
    }
}

// ------------------------------------------------------------------ k_bigu
// F[i, j] -= sum_{t in [k0, e)} G[i, t] S_t G[j, t] for j in [e, q), i in [j, f): 64 x 64 tiles,
// persistent CTAs over every group's tiles of the level; K streamed in chunks of 16 pivots through a
// 3-stage cp.async pipeline (G columns are contiguous along the rows: t-major tiles).
constexpr int UT2 = 128;
constexpr int UKC = 16;
constexpr int UST = 3;
constexpr int UPA2 = 64 + 4;                     // = 4 (mod 16): conflict-free f64 fragments

__device__ __forceinline__ void cpa8(double* dst, const double* src, bool v) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(v ? 8 : 0));
}
__device__ __forceinline__ void cpa16(double* dst, const double* src, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes));
}

__global__ void __launch_bounds__(UT2, 4) k_bigu(DevPlan P, const int2* __restrict__ groups, int ngroups,
                                                 const int64_t* __restrict__ scroff, double* scr, int* state,
                                                 unsigned* bars) {
    extern __shared__ __align__(16) double ubuf[];
    double (*As)[UKC][UPA2] = reinterpret_cast<double (*)[UKC][UPA2]>(ubuf);                    // G[i, t] (t-major)
    double (*Bs)[UKC][UPA2] = reinterpret_cast<double (*)[UKC][UPA2]>(ubuf + UST * UKC * UPA2); // G[j, t]
    __shared__ double sgn[UST][UKC];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tg = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    for (int gy = 0; gy < ngroups; ++gy) {
        GroupCtx G = group_ctx(P, groups, scroff, scr, state, bars, gy);
        const int e = G.st[S_E], k0 = G.st[S_K0];
        const int K = e - k0;
        if (K <= 0 || e >= G.q) continue;
        const int f = G.f, q = G.q, ld = G.ld;
        double* F = G.F;
        const int nI = (f - e + 63) / 64, nJ = (q - e + 63) / 64;
        const int64_t ntile = (int64_t)nJ * nI - (int64_t)nJ * (nJ - 1) / 2;    // J <= I
        const int nk = (K + UKC - 1) / UKC;
        for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
            int J = 0;
            int64_t rem = tile;
            while (rem >= nI - J) { rem -= nI - J; ++J; }
            const int I = J + (int)rem;
            const int i0 = e + 64 * I, j0 = e + 64 * J;
            auto load = [&](int buf, int kc) {
                const int t0 = kc * UKC;
                for (int x = tid; x < UKC * 32; x += UT2) {           // 16-byte pairs of rows
                    const int t = x >> 5, r2 = 2 * (x & 31);
                    const bool vt = t0 + t < K;
                    const double* ca = F + (size_t)(k0 + t0 + t) * ld;
                    const int gi = i0 + r2, gj = j0 + r2;
                    // rows i0.. are even-aligned only when i0 is even: copy pairs when aligned, else singles
                    if (((i0 & 1) == 0) && ((j0 & 1) == 0)) {
                        cpa16(&As[buf][t][r2], ca + (vt ? gi : 0), vt ? (gi + 1 < f ? 16 : (gi < f ? 8 : 0)) : 0);
                        cpa16(&Bs[buf][t][r2], ca + (vt ? gj : 0), vt ? (gj + 1 < q ? 16 : (gj < q ? 8 : 0)) : 0);
                    } else {
                        for (int h = 0; h < 2; ++h) {
                            cpa8(&As[buf][t][r2 + h], ca + (vt && gi + h < f ? gi + h : 0), vt && gi + h < f);
                            cpa8(&Bs[buf][t][r2 + h], ca + (vt && gj + h < q ? gj + h : 0), vt && gj + h < q);
                        }
                    }
                }
                if (tid < UKC) sgn[buf][tid] = (t0 + tid < K) ? G.A.sgn[k0 + t0 + tid] : 0.0;
                asm volatile("cp.async.commit_group;\n" ::);
            };
            __syncthreads();                                     // previous tile's smem reads done
#pragma unroll
            for (int st0 = 0; st0 < UST - 1; ++st0) {
                if (st0 < nk) load(st0, st0);
                else asm volatile("cp.async.commit_group;\n" ::);
            }
            double acc[4][4][2];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
            for (int kc = 0; kc < nk; ++kc) {
                const int buf = kc % UST;
                asm volatile("cp.async.wait_group %0;\n" ::"n"(UST - 2));
                __syncthreads();
                {
                    const int nx = kc + UST - 1;
                    if (nx < nk) load(nx % UST, nx);
                    else asm volatile("cp.async.commit_group;\n" ::);
                }
#pragma unroll
                for (int k4 = 0; k4 < UKC; k4 += 4) {
                    double a[4], b[4];
                    const double sg = sgn[buf][k4 + tg];
#pragma unroll
                    for (int mb = 0; mb < 4; ++mb) a[mb] = As[buf][k4 + tg][wm + 8 * mb + g];
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) b[nb] = Bs[buf][k4 + tg][wn + 8 * nb + g] * sg;
#pragma unroll
                    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                        for (int nb = 0; nb < 4; ++nb)
                            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                         : "+d"(acc[mb][nb][0]), "+d"(acc[mb][nb][1])
                                         : "d"(a[mb]), "d"(b[nb]));
                }
            }
            asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = i0 + wm + 8 * mb + g;
                        const int j = j0 + wn + 8 * nb + 2 * tg + h;
                        if (i < f && j < q && i >= j) atomicAdd(&F[i + (size_t)j * ld], -acc[mb][nb][h]);
                    }
        }
    }
}

// ------------------------------------------------------------------ k_bigfin
// CB rows of the FS columns to the upper part (G for eliminated columns, the updated W21 for
// delayed ones), D / inertia statistics, nd_out, flag.  Grid (ctas per group, groups).
__global__ void k_bigfin(DevPlan P, const int2* __restrict__ groups, const int64_t* __restrict__ scroff, double* scr,
                         int* state, unsigned* bars) {
    GroupCtx G = group_ctx(P, groups, scroff, scr, state, bars, blockIdx.y);
    if (G.st[S_INIT] < 0) {                                   // slack overflow: mirror the other kernels
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            P.nd_out[(size_t)G.sh * P.nf + G.s] = -1;
            P.flag[(size_t)G.sh * P.nf + G.s] = FL_OK;
        }
        return;
    }
    const int e = G.st[S_E], q = G.q, f = G.f, ld = G.ld;
    double* F = G.F;
    const int64_t tot = (int64_t)(f - q) * q;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
        const int ii = (int)(x / q), t = (int)(x - (int64_t)ii * q), i = q + ii;
        F[t + (size_t)i * ld] = F[i + (size_t)t * ld];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ShiftStat* st = P.stats + G.sh;
        const int ndo = q - e;
        P.nd_out[(size_t)G.sh * P.nf + G.s] = ndo;
        P.flag[(size_t)G.sh * P.nf + G.s] = FL_OK;
        if (G.st[S_NEG]) atomicAdd(&st->n_neg, (unsigned long long)G.st[S_NEG]);
        if (G.st[S_ZERO]) atomicAdd(&st->n_zero, (unsigned long long)G.st[S_ZERO]);
        if (G.st[S_POS]) atomicAdd(&st->n_pos, (unsigned long long)G.st[S_POS]);
        if (G.st[S_2X2]) atomicAdd(&st->n_2x2, (unsigned long long)G.st[S_2X2]);
        if (ndo) atomicAdd(&st->n_delayed, (unsigned long long)ndo);
    }
    // smallest |pivot| (singularity test), one CTA per group
    if (blockIdx.x == 0) {
        double mn = DBL_MAX;
        for (int t = threadIdx.x; t < e; t += blockDim.x) {
            const int kd = G.A.kind[t];
            if (kd == PK_ZERO) mn = 0.0;
            else if (kd == PK_1X1) mn = fmin(mn, fabs(G.A.d[t]));
            else if (kd == PK_2X2A) {
                const double d11 = G.A.d[t], d21 = G.A.ds[t], d22 = G.A.d[t + 1];
                const double det = d11 * d22 - d21 * d21;
                const double tr = 0.5 * (d11 + d22);
                const double disc = sqrt(0.25 * (d11 - d22) * (d11 - d22) + d21 * d21);
                const double big = fabs(tr) + disc;
                mn = fmin(mn, big > 0.0 ? fabs(det) / big : 0.0);
            }
        }
        for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        if ((threadIdx.x & 31) == 0 && mn < DBL_MAX) atomic_min_pos_double(&P.stats[G.sh].minpiv_bits, mn);
    }
}

int big_block() { return BNB; }
size_t big_scratch_doubles(int cap, int ncta) { return 2 * (size_t)cap + 2 * (size_t)ncta * (sizeof(Part) / 8) + 8; }

void launch_big_init(const DevPlan& P, const int2* groups, int ngroups, const int64_t* scroff, double* scr, int* state,
                     unsigned* bars, cudaStream_t st) {
    if (ngroups <= 0) return;
    k_biginit<<<ngroups, 256, 0, st>>>(P, groups, scroff, scr, state, bars);
}

int big_blocks(int qmax) { return (qmax + BNB - 2) / (BNB - 1) + 1; }   // each block eliminates >= BNB - 1 or finishes

void launch_big_panel(const DevPlan& P, const int2* groups, int ngroups, int ncta, const int64_t* scroff, double* scr,
                      int* state, unsigned* bars, cudaStream_t st) {
    if (ngroups <= 0) return;
    void* args[] = {(void*)&P, (void*)&groups, (void*)&scroff, (void*)&scr, (void*)&state, (void*)&bars};
    cudaLaunchCooperativeKernel((const void*)k_bigp, dim3(ncta, ngroups), dim3(BT), args, 0, st);
}

void launch_big_update(const DevPlan& P, const int2* groups, int ngroups, const int64_t* scroff, double* scr,
                       int* state, unsigned* bars, cudaStream_t st) {
    if (ngroups <= 0) return;
    const size_t usmem = sizeof(double) * 2 * UST * UKC * UPA2;
    static unsigned long long attr = 0;
    if (first_on_device(attr)) cudaFuncSetAttribute(k_bigu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usmem);
    k_bigu<<<148 * 4, UT2, usmem, st>>>(P, groups, ngroups, scroff, scr, state, bars);
}

void launch_big_fin(const DevPlan& P, const int2* groups, int ngroups, const int64_t* scroff, double* scr, int* state,
                    unsigned* bars, cudaStream_t st) {
    if (ngroups <= 0) return;
    k_bigfin<<<dim3(32, ngroups), 256, 0, st>>>(P, groups, scroff, scr, state, bars);
}

}  // namespace kep
