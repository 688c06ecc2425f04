// kernels.cu — numeric multifrontal LDL^T of A - sigma B, inertia only.
//
// Rows a1-a5 of SURVEY.md §8 (BASELINE.json north_star parts (1)-(5)):
//   a1 assembly of A - sigma B into the fronts of one elimination-tree level
//   a2 extend-add of the children's contribution blocks (+ delayed columns)
//   a3 Bunch-Kaufman partial LDL^T of the fully-summed (FS) block with the
//      threshold test and delayed pivots (reading R1)
//   a4 Schur-complement update of the contribution block
//   a5 inertia of D: 1x1 by sign, 2x2 by sign(det) (R2)
//
// Front layout (one dense column-major square per front, lower triangle used,
// leading dimension ld = f_s + nd_s):
//   [0, p)        own pivots (static order)
//   [p, p+nd)     columns delayed by the children, children in order
//   [p+nd, ld)    contribution-block (CB) rows, ascending elimination position
// After a3 the eliminated pivots sit in [0, e), the columns this front delays
// in [e, p+nd) and the CB rows are untouched in place, so the trailing block
// F[e:, e:] is exactly what the parent extend-adds.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdint>

#include "device.cuh"

namespace kep {

namespace {

constexpr double kAlpha = 0.6403882032022076;   // (1 + sqrt(17)) / 8, Bunch-Kaufman

struct MaxIdx {
    double v;
    int i;
};

__device__ __forceinline__ MaxIdx better(MaxIdx a, MaxIdx b) {
    // larger value wins; ties -> lower index (LAPACK idamax semantics)
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}

template <int NT>
__device__ MaxIdx block_max_idx(MaxIdx x, MaxIdx* sh) {
    for (int o = 16; o > 0; o >>= 1) {
        MaxIdx y;
        y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
        y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
        x = better(x, y);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        x = l < NT / 32 ? sh[l] : MaxIdx{-1.0, INT_MAX};
        for (int o = 16; o > 0; o >>= 1) {
            MaxIdx y;
            y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
            y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
            x = better(x, y);
        }
        if (l == 0) sh[0] = x;
    }
    __syncthreads();
    MaxIdx r = sh[0];
    __syncthreads();
    return r;
}

template <int NT>
__device__ double block_max(double x, double* sh) {
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        x = l < NT / 32 ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
        if (l == 0) sh[0] = x;
    }
    __syncthreads();
    double r = sh[0];
    __syncthreads();
    return r;
}

// symmetric access a(i, j) to the lower-stored front
__device__ __forceinline__ double symget(const double* F, int ld, int i, int j) {
    return i >= j ? F[i + (size_t)j * ld] : F[j + (size_t)i * ld];
}

// ---------------------------------------------------------------- a1 + a2
constexpr int kAsmThreads = 256;
constexpr int kAsmNW = kAsmThreads / 32;
constexpr int kAsmMapMax = 16384;         // child row positions staged in shared memory (uint16, all children)
constexpr int kAsmKids = 32;              // children handled by the gather path (one lane each)
constexpr int kAsmChunk = 128;            // parent rows per warp work chunk
constexpr int kAsmStripEnt = 32768;       // target lower-triangle entries per CTA (assembly_strips)

// Columns [lo, hi) of a lower triangle of order ld holding the x-th of S equal
// shares of its entries (column j has ld - j entries).
__device__ __forceinline__ void tri_split(int ld, int S, int x, int& lo, int& hi) {
    auto col_at = [&](int y) -> int {
        if (y <= 0) return 0;
        if (y >= S) return ld;
        const double T = 0.5 * (double)ld * (double)(ld + 1), A = T * (double)y / (double)S;
        const double b = (double)ld + 0.5;
        int j = (int)ceil(b - sqrt(fmax(b * b - 2.0 * A, 0.0)));
        return min(max(j, 0), ld);
    };
    lo = col_at(x);
    hi = col_at(x + 1);
}

struct AsmKid {                  // one child as seen by the parent's assembly
    const double* F;             // child front
    int ldc, ec, ndo, mc;        // leading dimension, first CB/delayed position, delayed count, CB+delayed count
    int moff;                    // offset of its row positions in s_pos
    int dof;                     // parent position of its first delayed column
    int wup;                     // fast-path child: CB rows of its delayed columns in the upper part
};

// Strip x of S of one front (columns [lo, hi), lower part).  Gather formulation:
// each warp owns whole parent columns and builds them in chunks of kAsmChunk rows
// in a private shared-memory buffer -- zero, original entries (alpha a - sigma b),
// then for each child in order the contiguous run of its CB column that lands in
// the chunk (child row positions increase with the child row index) -- and writes
// each chunk once, coalesced.  No atomics and no block barriers on this path;
// every parent entry is summed in a fixed order.  Entries of the children's
// delayed columns (rare) are added afterwards with RED adds, children in order.
// Fronts with more than kAsmKids children or kAsmMapMax child rows take the plain
// path: zero-fill, stores, RED adds.
__device__ __forceinline__ void assemble_strip(const DevPlan& P, const int s, const int xs, const int S, int only_flagged) {
    const int sh = blockIdx.y;
    if (only_flagged) {               // re-assembly of fronts whose fast-path pass failed (restore)
        const int fl = P.flag[(size_t)sh * P.nf + s];
        if (fl != FL_RERUN && fl != FL_REF) return;
    }
    ShiftStat* st = P.stats + sh;
    double* arena = P.arena + (size_t)sh * P.arena_stride;
    int32_t* nd_in = P.nd_in + (size_t)sh * P.nf;
    const int32_t* nd_out = P.nd_out + (size_t)sh * P.nf;
    int32_t* doff = P.doff + (size_t)sh * P.nf;
    __shared__ int s_nd, s_skip, s_msum, s_anyd;
    __shared__ double s_red[32];
    __shared__ uint16_t s_pos[kAsmMapMax];
    __shared__ AsmKid s_kid[kAsmKids];
    extern __shared__ double s_buf[];                          // [kAsmNW][kAsmChunk]
    const int c0 = P.child_ptr[s], c1 = P.child_ptr[s + 1];
    const int nch = c1 - c0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p = P.npiv[s];
    if (warp == 0) {                  // children: delayed counts (prefix), descriptors
        int off = 0, bad = 0, msum = 0, anyd = 0;
        for (int q0 = 0; q0 < nch; q0 += 32) {
            const int q = q0 + lane;
            int no = 0, mc = 0, c = -1;
            if (q < nch) {
                c = P.child_list[c0 + q];
                no = nd_out[c];
                if (no < 0) bad = 1;
            }
            const int nz = no > 0 ? no : 0;
            int inc = nz;                                         // inclusive warp prefix of delayed counts
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const int dof = off + inc - nz;
            if (q < nch) {
                if (xs == 0) doff[c] = dof;
                mc = nz + P.ncb[c];
                if (q < kAsmKids) {
                    const int fc = P.forder[c] + nd_in[c];
                    AsmKid k;
                    k.F = arena + P.arena_off[c];
                    k.ldc = ldpad(P.cap[c]);
                    k.ec = fc - mc;
                    k.ndo = nz;
                    k.mc = mc;
                    k.moff = 0;
                    k.dof = p + dof;
                    k.wup = P.flag[(size_t)sh * P.nf + c] == FL_OK && nz > 0;
                    s_kid[q] = k;
                }
            }
            int minc = mc;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, minc, o);
                if (lane >= o) minc += y;
            }
            if (q < nch && q < kAsmKids) s_kid[q].moff = msum + minc - mc;
            msum += __shfl_sync(0xffffffffu, minc, 31);
            off += __shfl_sync(0xffffffffu, inc, 31);
            anyd |= __any_sync(0xffffffffu, nz > 0);
            bad = __any_sync(0xffffffffu, bad);
        }
        if (lane == 0) {
            const int need = P.forder[s] + off;
            if (need > P.cap[s]) {
                bad = 1;
                if (xs == 0) atomicMax(&st->need_slack, off);
            }
            if (bad && xs == 0) atomicOr(&st->flags, FLAG_OVERFLOW);
            s_skip = bad;
            s_nd = off;
            s_msum = (nch <= kAsmKids) ? msum : INT_MAX;
            s_anyd = anyd;
            if (xs == 0) nd_in[s] = bad ? -1 : off;
        }
    }
    __syncthreads();
    if (s_skip) return;
    const int nd = s_nd, fo = P.forder[s] + nd, ld = ldpad(P.cap[s]);   // order, leading dimension
    double* F = arena + P.arena_off[s];
    int clo, chi;
    tri_split(fo, S, xs, clo, chi);
    const bool gather = s_msum <= kAsmMapMax;
    if (xs == 0) {   // labels of the FS positions: own pivots, then each child's delayed variables
        const AuxRec A = aux_rec(P, sh, s, P.cap[s] - P.ncb[s]);
        for (int i = tid; i < p; i += kAsmThreads) A.label[i] = P.piv_first[s] + i;
        if (s_anyd) {
            int off = 0;
            for (int q = c0; q < c1; ++q) {
                const int c = P.child_list[q];
                const int ndo = nd_out[c];
                if (ndo <= 0) continue;
                const AuxRec C = aux_rec(P, sh, c, P.cap[c] - P.ncb[c]);
                const int ec = P.npiv[c] + nd_in[c] - ndo;
                for (int j = tid; j < ndo; j += kAsmThreads) A.label[p + off + j] = C.label[C.perm[ec + j]];
                off += ndo;
            }
        }
    }
    const double sigma = P.sigma[sh], alpha = P.alpha[sh];
    const int64_t a0 = P.asm_ptr[s];
    const int32_t* acol = P.asm_col + P.piv_first[s] + s;
    double mx = 0.0;
    if (gather) {
        // parent positions of every child row, all children (one barrier)
        for (int q = 0; q < nch; ++q) {
            const AsmKid& k = s_kid[q];
            const int32_t* __restrict__ rm = P.rmap + P.rmap_ptr[P.child_list[c0 + q]];
            const int dof = k.dof;
            for (int x = tid; x < k.mc; x += kAsmThreads) {
                int v;
                if (x < k.ndo) v = dof + x;
                else { const int r = rm[x - k.ndo]; v = r < p ? r : r + nd; }
                s_pos[k.moff + x] = (uint16_t)v;
            }
        }
        __syncthreads();
        double* buf = s_buf + warp * kAsmChunk;
        // lane q < nch tracks child q: jk = its column landing in parent column c, ia = next row
        for (int c = clo + warp; c < chi; c += kAsmNW) {
            int jk = -1, ia = 0, mcq = 0, mo = 0;
            if (lane < nch) {
                const AsmKid& k = s_kid[lane];
                mcq = k.mc; mo = k.moff;
                int lo = k.ndo, hi = k.mc;                        // first non-delayed row with pos >= c
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if ((int)s_pos[mo + mid] < c) lo = mid + 1; else hi = mid;
                }
                if (lo < k.mc && (int)s_pos[mo + lo] == c) { jk = lo; ia = lo; }
            }
            const int e0 = c < p ? acol[c] : 0, e1 = c < p ? acol[c + 1] : 0;
            for (int r0 = c; r0 < fo; r0 += kAsmChunk) {
                const int r1 = min(r0 + kAsmChunk, fo);
#pragma unroll
                for (int u = 0; u < kAsmChunk / 32; ++u) buf[lane + 32 * u] = 0.0;
                __syncwarp();
                for (int e = e0 + lane; e < e1; e += 32) {        // original entries of column c in [r0, r1)
                    const uint32_t rc = P.asm_rc[a0 + e];
                    const double av = P.a[a0 + e], bv = P.b[a0 + e];     // (one round trip)
                    const int lr = (int)(rc >> 16);
                    const int r = lr < p ? lr : lr + nd;
                    if (r >= r0 && r < r1) {
                        const double v = fma(-sigma, bv, alpha * av);   // alpha A - sigma B
                        buf[r - r0] = v;
                        mx = fmax(mx, fabs(v));
                    }
                }
                int ib = ia;                                      // child rows [ia, ib) land in [r0, r1)
                if (jk >= 0) {
                    int lo = ia, hi = min(mcq, ia + kAsmChunk);
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if ((int)s_pos[mo + mid] < r1) lo = mid + 1; else hi = mid;
                    }
                    ib = lo;
                }
                unsigned act = __ballot_sync(0xffffffffu, jk >= 0 && ib > ia);
                __syncwarp();
                // children in order; the next child's run is loaded while the current one is added
                constexpr int UC = kAsmChunk / 32;
                double v[UC];
                int i0 = 0, i1 = 0, mof = 0;
                auto fetch = [&](int q, double* w, int& a0_, int& a1_, int& mo_) {
                    const int j = __shfl_sync(0xffffffffu, jk, q);
                    a0_ = __shfl_sync(0xffffffffu, ia, q);
                    a1_ = __shfl_sync(0xffffffffu, ib, q);
                    const AsmKid& k = s_kid[q];
                    mo_ = k.moff;
                    const double* __restrict__ colc = k.F + (size_t)(k.ec + j) * k.ldc + k.ec;
#pragma unroll
                    for (int u = 0; u < UC; ++u) {
                        const int i = a0_ + lane + 32 * u;
                        w[u] = i < a1_ ? colc[i] : 0.0;
                    }
                };
                if (act) { fetch(__ffs(act) - 1, v, i0, i1, mof); act &= act - 1; }
                for (bool more = i1 > i0; more;) {
                    double vn[UC];
                    int n0 = 0, n1 = 0, nmo = 0;
                    more = act != 0;
                    if (more) { fetch(__ffs(act) - 1, vn, n0, n1, nmo); act &= act - 1; }
#pragma unroll
                    for (int u = 0; u < UC; ++u) {
                        const int i = i0 + lane + 32 * u;
                        if (i < i1) buf[(int)s_pos[mof + i] - r0] += v[u];
                    }
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < UC; ++u) v[u] = vn[u];
                    i0 = n0; i1 = n1; mof = nmo;
                }
                ia = ib;
                double* dst = F + (size_t)c * ld;
#pragma unroll
                for (int u = 0; u < kAsmChunk / 32; ++u) {
                    const int r = r0 + lane + 32 * u;
                    if (r < r1) dst[r] = buf[lane + 32 * u];
                }
                __syncwarp();
            }
        }
    } else {
        for (int j = clo + warp; j < chi; j += kAsmNW)
            for (int i = j + lane; i < fo; i += 32) F[i + (size_t)j * ld] = 0.0;
        __syncthreads();
        const int e0 = clo < p ? acol[clo] : acol[p], e1 = clo < p ? acol[min(chi, p)] : acol[p];
        for (int e = e0 + tid; e < e1; e += kAsmThreads) {
            const uint32_t rc = P.asm_rc[a0 + e];
            const int lr = (int)(rc >> 16), lc = (int)(rc & 0xffffu);
            const int r = lr < p ? lr : lr + nd;
            const double v = fma(-sigma, P.b[a0 + e], alpha * P.a[a0 + e]);
            F[r + (size_t)lc * ld] = v;
            mx = fmax(mx, fabs(v));
        }
    }
    mx = block_max<kAsmThreads>(mx, s_red);                     // (barrier: the gathered columns are written)
    if (tid == 0 && mx > 0.0) atomic_max_pos_double(&st->smax_bits, mx);
    if (gather && !s_anyd) return;
    // RED adds, children in order: delayed columns only (gather path) or everything (plain path)
    int doffs = 0;
    for (int q = 0; q < nch; ++q) {
        const int c = P.child_list[c0 + q];
        const int ndo = nd_out[c];
        const int dof = p + doffs;
        doffs += ndo > 0 ? ndo : 0;
        if (gather && ndo <= 0) continue;
        const int fc = P.forder[c] + nd_in[c];
        const int ldc = ldpad(P.cap[c]);
        const int mc = ndo + P.ncb[c];
        const int ec = fc - mc;
        const double* __restrict__ Fc = arena + P.arena_off[c];
        const bool wup = P.flag[(size_t)sh * P.nf + c] == FL_OK && ndo > 0;
        const int32_t* __restrict__ rm = P.rmap + P.rmap_ptr[c];
        auto pos = [&](int x) -> int {
            if (x < ndo) return dof + x;
            const int r = rm[x - ndo];
            return r < p ? r : r + nd;
        };
        const int jend = gather ? ndo : mc;
        __syncthreads();                                          // previous child's adds issued in order
        for (int j = warp; j < jend; j += kAsmNW) {
            const int pj = pos(j);
            if (j >= ndo && (pj < clo || pj >= chi)) continue;
            const double* __restrict__ colc = Fc + (size_t)(ec + j) * ldc + ec;
            for (int i = j + lane; i < mc; i += 32) {
                const int pi = pos(i);
                const int hi = pi > pj ? pi : pj, lo = pi > pj ? pj : pi;
                if (lo < clo || lo >= chi) continue;
                const double v = (wup && j < ndo && i >= ndo) ? Fc[(ec + j) + (size_t)(ec + i) * ldc] : colc[i];
                atomicAdd(&F[hi + (size_t)lo * ld], v);
            }
        }
    }
}

__global__ void __launch_bounds__(kAsmThreads, 4) k_assemble(DevPlan P, const int4* __restrict__ items) {
    const int4 itm = items[blockIdx.x];
    assemble_strip(P, itm.x, itm.y, itm.z, 0);
}

// restore of fronts whose fast-path pass failed: the same assembly, flagged fronts only;
// item (front, x0, S, R): strips x0, x0 + R, ... (few CTAs per front: most fronts exit at once)
__global__ void __launch_bounds__(kAsmThreads, 4) k_reassemble(DevPlan P, const int4* __restrict__ items) {
    const int4 itm = items[blockIdx.x];
    for (int x = itm.y; x < itm.z; x += itm.w) {
        assemble_strip(P, itm.x, x, itm.z, 1);
        __syncthreads();
    }
}

// ---------------------------------------------------------------- a1 + a2, small fronts
// Levels of small fronts (short columns: the gather form's per-column child searches
// dominate there): whole-front CTAs (S per front when the level is small), zero-fill,
// stores, then the children's entries with fire-and-forget RED adds, children in order.
constexpr int kAsmRedThreads = 256;
constexpr int kAsmRedMapMax = 8192;       // child CB positions staged in shared memory

// One front of a level, S CTAs per front (blockIdx.x = front * S + x): CTA x
// owns the parent columns [lo, hi): zero-fill, original entries (alpha a - sigma b),
// then the children's CB entries landing in those columns, children in order.
// Each parent entry belongs to one CTA, so the sum order is fixed (deterministic).
__device__ __forceinline__ void assemble_front_red(const DevPlan& P, const int32_t* __restrict__ list, int S,
                                               int only_flagged) {
    const int s = list[blockIdx.x / S];
    const int xs = blockIdx.x % S;
    const int sh = blockIdx.y;
    if (only_flagged) {               // re-assembly of fronts whose fast-path pass failed (restore)
        const int fl = P.flag[(size_t)sh * P.nf + s];
        if (fl != FL_RERUN && fl != FL_REF) return;
    }
    ShiftStat* st = P.stats + sh;
    double* arena = P.arena + (size_t)sh * P.arena_stride;
    int32_t* nd_in = P.nd_in + (size_t)sh * P.nf;
    const int32_t* nd_out = P.nd_out + (size_t)sh * P.nf;
    int32_t* doff = P.doff + (size_t)sh * P.nf;
    __shared__ int s_nd, s_skip;
    __shared__ double s_red[32];
    __shared__ int s_pos[kAsmRedMapMax];
    const int c0 = P.child_ptr[s], c1 = P.child_ptr[s + 1];
    if (threadIdx.x == 0) {
        int off = 0, bad = 0;
        for (int q = c0; q < c1; ++q) {
            const int c = P.child_list[q];
            const int no = nd_out[c];
            if (no < 0) bad = 1;
            if (xs == 0) doff[c] = off;
            off += no > 0 ? no : 0;
        }
        const int need = P.forder[s] + off;
        if (need > P.cap[s]) {
            bad = 1;
            if (xs == 0) atomicMax(&st->need_slack, off);
        }
        if (bad && xs == 0) atomicOr(&st->flags, FLAG_OVERFLOW);
        s_skip = bad;
        s_nd = off;
        if (xs == 0) nd_in[s] = bad ? -1 : off;
    }
    __syncthreads();
    if (s_skip) return;
    const int nd = s_nd, p = P.npiv[s], fo = P.forder[s] + nd, ld = ldpad(P.cap[s]);   // order, leading dimension
    double* F = arena + P.arena_off[s];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kAsmRedThreads / 32;
    int clo, chi;
    tri_split(fo, S, xs, clo, chi);
    if (xs == 0) {   // labels of the FS positions: own pivots, then each child's delayed variables
        const AuxRec A = aux_rec(P, sh, s, P.cap[s] - P.ncb[s]);
        for (int i = threadIdx.x; i < p; i += kAsmRedThreads) A.label[i] = P.piv_first[s] + i;
        int off = 0;
        for (int q = c0; q < c1; ++q) {
            const int c = P.child_list[q];
            const int ndo = nd_out[c];
            if (ndo <= 0) continue;
            const AuxRec C = aux_rec(P, sh, c, P.cap[c] - P.ncb[c]);
            const int ec = P.npiv[c] + nd_in[c] - ndo;
            for (int j = threadIdx.x; j < ndo; j += kAsmRedThreads) A.label[p + off + j] = C.label[C.perm[ec + j]];
            off += ndo;
        }
    }
    for (int j = clo + warp; j < chi; j += nw)
        for (int i = j + lane; i < fo; i += 32) F[i + (size_t)j * ld] = 0.0;
    __syncthreads();
    const double sigma = P.sigma[sh], alpha = P.alpha[sh];
    double mx = 0.0;
    // original entries of the strip's columns only (they sit in the pivot columns; asm_col: first
    // entry of each local pivot column)
    const int32_t* acol = P.asm_col + P.piv_first[s] + s;
    const int64_t k0 = P.asm_ptr[s] + acol[min(clo, p)], k1 = P.asm_ptr[s] + acol[min(chi, p)];
    for (int64_t k = k0 + threadIdx.x; k < k1; k += kAsmRedThreads) {
        const uint32_t rc = P.asm_rc[k];
        const int lr = (int)(rc >> 16), lc = (int)(rc & 0xffffu);
        const int r = lr < p ? lr : lr + nd;
        const double v = fma(-sigma, P.b[k], alpha * P.a[k]);      // alpha A - sigma B (alpha = 1: A - sigma B)
        F[r + (size_t)lc * ld] = v;
        mx = fmax(mx, fabs(v));
    }
    mx = block_max<kAsmRedThreads>(mx, s_red);
    if (threadIdx.x == 0 && mx > 0.0) atomic_max_pos_double(&st->smax_bits, mx);
    // a2: extend-add, children in a fixed order
    int off = 0;
    for (int q = c0; q < c1; ++q) {
        const int c = P.child_list[q];
        const int ndo = nd_out[c];
        const int fc = P.forder[c] + nd_in[c];       // child order
        const int ldc = ldpad(P.cap[c]);             // child leading dimension
        const int mc = ndo + P.ncb[c];
        const int ec = fc - mc;
        const double* __restrict__ Fc = arena + P.arena_off[c];
        double* __restrict__ Fp = F;
        // fast-path children keep the CB rows of their delayed columns in W21 (upper part)
        const bool wup = P.flag[(size_t)sh * P.nf + c] == FL_OK && ndo > 0;
        const int32_t* __restrict__ rm = P.rmap + P.rmap_ptr[c];
        const int dof = p + off;
        off += ndo > 0 ? ndo : 0;
        const bool staged = mc <= kAsmRedMapMax;
        __syncthreads();                                         // s_pos reuse
        if (staged)
            for (int x = threadIdx.x; x < mc; x += kAsmRedThreads) {
                int v;
                if (x < ndo) v = dof + x;
                else { const int r = rm[x - ndo]; v = r < p ? r : r + nd; }
                s_pos[x] = v;
            }
        __syncthreads();
        auto pos = [&](int x) -> int {
            if (staged) return s_pos[x];
            if (x < ndo) return dof + x;
            const int r = rm[x - ndo];
            return r < p ? r : r + nd;
        };
        constexpr int U = 4;                                     // rows in flight per lane
        for (int j = warp; j < mc; j += nw) {
            const int pj = pos(j);
            // non-delayed child columns land in parent column pj (positions increase with the
            // child index there); delayed columns are filtered entry by entry
            if (j >= ndo && (pj < clo || pj >= chi)) continue;
            const double* __restrict__ colc = Fc + (size_t)(ec + j) * ldc + ec;
            for (int i0 = j; i0 < mc; i0 += 32 * U) {
                double v[U];
                size_t dst[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int i = i0 + lane + 32 * u;
                    dst[u] = SIZE_MAX;
                    v[u] = 0.0;
                    if (i < mc) {
                        const int pi = pos(i);
                        const int hi = pi > pj ? pi : pj, lo = pi > pj ? pj : pi;
                        if (lo >= clo && lo < chi) {
                            dst[u] = hi + (size_t)lo * ld;
                            v[u] = (wup && j < ndo && i >= ndo) ? __ldcs(Fc + (ec + j) + (size_t)(ec + i) * ldc)
                                                                : __ldcs(colc + i);   // read once: evict-first
                        }
                    }
                }
                // one writer per parent entry and child (children ordered by the barrier
                // between them): fire-and-forget RED adds, no load latency
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (dst[u] != SIZE_MAX) atomicAdd(&Fp[dst[u]], v[u]);
            }
        }
    }
}

// ---------------------------------------------------------------- a1 + a2, shared-memory strips
// One CTA per strip of a front (columns [clo, chi), at most kSmStripEnt lower entries): the strip
// is built in shared memory -- zero, the original entries (alpha a - sigma b), then each child's
// entries landing in it, children in order (one writer per entry and child: plain adds, no
// atomics; deterministic) -- and stored once, column by column, coalesced.  HBM traffic is the
// ideal one: 8 B written per front entry, every child entry read once (by the CTA owning its
// parent column), no zero-fill pass, no read-modify-write.
constexpr int kSmStripEnt = 4096;         // doubles of shared memory per strip (32 KB)
constexpr int kSmMap = 4096;              // child positions staged in shared memory

__global__ void __launch_bounds__(kAsmRedThreads, 5) k_asm_smem(DevPlan P, const int4* __restrict__ items) {
    extern __shared__ double sbuf[];                           // [kSmStripEnt]
    __shared__ uint16_t s_pos[kSmMap];
    __shared__ int s_nd, s_skip;
    __shared__ double s_red[32];
    const int4 itm = items[blockIdx.x];
    const int s = itm.x, xs = itm.y, S = itm.z;
    const int sh = blockIdx.y;
    ShiftStat* st = P.stats + sh;
    double* arena = P.arena + (size_t)sh * P.arena_stride;
    int32_t* nd_in = P.nd_in + (size_t)sh * P.nf;
    const int32_t* nd_out = P.nd_out + (size_t)sh * P.nf;
    int32_t* doff = P.doff + (size_t)sh * P.nf;
    const int c0 = P.child_ptr[s], c1 = P.child_ptr[s + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = kAsmRedThreads / 32;
    if (tid == 0) {
        int off = 0, bad = 0;
        for (int q = c0; q < c1; ++q) {
            const int c = P.child_list[q];
            const int no = nd_out[c];
            if (no < 0) bad = 1;
            if (xs == 0) doff[c] = off;
            off += no > 0 ? no : 0;
        }
        const int need = P.forder[s] + off;
        if (need > P.cap[s]) {
            bad = 1;
            if (xs == 0) atomicMax(&st->need_slack, off);
        }
        if (bad && xs == 0) atomicOr(&st->flags, FLAG_OVERFLOW);
        s_skip = bad;
        s_nd = off;
        if (xs == 0) nd_in[s] = bad ? -1 : off;
    }
    __syncthreads();
    if (s_skip) return;
    const int nd = s_nd, p = P.npiv[s], fo = P.forder[s] + nd, ld = ldpad(P.cap[s]);
    double* F = arena + P.arena_off[s];
    if (xs == 0) {   // labels of the FS positions: own pivots, then each child's delayed variables
        const AuxRec A = aux_rec(P, sh, s, P.cap[s] - P.ncb[s]);
        for (int i = tid; i < p; i += kAsmRedThreads) A.label[i] = P.piv_first[s] + i;
        int off = 0;
        for (int q = c0; q < c1; ++q) {
            const int c = P.child_list[q];
            const int ndo = nd_out[c];
            if (ndo <= 0) continue;
            const AuxRec C = aux_rec(P, sh, c, P.cap[c] - P.ncb[c]);
            const int ec = P.npiv[c] + nd_in[c] - ndo;
            for (int j = tid; j < ndo; j += kAsmRedThreads) A.label[p + off + j] = C.label[C.perm[ec + j]];
            off += ndo;
        }
    }
    int clo, chi;
    tri_split(fo, S, xs, clo, chi);
    // entry offset of column j (row j) inside the strip
    auto colbase = [&](int j) -> int {
        return (int)((int64_t)(j - clo) * fo - (((int64_t)j * (j - 1) - (int64_t)clo * (clo - 1)) >> 1));
    };
    const int ent = colbase(chi);
    for (int x = tid; x < ent; x += kAsmRedThreads) sbuf[x] = 0.0;
    __syncthreads();
    const double sigma = P.sigma[sh], alpha = P.alpha[sh];
    double mx = 0.0;
    {   // original entries of the strip's columns (asm_col: first entry of each local pivot column)
        const int64_t a0 = P.asm_ptr[s];
        const int32_t* acol = P.asm_col + P.piv_first[s] + s;
        const int jl = min(clo, p), jh = min(chi, p);
        const int64_t k0 = a0 + acol[jl], k1 = a0 + acol[jh];
        for (int64_t k = k0 + tid; k < k1; k += kAsmRedThreads) {
            const uint32_t rc = P.asm_rc[k];
            const int lr = (int)(rc >> 16), lc = (int)(rc & 0xffffu);
            const int r = lr < p ? lr : lr + nd;
            const double v = fma(-sigma, P.b[k], alpha * P.a[k]);
            sbuf[colbase(lc) + (r - lc)] = v;
            mx = fmax(mx, fabs(v));
        }
    }
    mx = block_max<kAsmRedThreads>(mx, s_red);               // (barrier: originals are in)
    if (tid == 0 && mx > 0.0) atomic_max_pos_double(&st->smax_bits, mx);
    int off = 0;
    for (int q = c0; q < c1; ++q) {
        const int c = P.child_list[q];
        const int ndo = nd_out[c] > 0 ? nd_out[c] : 0;
        const int fc = P.forder[c] + nd_in[c];
        const int ldc = ldpad(P.cap[c]);
        const int mc = ndo + P.ncb[c];
        const int ec = fc - mc;
        const double* __restrict__ Fc = arena + P.arena_off[c];
        const bool wup = P.flag[(size_t)sh * P.nf + c] == FL_OK && ndo > 0;
        const int32_t* __restrict__ rm = P.rmap + P.rmap_ptr[c];
        const int dof = p + off;
        off += ndo;
        const bool staged = mc <= kSmMap;
        __syncthreads();                                      // previous child's adds and s_pos reads done
        if (staged)
            for (int x = tid; x < mc; x += kAsmRedThreads) {
                int v;
                if (x < ndo) v = dof + x;
                else { const int r = rm[x - ndo]; v = r < p ? r : r + nd; }
                s_pos[x] = (uint16_t)v;
            }
        __syncthreads();
        auto pos = [&](int x) -> int {
            if (staged) return s_pos[x];
            if (x < ndo) return dof + x;
            const int r = rm[x - ndo];
            return r < p ? r : r + nd;
        };
        // non-delayed child columns landing in the strip: a contiguous range (positions increase)
        int xa = ndo, xb = mc;
        {
            int lo = ndo, hi = mc;                            // first x with pos(x) >= clo
            while (lo < hi) { const int m = (lo + hi) >> 1; if (pos(m) < clo) lo = m + 1; else hi = m; }
            xa = lo;
            hi = mc;                                          // first x with pos(x) >= chi
            while (lo < hi) { const int m = (lo + hi) >> 1; if (pos(m) < chi) lo = m + 1; else hi = m; }
            xb = lo;
        }
        for (int x = xa + warp; x < xb; x += nw) {
            const int pj = pos(x);
            const int cb = colbase(pj) - pj;
            const double* __restrict__ colc = Fc + (size_t)(ec + x) * ldc + ec;
            constexpr int U = 4;                              // loads in flight per lane
            for (int y0 = x + lane; y0 < mc; y0 += 32 * U) {
                double v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) { const int y = y0 + 32 * u; v[u] = y < mc ? __ldg(colc + y) : 0.0; }
#pragma unroll
                for (int u = 0; u < U; ++u) { const int y = y0 + 32 * u; if (y < mc) sbuf[cb + pos(y)] += v[u]; }
            }
        }
        // delayed columns (rare): every entry filtered by its lower-triangle column
        for (int x = warp; x < ndo; x += nw) {
            const int pj = pos(x);
            for (int y = x + lane; y < mc; y += 32) {
                const int pi = pos(y);
                const int hi = pi > pj ? pi : pj, lo = pi > pj ? pj : pi;
                if (lo < clo || lo >= chi) continue;
                const double v = (wup && y >= ndo) ? Fc[(ec + x) + (size_t)(ec + y) * ldc]
                                                   : Fc[(ec + y) + (size_t)(ec + x) * ldc];
                sbuf[colbase(lo) + (hi - lo)] += v;
            }
        }
    }
    __syncthreads();
    for (int j = clo + warp; j < chi; j += nw) {               // one coalesced store per column
        const int cb = colbase(j) - j;
        double* __restrict__ Fj = F + (size_t)j * ld;
        for (int i = j + lane; i < fo; i += 32) Fj[i] = sbuf[cb + i];
    }
}

__global__ void __launch_bounds__(kAsmRedThreads) k_assemble_red(DevPlan P, const int32_t* __restrict__ list, int S) {
    assemble_front_red(P, list, S, 0);
}


// ---------------------------------------------------------------- a3 + a4 + a5 (reference)
constexpr int kRefThreads = 256;

__device__ void sym_swap(double* F, int ld, int f, int a, int b) {
    // symmetric row/column interchange of positions a < b (lower storage)
    if (a == b) return;
    for (int t = threadIdx.x; t < f; t += blockDim.x) {
        if (t < a) {
            double x = F[a + (size_t)t * ld]; F[a + (size_t)t * ld] = F[b + (size_t)t * ld]; F[b + (size_t)t * ld] = x;
        } else if (t == a) {
            double x = F[a + (size_t)a * ld]; F[a + (size_t)a * ld] = F[b + (size_t)b * ld]; F[b + (size_t)b * ld] = x;
        } else if (t < b) {
            double x = F[t + (size_t)a * ld]; F[t + (size_t)a * ld] = F[b + (size_t)t * ld]; F[b + (size_t)t * ld] = x;
        } else if (t > b) {
            double x = F[t + (size_t)a * ld]; F[t + (size_t)a * ld] = F[t + (size_t)b * ld]; F[t + (size_t)b * ld] = x;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kRefThreads) k_factor_ref(DevPlan P, const int32_t* __restrict__ fronts, int only_flagged) {
    const int s = fronts[blockIdx.x];
    const int sh = blockIdx.y;
    if (only_flagged && P.flag[(size_t)sh * P.nf + s] == 0) return;   // fast path kept this front
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
    const int f = P.forder[s] + nd, q = p + nd, ld = ldpad(P.cap[s]);
    const bool root = (c == 0);
    const double u = P.u;
    const AuxRec A = aux_rec(P, sh, s, P.cap[s] - c);
    if (threadIdx.x == 0) P.flag[(size_t)sh * P.nf + s] = FL_REF;      // factor layout: all of L in the lower part
    for (int i = threadIdx.x; i < q; i += kRefThreads) A.perm[i] = i;
    __syncthreads();
    __shared__ MaxIdx s_mi[32];
    __shared__ double s_red[32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = kRefThreads / 32;
    unsigned long long c_neg = 0, c_zero = 0, c_pos = 0, c_2x2 = 0, c_del = 0;
    double minpiv = DBL_MAX;
    int e = 0, qe = q;
    while (e < qe) {
        const int k = e;
        // column k: FS candidates (k, qe) -> (gC, r); all active rows (k, f) -> gR
        MaxIdx mC{-1.0, INT_MAX};
        double mR = 0.0;
        for (int i = k + 1 + tid; i < f; i += kRefThreads) {
            const double x = fabs(F[i + (size_t)k * ld]);
            if (i < qe) mC = better(mC, MaxIdx{x, i});
            mR = fmax(mR, x);
        }
        mC = block_max_idx<kRefThreads>(mC, s_mi);
        const double gR = block_max<kRefThreads>(mR, s_red);
        double gC = mC.v > 0.0 ? mC.v : 0.0;
        const int r = mC.v >= 0.0 ? mC.i : k;
        const double akk = fabs(F[k + (size_t)k * ld]);
        if (akk == 0.0 && gR == 0.0) {          // zero column: exact zero pivot
            if (threadIdx.x == 0) { A.kind[k] = PK_ZERO; A.d[k] = 0.0; A.ds[k] = 0.0; }
            c_zero++;
            minpiv = 0.0;
            e++;
            continue;
        }
        int kind = 1, j = k;
        double rho = 0.0;
        if (akk < kAlpha * gC) {
            double m = 0.0;
            for (int i = k + tid; i < qe; i += kRefThreads)
                if (i != r) m = fmax(m, fabs(symget(F, ld, i, r)));
            rho = block_max<kRefThreads>(m, s_red);
            if (akk * rho >= kAlpha * gC * gC) { kind = 1; j = k; }
            else if (fabs(F[r + (size_t)r * ld]) >= kAlpha * rho) { kind = 1; j = r; }
            else { kind = 2; j = r; }
        }
        if (!root) {
            bool ok;
            if (kind == 1) {
                double cm;
                if (j == k) cm = gR;
                else {
                    double m = 0.0;
                    for (int i = k + tid; i < f; i += kRefThreads)
                        if (i != j) m = fmax(m, fabs(symget(F, ld, i, j)));
                    cm = block_max<kRefThreads>(m, s_red);
                }
                ok = fabs(F[j + (size_t)j * ld]) >= u * cm;
            } else {
                double m1 = 0.0, m2 = 0.0;
                for (int i = k + tid; i < f; i += kRefThreads) {
                    if (i != k && i != r) {
                        m1 = fmax(m1, fabs(F[i + (size_t)k * ld]));
                        m2 = fmax(m2, fabs(symget(F, ld, i, r)));
                    }
                }
                const double gk = block_max<kRefThreads>(m1, s_red);
                const double gr = block_max<kRefThreads>(m2, s_red);
                const double a11 = F[k + (size_t)k * ld], a21 = F[r + (size_t)k * ld], a22 = F[r + (size_t)r * ld];
                const double det = a11 * a22 - a21 * a21;
                if (det == 0.0) ok = false;
                else {
                    const double ad = fabs(det);
                    const double t1 = (fabs(a22) * gk + fabs(a21) * gr) / ad;
                    const double t2 = (fabs(a21) * gk + fabs(a11) * gr) / ad;
                    ok = t1 <= 1.0 / u && t2 <= 1.0 / u;
                }
            }
            __syncthreads();                      // every thread has read the pivot entries
            if (!ok) {                            // delay column k to the parent
                if (threadIdx.x == 0) { const int x = A.perm[k]; A.perm[k] = A.perm[qe - 1]; A.perm[qe - 1] = x; }
                sym_swap(F, ld, f, k, qe - 1);
                qe--;
                c_del++;
                continue;
            }
        }
        if (root) __syncthreads();                // (non-root fronts synchronised above)
        if (kind == 1) {
            if (threadIdx.x == 0 && j != k) { const int x = A.perm[k]; A.perm[k] = A.perm[j]; A.perm[j] = x; }
            sym_swap(F, ld, f, k, j);
            const double d = F[k + (size_t)k * ld];
            if (threadIdx.x == 0) { A.kind[k] = PK_1X1; A.d[k] = d; A.ds[k] = 0.0; }
            const double dinv = 1.0 / d;
            for (int jj = k + 1 + warp; jj < f; jj += nw) {
                const double wj = F[jj + (size_t)k * ld] * dinv;
                double* colj = F + (size_t)jj * ld;
                const double* colk = F + (size_t)k * ld;
                for (int i = jj + lane; i < f; i += 32) colj[i] = fma(-colk[i], wj, colj[i]);
            }
            __syncthreads();
            for (int i = k + 1 + tid; i < f; i += kRefThreads) F[i + (size_t)k * ld] *= dinv;
            __syncthreads();
            if (d < 0.0) c_neg++; else if (d > 0.0) c_pos++; else c_zero++;
            minpiv = fmin(minpiv, fabs(d));
            e += 1;
        } else {
            if (threadIdx.x == 0 && r != k + 1) { const int x = A.perm[k + 1]; A.perm[k + 1] = A.perm[r]; A.perm[r] = x; }
            sym_swap(F, ld, f, k + 1, r);
            const double d11 = F[k + (size_t)k * ld], d21 = F[k + 1 + (size_t)k * ld], d22 = F[k + 1 + (size_t)(k + 1) * ld];
            if (threadIdx.x == 0) {
                A.kind[k] = PK_2X2A; A.d[k] = d11; A.ds[k] = d21;
                A.kind[k + 1] = PK_2X2B; A.d[k + 1] = d22; A.ds[k + 1] = 0.0;
            }
            const double det = d11 * d22 - d21 * d21;
            const double i11 = d22 / det, i21 = -d21 / det, i22 = d11 / det;
            const double* col1 = F + (size_t)k * ld;
            const double* col2 = F + (size_t)(k + 1) * ld;
            for (int jj = k + 2 + warp; jj < f; jj += nw) {
                const double w1 = col1[jj], w2 = col2[jj];
                const double l1 = w1 * i11 + w2 * i21, l2 = w1 * i21 + w2 * i22;
                double* colj = F + (size_t)jj * ld;
                for (int i = jj + lane; i < f; i += 32) colj[i] = colj[i] - col1[i] * l1 - col2[i] * l2;
            }
            __syncthreads();
            for (int i = k + 2 + tid; i < f; i += kRefThreads) {
                const double w1 = F[i + (size_t)k * ld], w2 = F[i + (size_t)(k + 1) * ld];
                F[i + (size_t)k * ld] = w1 * i11 + w2 * i21;
                F[i + (size_t)(k + 1) * ld] = w1 * i21 + w2 * i22;
            }
            __syncthreads();
            // a5: sign(det) in the scaled form (d11/d21)(d22/d21) - 1
            const double t = (d11 / d21) * (d22 / d21) - 1.0;
            if (t < 0.0) { c_neg++; c_pos++; }
            else if (t > 0.0) { if (d11 < 0.0) c_neg += 2; else c_pos += 2; }
            else { c_zero++; if (d11 + d22 < 0.0) c_neg++; else c_pos++; }
            const double tr = 0.5 * (d11 + d22);
            const double disc = sqrt(0.25 * (d11 - d22) * (d11 - d22) + d21 * d21);
            const double big = fabs(tr) + disc;
            minpiv = fmin(minpiv, big > 0.0 ? fabs(det) / big : 0.0);
            c_2x2++;
            e += 2;
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

__global__ void k_gather(const double* __restrict__ src, const int64_t* __restrict__ idx,
                         double* __restrict__ dst, int64_t n) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = src[idx[k]];
}

__global__ void k_reset_stats(ShiftStat* st, int batch) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < batch) {
        ShiftStat z;
        z.n_neg = z.n_zero = z.n_pos = z.n_2x2 = z.n_delayed = z.n_redo = 0;
        z.minpiv_bits = (unsigned long long)__double_as_longlong(DBL_MAX);
        z.smax_bits = 0;
        z.flags = 0;
        z.need_slack = 0;
        st[i] = z;
    }
}

}  // namespace

// items: (front, strip x, strips S, R) per CTA (api.cu build_lists)
void launch_assemble(const DevPlan& P, const int4* items, int nitems, int batch, bool only_flagged, cudaStream_t st) {
    if (nitems <= 0) return;
    const size_t smem = sizeof(double) * kAsmNW * kAsmChunk;
    static unsigned long long attr = 0;                 // static + dynamic shared memory above 48 KB: opt in
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(k_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_reassemble, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        
    }
    if (only_flagged) k_reassemble<<<dim3(nitems, batch), kAsmThreads, smem, st>>>(P, items);
    else k_assemble<<<dim3(nitems, batch), kAsmThreads, smem, st>>>(P, items);
}

int smem_strips(int cap) {
    const int64_t T = (int64_t)cap * (cap + 1) / 2;
    const int64_t room = kSmStripEnt - cap;                    // a strip holds T / S entries + one column
    return room <= 0 ? 0 : (int)std::max<int64_t>(1, (T + room - 1) / room);
}

void launch_asm_smem(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st) {
    if (nitems <= 0) return;
    const size_t smem = sizeof(double) * kSmStripEnt;
    static unsigned long long attr = 0;
    if (first_on_device(attr)) cudaFuncSetAttribute(k_asm_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_asm_smem<<<dim3(nitems, batch), kAsmRedThreads, smem, st>>>(P, items);
}

int assembly_strips(int forder) {
    const int64_t T = (int64_t)forder * (forder + 1) / 2;
    return (int)std::max<int64_t>(1, (T + kAsmStripEnt - 1) / kAsmStripEnt);
}

void launch_assemble_red(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int fmax, cudaStream_t st) {
    if (nfronts <= 0) return;
    // CTAs per front: enough to give ~4 resident CTAs per SM on the whole level (column strips of at
    // most 64 KB for L2 residency between the zero fill and the RED adds were measured slower at c4:
    // 8192 entries 122 ms, 16384 97 ms, whole fronts 95 ms per 8-shift batch)
    (void)fmax;
    int S = (int)((4 * 148 + (int64_t)nfronts * batch - 1) / ((int64_t)nfronts * batch));
    S = std::max(1, std::min(S, 16));
    k_assemble_red<<<dim3(nfronts * S, batch), kAsmRedThreads, 0, st>>>(P, fronts, S);
}

void launch_factor_list(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, cudaStream_t st,
                        bool only_flagged) {
    if (nfronts <= 0) return;
    k_factor_ref<<<dim3(nfronts, batch), kRefThreads, 0, st>>>(P, fronts, only_flagged ? 1 : 0);
}

void launch_gather(const double* src, const int64_t* idx, double* dst, int64_t n, cudaStream_t st) {
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (blocks < 1) blocks = 1;
    k_gather<<<blocks, 256, 0, st>>>(src, idx, dst, n);
}

void launch_reset_stats(ShiftStat* st, int batch, cudaStream_t s) {
    k_reset_stats<<<(batch + 127) / 128, 128, 0, s>>>(st, batch);
}

}  // namespace kep
