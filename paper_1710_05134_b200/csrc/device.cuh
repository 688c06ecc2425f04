// device.cuh — device-side plan, per-shift state and shared helpers.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace kep {

// Per-shift counters (one per shift of a batch); reset before every batch.
struct ShiftStat {
    unsigned long long n_neg, n_zero, n_pos, n_2x2, n_delayed, n_redo;
    unsigned long long minpiv_bits;   // min |pivot| as positive-double bits (init +inf)
    unsigned long long smax_bits;     // max |a - sigma b| as positive-double bits (init 0)
    int flags;                        // bit 0: delayed-pivot slack overflow
    int need_slack;                   // largest (nd_in) seen that overflowed
};

constexpr int FLAG_OVERFLOW = 1;

// Static per-pattern plan + batch state, passed by value to every kernel.
struct DevPlan {
    int32_t nf;
    const int32_t* forder;       // f_s (no delays)
    const int32_t* npiv;         // p_s
    const int32_t* ncb;          // c_s
    const int32_t* cap;          // f_s + slack
    const int32_t* child_ptr;
    const int32_t* child_list;
    const int32_t* level_fronts;
    const int32_t* piv_first;    // [nf+1] first pivot position of each front
    const int32_t* cb_ptr;       // [nf+1]
    const int32_t* cb_rows;      // CB row positions of each front
    const int64_t* arena_off;    // doubles, within one shift's arena
    const int64_t* asm_ptr;
    const uint32_t* asm_rc;      // (lrow << 16) | lcol
    const int32_t* asm_col;      // [piv_first[s] + s + j] first entry of local column j (j <= p), relative to asm_ptr[s]
    const double* a;             // A values in assembly order
    const double* b;             // B values in assembly order
    const int64_t* rmap_ptr;
    const int32_t* rmap;
    // batch state
    double* arena;               // [batch][arena_stride]
    int64_t arena_stride;
    int32_t* nd_in;              // [batch][nf]
    int32_t* nd_out;             // [batch][nf]
    int32_t* doff;               // [batch][nf] offset of a child's delayed block in its parent
    ShiftStat* stats;            // [batch]
    const double* sigma;         // [batch]
    const double* alpha;         // [batch] the front assembles alpha A - sigma B (1 except for B-solves)
    double u;                    // threshold pivoting parameter
    // fast path (kernels_front.cu): per-front pivot records and redo flags
    double* aux;                 // [batch][aux_stride]
    int64_t aux_stride;          // doubles per shift
    const int64_t* aux_off;      // [nf] record offset (entries; AUX_W doubles each)
    int32_t* flag;               // [batch][nf] fast-path state of the front, FL_* below
    int32_t* forced;             // [batch][nf][FMAX+1] count, then S1 steps at which to delay
    int32_t* fstate;             // [batch][nf][FSTATE_W] k_fsp state: e, qe, step, forced cursor, block start
    int32_t* pending;            // count of fronts flagged FL_RERUN in the current level
    double* gscratch;            // [batch][gscratch_stride] k_fsp block columns of FS blocks too large for smem
    int64_t gscratch_stride;
    const int64_t* goff;         // [nf] scratch offset, -1 = shared memory
    double* xscr;                // [batch][xstride] k_l21x_prep blocks X = [L_bb^-T | L_bb^-T D^-1 M] (one level)
    int64_t xstride;
    const int64_t* xoff;         // [nf] offset in the level's X scratch (k_l21<2> fronts)
    int32_t debug;               // KEP_DEBUG set: diagnostic printf in rare paths
    // TMA: one 2-D tensor map (x = ld doubles, y = arena rows of ld) per distinct leading dimension
    // and shift of the batch; fronts start at multiples of their ld (plan_memory)
    const CUtensorMap* tmaps;    // [batch][ntmap]
    const int32_t* tmap_idx;     // [nf] index of the front's leading dimension
    int32_t ntmap;
};

// pivot kinds recorded per eliminated position
constexpr int PK_1X1 = 0, PK_2X2A = 1, PK_2X2B = 2, PK_ZERO = 3;
constexpr int AUX_W = 11;        // doubles per position: diag backup, d, ds, fa, fb, cm, (kind, perm), (step, label),
                                 // sgn, gca, gcb
// front states: FL_OK = factorised, FL_REF = hand to the unblocked kernel,
// FL_RERUN = rerun the fast path with one more forced delay, FL_ACTIVE = in the current fast pass
// FL_REFN = handed to the unblocked kernel by this pass's k_check (k_rerun_lists re-assembles it once
// and turns it into FL_REF)
constexpr int FL_OK = 0, FL_REF = 1, FL_RERUN = 2, FL_ACTIVE = 3, FL_REFN = 5;
constexpr int FSTATE_W = 8;
constexpr int FMAX = 6;          // forced delays per front before falling back to the unblocked kernel

struct AuxRec {
    double *diag, *d, *ds, *fa, *fb;
    unsigned long long* cm;      // CB column maxima of W21 (positive-double bits)
    int *kind, *perm, *step;
    int* label;                  // assembly-order variable (elimination position) of each FS position
    double* sgn;                 // +-1: sign of the eigenvalue of D carried by the G column (k_schur)
    double *gca, *gcb;           // G[:, t] = W21[:, t] gca[t] + W21[:, t +- 1] gcb[t] (2x2 partner)
};

__device__ __forceinline__ AuxRec aux_rec(const DevPlan& P, int sh, int s, int Q) {
    double* b = P.aux + (size_t)sh * P.aux_stride + (size_t)P.aux_off[s] * AUX_W;
    AuxRec A;
    A.diag = b; A.d = b + Q; A.ds = b + 2 * Q; A.fa = b + 3 * Q; A.fb = b + 4 * Q;
    A.cm = (unsigned long long*)(b + 5 * Q);
    A.kind = (int*)(b + 6 * Q);
    A.perm = A.kind + Q;
    A.step = (int*)(b + 7 * Q);
    A.label = A.step + Q;
    A.sgn = b + 8 * Q;
    A.gca = b + 9 * Q;
    A.gcb = b + 10 * Q;
    return A;
}

// Eigen-decomposition of a 2x2 pivot block D = [d11 d21; d21 d22] = Q diag(l1, l2) Q^T,
// Q = [cs -sn; sn cs] (Jacobi rotation).  With it the Schur update of a front is
// W21 D^-1 W21^T = G S G^T,  G = W21 Q |Lambda|^-1/2 S,  S = sign(Lambda)
// (1x1 pivots: G = W21 sign(d) / sqrt|d|), so k_schur multiplies G by G with sign
// flips only.
__device__ __forceinline__ void pair_eig(double d11, double d21, double d22, double& cs, double& sn, double& l1,
                                         double& l2) {
    const double th = 0.5 * atan2(2.0 * d21, d11 - d22);
    cs = cos(th);
    sn = sin(th);
    l1 = d11 * cs * cs + 2.0 * d21 * cs * sn + d22 * sn * sn;
    l2 = d11 * sn * sn - 2.0 * d21 * cs * sn + d22 * cs * cs;
}

// Leading dimension of a front of order f: even, so rows start 16-byte aligned
// (arena offsets are 256-byte aligned) and the GEMM kernels stage with 16-byte copies.
__host__ __device__ __forceinline__ int ldpad(int f) { return (f + 1) & ~1; }

// Shared-memory opt-in (cudaFuncSetAttribute) applies per device: `mask` holds one bit per
// device ordinal; returns true the first time it is called for the current device.
inline bool first_on_device(unsigned long long& mask) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    const unsigned long long old = __atomic_fetch_or(&mask, bit, __ATOMIC_ACQ_REL);
    return (old & bit) == 0;
}

__device__ __forceinline__ void atomic_max_pos_double(unsigned long long* addr, double v) {
    atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_min_pos_double(unsigned long long* addr, double v) {
    atomicMin(addr, (unsigned long long)__double_as_longlong(v));
}

// Retained factors of one shift (kep_factor; kernels_solve.cu).  Per front s:
// panel f_s x e_s (ld f_s) at panel + poff[s], row labels at lab + loff[s],
// D / kind at qoff[s] (same entry offsets as the aux records), hdr = (e, f, q, path).
struct StorePlan {
    double* panel;
    const int64_t* poff;
    int32_t* lab;
    const int64_t* loff;
    double* d;
    double* ds;
    int32_t* kind;
    int32_t* perm;               // [qoff] local pivot permutation of the FS positions (k_fwd's extend-add)
    const int64_t* qoff;
    int4* hdr;
    // solve scratch: per front the update vector passed to the parent (f - e rows, at uoff = loff)
    // and, for fronts too large for shared memory, the front vector itself (at yoff, -1 otherwise)
    double* upd;
    double* ybuf;
    const int64_t* yoff;
};

// Launchers (kernels.cu, kernels_front.cu, kernels_fast.cu, kernels_solve.cu)
void launch_assemble(const DevPlan& P, const int4* items, int nitems, int batch, bool only_flagged, cudaStream_t st);
void launch_assemble_red(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int fmax, cudaStream_t st);
int assembly_strips(int forder);     // CTAs (column strips) per front of the given order
int smem_strips(int cap);            // k_asm_smem strips of a front of capacity cap (0: too large)
void launch_asm_smem(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st);
void launch_fsp(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int qmax, int mode, cudaStream_t st);
void launch_fsu(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st);
int fs_iters(int qmax, int64_t nblocks);   // k_fsp launches that finish every front of a level
double fs_cost(int qmax, int64_t nblocks);  // planning model of a group's k_fsp/k_fsu passes
bool fs_uses_gls(int qmax);                 // the level's block columns live in global scratch
int fs_rows_pad(int qmax);
size_t fs_gls_doubles(int nb, int RS);
void launch_store(const DevPlan& P, const StorePlan& T, const int32_t* fronts, int nfronts, cudaStream_t st);
void launch_fwd(const DevPlan& P, const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, double* x,
                cudaStream_t st);
void launch_bwd(const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, double* x, cudaStream_t st);
int solve_max_front();       // largest front whose solve vectors fit shared memory
int solve_big_front();       // fronts larger than this: blocked multi-CTA solves (vectors in global scratch)
void launch_fwd_big(const DevPlan& P, const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, int emax,
                    double* x, cudaStream_t st);
void launch_bwd_big(const StorePlan& T, const int32_t* fronts, int nfronts, int fmax, int emax, double* x,
                    cudaStream_t st);
// kth.cu: Lanczos building blocks
void launch_spmv2(const int64_t* rp, const int32_t* ci, const double* va, const double* vb, const double* x, double* ya,
                  double* yb, int64_t n, cudaStream_t st);
void launch_gemv_t(const double* V, int64_t ldv, int j, const double* r, int64_t n, double* out, cudaStream_t st);
void launch_combine(const double* V, int64_t ldv, int j, const double* c, double cv, double beta_y, double* y,
                    double a1, const double* x1, double a2, const double* x2, int64_t n, cudaStream_t st);
void launch_ritz(const double* W, int64_t ldw, int j, const double* C, const double* r, const double* g, int m,
                 double* X, int64_t ldx, int64_t n, cudaStream_t st);
void launch_l21(const DevPlan& P, const int4* items, int nitems, int batch, int mode, cudaStream_t st);
int l21_mode(int qcap);              // 1: k_l21d<64,1> (q <= 64); 3: k_l21d<128,4> (q <= 128); 2: GEMM in-block solve (X scratch); 0: triangle
int64_t l21_x_doubles(int qcap);     // X scratch of one front (k_l21x_prep)
// compact per-pass lists of the fronts flagged for a rerun (k_rerun_lists)
struct RerunLists {
    const int4 *d1, *d2;         // [nf] per fast front: (l21 mode, l21 item off, cnt, uitem off), (ucnt, re-assembly off, cnt, -)
    const int4* sl[4];           // static l21 item lists by mode
    const int4 *su, *sa;         // static k_fsu tiles, re-assembly strips
    int32_t* fr;                 // out: fronts flagged FL_RERUN (re-assembly strips: FL_RERUN or FL_REF)
    int4* l[4];                  // out: their l21 tiles by mode
    int4 *u, *a;                 // out: their k_fsu tiles, re-assembly strips
    int32_t* x;                  // out: their k_l21x_prep fronts
    int32_t* cnt;                // out [8]: fronts, l21 modes 0 1 2, fsu, re-assembly, prep, l21 mode 3
};
void launch_rerun_lists(const DevPlan& P, const int32_t* fl, int n, int batch, const RerunLists& R, cudaStream_t st);
void launch_l21x_prep(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, cudaStream_t st);
void launch_check(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, cudaStream_t st);
int front_nb_for(int qmax, int64_t nblocks = 0);   // block width (0: too large, use the reference kernel)
void launch_schur(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st);
void launch_schur_tma(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st);
// host: encode the 2-D tensor map of one (arena base, leading dimension) pair (TMA box 16 x 64 doubles,
// 128-byte swizzle); false if the driver entry point is unavailable
bool encode_front_tmap(CUtensorMap* out, double* arena_base, int64_t arena_doubles, int ld);
void launch_schur_small(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int cmax, int kmax,
                        cudaStream_t st);
bool schur_small_ok(int c, int qcap);     // front handled by k_schur_small
void launch_factor_list(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, cudaStream_t st,
                        bool only_flagged = false);
// kernels_resid.cu: front-local factor residual (kep_factor_residual)
int resid_tile();
void launch_capture(const DevPlan& P, const int32_t* fronts, int nfronts, double* F0, cudaStream_t st);
void launch_resid(const DevPlan& P, const StorePlan& T, const int4* items, int nitems, const double* F0, double* out,
                  cudaStream_t st);
// kernels_small.cu: whole-panel-in-shared-memory partial LDL^T of small fronts
void launch_small(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int cap_doubles, int threads,
                  cudaStream_t st);
// kernels_big.cu: multi-CTA partial LDL^T of the large fronts of the top levels
int big_block();
size_t big_scratch_doubles(int cap, int ncta);
int big_blocks(int qmax);        // k_bigp launches that finish every group of FS capacity <= qmax
void launch_big_init(const DevPlan& P, const int2* groups, int ngroups, const int64_t* scroff, double* scr, int* state,
                     unsigned* bars, cudaStream_t st);
void launch_big_panel(const DevPlan& P, const int2* groups, int ngroups, int ncta, const int64_t* scroff, double* scr,
                      int* state, unsigned* bars, cudaStream_t st);
void launch_big_update(const DevPlan& P, const int2* groups, int ngroups, const int64_t* scroff, double* scr,
                       int* state, unsigned* bars, cudaStream_t st);
void launch_big_fin(const DevPlan& P, const int2* groups, int ngroups, const int64_t* scroff, double* scr, int* state,
                    unsigned* bars, cudaStream_t st);
void launch_gather(const double* src, const int64_t* idx, double* dst, int64_t n, cudaStream_t st);
void launch_reset_stats(ShiftStat* st, int batch, cudaStream_t s);

}  // namespace kep

#include <vector>
namespace kep {
bool tridiag_eigen(std::vector<double>& d, std::vector<double> e, std::vector<double>& Z);
}  // namespace kep
