// api.cu — the C ABI (include/kep.h): context, device memory, shift batches.
//
// Boundary of SURVEY.md §8(b): kep_analyze (pattern-only setup, untimed),
// kep_set_values, kep_inertia / kep_inertia_many (the timed hot path).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <ctime>
#include <numeric>
#include <cstdio>
#include <cstdlib>
#include <cfloat>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/kep.h"
#include "device.cuh"
#include "symbolic.h"

using kep::DevPlan;
using kep::ShiftStat;
using kep::Symbolic;

struct kep_ctx {
    Symbolic sym;
    kep_opts opts;
    std::string err;
    bool have_device = false;
    int device = -1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool values_set = false;
    int batch_cap = 1;
    // device arrays (static)
    int32_t *d_forder = nullptr, *d_npiv = nullptr, *d_ncb = nullptr, *d_cap = nullptr;
    int32_t *d_child_ptr = nullptr, *d_child_list = nullptr, *d_level_fronts = nullptr;
    int32_t *d_piv_first = nullptr, *d_cb_ptr = nullptr, *d_cb_rows = nullptr;
    int64_t *d_perm = nullptr, *d_iperm = nullptr;          // elimination position <-> dof
    // full symmetric CSR of the union pattern (stage-1/3 SpMV): 20 B per stored nonzero
    int64_t *d_csr_rp = nullptr, *d_csr_src = nullptr;
    int32_t* d_csr_ci = nullptr;
    double *d_csr_a = nullptr, *d_csr_b = nullptr;
    int64_t csr_nnz = 0;
    int64_t *d_arena_off = nullptr, *d_asm_ptr = nullptr, *d_asm_src = nullptr, *d_rmap_ptr = nullptr;
    uint32_t* d_asm_rc = nullptr;
    int32_t* d_asm_col = nullptr;
    double* d_stage = nullptr;                  // kep_set_values: device copy of the host values (2 nnz)
    // rerun passes: per fast front list descriptors and the compact lists (k_rerun_lists)
    int4 *d_rr_d1 = nullptr, *d_rr_d2 = nullptr;
    int32_t *d_rr_fr = nullptr, *d_rr_x = nullptr, *d_rr_cnt = nullptr;
    int4 *d_rr_l[4] = {nullptr, nullptr, nullptr, nullptr}, *d_rr_u = nullptr, *d_rr_a = nullptr;
    int32_t* d_rmap = nullptr;
    double *d_a = nullptr, *d_b = nullptr;
    // batch state
    double* d_arena = nullptr;
    size_t arena_alloc_doubles = 0;
    int32_t *d_nd_in = nullptr, *d_nd_out = nullptr, *d_doff = nullptr;
    ShiftStat* d_stats = nullptr;
    double* d_sigma = nullptr;
    double* d_alpha = nullptr;
    std::vector<ShiftStat> h_stats;
    // per-level launch lists: fast (panel + Schur) and reference fronts
    int32_t* d_lists = nullptr;                 // [fast fronts of all levels | ref fronts of all levels]
    int4* d_items = nullptr;                    // Schur tiles (front, I, J, 0)
    int4* d_litems = nullptr;                   // k_l21 row tiles (front, I, 0, 0)
    int4* d_lsitems = nullptr;                  // k_l21d<64,1> row tiles (FS capacity <= 64; k_l21<1> if off)
    int4* d_lditems = nullptr;                  // k_l21d<128,4> row tiles (FS capacity 65..128)
    int4* d_lxitems = nullptr;                  // k_l21<2> row tiles (GEMM in-block solve)
    int32_t* d_xfronts = nullptr;               // k_l21x_prep fronts per level
    int64_t* d_xoff = nullptr;                  // X scratch offsets (within the level)
    double* d_xscr = nullptr;
    int64_t xstride = 0;
    std::vector<int64_t> lsitem_off, lsitem_cnt, lxitem_off, lxitem_cnt, lditem_off, lditem_cnt, xfront_off, xfront_cnt;
    struct FsGroup {
        int64_t foff, fcnt, uoff, ucnt; int qmax;
        int64_t loff[4], lcnt[4];                  // the group's range of each k_l21 mode list (mode 0, 1, 2, 3)
        int64_t xoff, xcnt;                        // ... and of the level's k_l21x_prep fronts
    };
    std::vector<std::vector<FsGroup>> fs_groups;   // per level: fast fronts by FS capacity (k_fsp/k_fsu passes)
    int4* d_aitems = nullptr;                   // k_assemble strips (front, x, S, 0): all fronts, then fast fronts
    std::vector<int64_t> aitem_off, aitem_cnt, raitem_off, raitem_cnt;
    int4* d_smitems = nullptr;                  // k_asm_smem strips (front, x, S, 0) per level
    std::vector<int64_t> smitem_off, smitem_cnt;
    std::vector<char> asm_red;                  // per level: small fronts, k_assemble_red
    std::vector<int> level_fmax;                // per level: largest front capacity (k_assemble_red strips)
    std::vector<int64_t> fast_off, fast_cnt, ref_off, ref_cnt, item_off, item_cnt, litem_off, litem_cnt;
    // fast-path pivot records: per-front offsets (entries), per shift stride (doubles)
    int64_t* d_aux_off = nullptr;
    int64_t aux_stride = 0;
    double* d_aux = nullptr;
    int32_t* d_flag = nullptr;
    int32_t* d_forced = nullptr;
    int32_t* d_fstate = nullptr;
    int32_t* d_pending = nullptr;                // fronts flagged for a fast-path rerun (per level)
    int4* d_uitems = nullptr;                   // k_fsu tiles (front, I, J, 0)
    int64_t* d_goff = nullptr;                  // k_fsp global scratch offsets (-1: shared memory)
    int64_t gscratch_stride = 0;
    double* d_gscratch = nullptr;
    std::vector<int64_t> uitem_off, uitem_cnt, small_off, small_cnt;
    std::vector<int> small_cmax, small_kmax;    // per level: largest CB order / pivot count of the k_schur_small fronts
    // k_small (whole FS panel in shared memory): per level list offsets, shared-memory cap, threads
    int32_t* d_smfronts = nullptr;
    struct SmGroup { int64_t off, cnt; int cap, th; };
    // k_bigp/k_bigu/k_bigfin (multi-CTA partial LDL^T of the few large fronts of a level): per level the
    // groups (front, shift) shift-major for big_m shifts, their scratch offsets, the largest FS block
    int big_m = 0;                              // shifts the big-front groups are planned for
    std::vector<int64_t> big_goff, big_nf;      // per level: first group, big fronts
    std::vector<int> big_qmax;
    int2* d_big_groups = nullptr;
    int64_t* d_big_scroff = nullptr;
    double* d_big_scr = nullptr;
    int* d_big_state = nullptr;
    unsigned* d_big_bars = nullptr;
    std::vector<std::vector<SmGroup>> sm_groups;    // per level: size classes of the k_small fronts
    int32_t* d_small = nullptr;                  // fronts whose Schur update runs in k_schur_small
    std::vector<int> level_qmax;                // per level: max p + slack over its fast fronts
    std::vector<double> item_flops;             // per level: algorithmic a4 flops of its fast fronts
    std::vector<kep_factorization*> factors;    // live factors (released by kep_destroy)
    // kep_factor_residual: captured fronts, per-front sum of squares, residual tiles per level
    double* d_f0 = nullptr;
    double* d_resid = nullptr;
    int4* d_ritems = nullptr;
    std::vector<int64_t> ritem_off, ritem_cnt;
    // TMA tensor maps of the arena (k_schur_tma): [batch][distinct leading dimensions]
    CUtensorMap* d_tmaps = nullptr;
    int32_t* d_tmap_idx = nullptr;
    int32_t ntmap = 0;
    bool use_tma = false;
    std::vector<char> tma_level;                // per level: Schur tiles through k_schur_tma (long K)
    // profiling
    kep_profile prof;
    std::vector<cudaEvent_t> ev_pool;
    // FS-size groups of a level are disjoint front sets: groups 1.. run on forked streams so their
    // latency-bound k_fsp/k_fsu chains overlap (KEP_FS_STREAMS=0: one stream)
    cudaStream_t fs_streams[7] = {};
    cudaEvent_t fs_fork = nullptr, fs_join[7] = {};
    std::vector<int> ev_class;
    std::vector<int> ev_level;
    std::vector<std::array<double, KEP_K_NCLASS>> lvl_ms;    // KEP_PROFILE_LEVELS: per level and class
};

// Retained factors of one shift.
struct kep_factorization {
    kep_ctx* ctx = nullptr;
    double sigma = 0.0, alpha = 1.0;
    int64_t nu = 0;
    kep_inertia_info info{};
    // store (device) + offsets and level structure captured at creation
    double* panel = nullptr;
    int32_t* lab = nullptr;
    double *d = nullptr, *ds = nullptr;
    int32_t* kind = nullptr;
    int32_t* perm = nullptr;
    int4* hdr = nullptr;
    int64_t *poff = nullptr, *loff = nullptr, *qoff = nullptr, *yoff = nullptr;
    double *upd = nullptr, *ybuf = nullptr;                 // solve scratch (update vectors, big fronts' vectors)
    std::vector<int64_t> h_poff, h_loff, h_qoff, h_yoff;
    std::vector<int> level_fmax;                 // per level: max front capacity (shared memory of the solves)
    std::vector<int64_t> big_off, big_cnt;       // per level: fronts solved by the blocked kernels
    std::vector<int> big_fmax, big_emax;
    int32_t* d_bigf = nullptr;
    double *xw = nullptr, *bw = nullptr;         // work vectors (n)
    int64_t panel_doubles = 0, lab_ints = 0, q_entries = 0;
    kep::StorePlan plan() const {
        kep::StorePlan T;
        T.panel = panel; T.poff = poff; T.lab = lab; T.loff = loff;
        T.d = d; T.ds = ds; T.kind = kind; T.perm = perm; T.qoff = qoff; T.hdr = hdr;
        T.upd = upd; T.ybuf = ybuf; T.yoff = yoff;
        return T;
    }
};

namespace {

thread_local std::string g_err;
constexpr int kReruns = 2;      // fast-path reruns per level before the unblocked fallback
constexpr int kSmallDelay = 8;  // k_small eligibility: the panel with this many delayed-in columns fits kSmallCap
constexpr int kAsmSmemCap = 2048;   // k_asm_smem on levels whose fronts all have at most this capacity
constexpr int kBigQ = 2048;        // big fronts: FS capacity at least this (c4 root, 1216: faster on k_fsp) ...
constexpr int kBigGroups = 74;      // ... on levels with at most this many (front, shift) groups (>= 2 SMs each)
constexpr int kSmallMaxPiv = 16;   // k_small: fronts with at most this many own pivots
constexpr int kSmallPlan = 2;   // k_small size class: planned delayed-in columns (more, beyond the class cap: k_factor_ref)
constexpr int64_t kSmallCap = 24 * 1024;   // k_small: FS panel budget in doubles (192 KB of shared memory)

kep_status fail(kep_ctx* c, kep_status s, const std::string& msg) {
    if (c) c->err = msg;
    g_err = msg;
    return s;
}

#define KEP_CUDA(ctx, call)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? KEP_ENOMEM : KEP_ECUDA,        \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

template <class T>
cudaError_t upload(T** dptr, const std::vector<T>& h) {
    size_t bytes = std::max<size_t>(h.size(), 1) * sizeof(T);
    cudaError_t e = cudaMalloc((void**)dptr, bytes);
    if (e != cudaSuccess) return e;
    if (!h.empty()) e = cudaMemcpy(*dptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

void free_batch(kep_ctx* c) {
    cudaFree(c->d_arena); c->d_arena = nullptr; c->arena_alloc_doubles = 0;
    cudaFree(c->d_nd_in); c->d_nd_in = nullptr;
    cudaFree(c->d_nd_out); c->d_nd_out = nullptr;
    cudaFree(c->d_doff); c->d_doff = nullptr;
    cudaFree(c->d_stats); c->d_stats = nullptr;
    cudaFree(c->d_sigma); c->d_sigma = nullptr;
    cudaFree(c->d_alpha); c->d_alpha = nullptr;
    cudaFree(c->d_aux); c->d_aux = nullptr;
    cudaFree(c->d_flag); c->d_flag = nullptr;
    cudaFree(c->d_forced); c->d_forced = nullptr;
    cudaFree(c->d_fstate); c->d_fstate = nullptr;
    cudaFree(c->d_gscratch); c->d_gscratch = nullptr;
    cudaFree(c->d_xscr); c->d_xscr = nullptr;
    cudaFree(c->d_pending); c->d_pending = nullptr;
}

// (Re)allocate the per-batch state for the current memory plan.
kep_status alloc_batch(kep_ctx* c) {
    free_batch(c);
    size_t freeb = 0, totalb = 0;
    KEP_CUDA(c, cudaMemGetInfo(&freeb, &totalb));
    const size_t per_shift =
        ((size_t)c->sym.arena_doubles + (size_t)c->aux_stride + (size_t)c->gscratch_stride + (size_t)c->xstride) * sizeof(double);
    int cap = std::max(1, c->opts.max_batch);
    const size_t budget = (size_t)(0.85 * (double)freeb);
    while (cap > 1 && per_shift * (size_t)cap > budget) cap--;
    if (per_shift > budget) return fail(c, KEP_ENOMEM, "front arena of one shift does not fit in device memory");
    c->batch_cap = cap;
    c->arena_alloc_doubles = (size_t)c->sym.arena_doubles * cap;
    KEP_CUDA(c, cudaMalloc(&c->d_arena, c->arena_alloc_doubles * sizeof(double)));
    const size_t nfb = (size_t)std::max<int64_t>(c->sym.nf, 1) * cap * sizeof(int32_t);
    KEP_CUDA(c, cudaMalloc(&c->d_nd_in, nfb));
    KEP_CUDA(c, cudaMalloc(&c->d_nd_out, nfb));
    KEP_CUDA(c, cudaMalloc(&c->d_doff, nfb));
    KEP_CUDA(c, cudaMalloc(&c->d_stats, sizeof(ShiftStat) * cap));
    KEP_CUDA(c, cudaMalloc(&c->d_sigma, sizeof(double) * cap));
    KEP_CUDA(c, cudaMalloc(&c->d_alpha, sizeof(double) * cap));
    KEP_CUDA(c, cudaMalloc(&c->d_aux, sizeof(double) * std::max<int64_t>(c->aux_stride, 1) * cap));
    KEP_CUDA(c, cudaMalloc(&c->d_flag, nfb));
    KEP_CUDA(c, cudaMemset(c->d_flag, 0, nfb));
    KEP_CUDA(c, cudaMalloc(&c->d_forced, nfb * (kep::FMAX + 1)));
    KEP_CUDA(c, cudaMalloc(&c->d_fstate, nfb * kep::FSTATE_W));
    KEP_CUDA(c, cudaMalloc(&c->d_gscratch, sizeof(double) * std::max<int64_t>(c->gscratch_stride, 1) * cap));
    KEP_CUDA(c, cudaMalloc(&c->d_xscr, sizeof(double) * std::max<int64_t>(c->xstride, 1) * cap));
    KEP_CUDA(c, cudaMalloc(&c->d_pending, 2 * sizeof(int32_t)));
    c->h_stats.resize(cap);
    // tensor maps: one per (distinct front leading dimension, shift of the batch)
    cudaFree(c->d_tmaps); c->d_tmaps = nullptr;
    cudaFree(c->d_tmap_idx); c->d_tmap_idx = nullptr;
    c->use_tma = false;
    if (!getenv("KEP_NO_TMA")) {
        const Symbolic& S = c->sym;
        std::vector<int> lds;
        std::vector<int32_t> idx(std::max<int64_t>(S.nf, 1), 0);
        for (int64_t s = 0; s < S.nf; ++s) lds.push_back(kep::ldpad(S.capacity[s]));
        std::sort(lds.begin(), lds.end());
        lds.erase(std::unique(lds.begin(), lds.end()), lds.end());
        for (int64_t s = 0; s < S.nf; ++s)
            idx[s] = (int32_t)(std::lower_bound(lds.begin(), lds.end(), kep::ldpad(S.capacity[s])) - lds.begin());
        std::vector<CUtensorMap> maps((size_t)cap * lds.size());
        bool ok = !lds.empty();
        for (int b = 0; b < cap && ok; ++b)
            for (size_t k = 0; k < lds.size() && ok; ++k)
                ok = kep::encode_front_tmap(&maps[(size_t)b * lds.size() + k], c->d_arena + (size_t)b * S.arena_doubles,
                                            S.arena_doubles, lds[k]);
        if (ok) {
            KEP_CUDA(c, upload(&c->d_tmaps, maps));
            KEP_CUDA(c, upload(&c->d_tmap_idx, idx));
            c->ntmap = (int32_t)lds.size();
            c->use_tma = true;
        }
    }
    return KEP_OK;
}

int nl_all(const Symbolic& S) { return (int)S.level_ptr.size() - 1; }

// Split every level into fronts for the blocked panel kernel (+ DMMA Schur
// tiles) and fronts for the reference kernel; build the Schur work items.
kep_status build_lists(kep_ctx* c) {
    const Symbolic& S = c->sym;
    // fast (blocked) path, or the unblocked kernel (variant 1; FS blocks beyond the fast kernels)
    // (routing tiny fronts to the unblocked kernel measured slower at c4: its fronts live in HBM)
    // k_small: the FS panel (f x (p + kSmallDelay)) fits the shared-memory budget (non-root fronts)
    const bool use_small = c->opts.kernel_variant == 0 && !getenv("KEP_NO_SMALL");
    auto is_small = [&](int s) {
        const int64_t qq = (int64_t)S.npiv[s] + kSmallDelay;
        // (measured at c4: faster than the k_fsp/k_l21/k_check path up to ~16 pivots, slower beyond)
        return use_small && S.ncb[s] > 0 && S.npiv[s] <= kSmallMaxPiv && (int64_t)S.forder[s] * qq <= kSmallCap;
    };
    // big fronts: levels with few large FS blocks (all SMs on them, kernels_big.cu)
    if (c->big_m <= 0) c->big_m = std::max(1, c->opts.max_batch);
    std::vector<char> big(std::max<int64_t>(S.nf, 1), 0);
    int bigq = kBigQ;
    if (const char* e = getenv("KEP_BIG_Q")) bigq = std::max(2, atoi(e));      // testing: route smaller fronts
    if (c->opts.kernel_variant == 0 && !getenv("KEP_NO_BIG")) {
        for (int L = 0; L + 1 < (int)S.level_ptr.size(); ++L) {
            int nb = 0;
            for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k)
                nb += S.capacity[S.level_fronts[k]] - S.ncb[S.level_fronts[k]] >= bigq;
            if (nb == 0 || nb * c->big_m > kBigGroups) continue;
            for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k)
                if (S.capacity[S.level_fronts[k]] - S.ncb[S.level_fronts[k]] >= bigq) big[S.level_fronts[k]] = 1;
        }
    }
    auto is_big = [&](int s) { return big[s] != 0; };
    auto is_fast = [&](int s) {
        return c->opts.kernel_variant == 0 && !is_small(s) && !is_big(s) && kep::front_nb_for(S.capacity[s] - S.ncb[s]) > 0;
    };
    std::vector<int2> bgroups;
    std::vector<int64_t> bscr;
    int64_t bscr_acc = 0, bscr_max = 0;
    c->big_goff.assign(nl_all(S), 0); c->big_nf.assign(nl_all(S), 0); c->big_qmax.assign(nl_all(S), 0);
    const int nl = (int)S.level_ptr.size() - 1;
    std::vector<int32_t> smf;
    c->sm_groups.assign(nl, {});
    c->item_flops.assign(nl, 0.0);
    std::vector<int32_t> fast, ref;
    std::vector<int4> items, litems, lsitems, lxitems, lditems, uitems;
    std::vector<int32_t> xfronts;
    std::vector<int64_t> xoff(S.nf > 0 ? S.nf : 1, 0);
    int64_t xmax = 0;
    std::vector<int4> rd1(S.nf > 0 ? S.nf : 1, make_int4(0, 0, 0, 0)), rd2(S.nf > 0 ? S.nf : 1, make_int4(0, 0, 0, 0));
    int64_t mx_f = 1, mx_l[4] = {1, 1, 1, 1}, mx_u = 1, mx_a = 1;
    std::vector<int32_t> small;
    c->litem_off.assign(nl, 0); c->litem_cnt.assign(nl, 0);
    c->lsitem_off.assign(nl, 0); c->lsitem_cnt.assign(nl, 0);
    c->lditem_off.assign(nl, 0); c->lditem_cnt.assign(nl, 0);
    c->lxitem_off.assign(nl, 0); c->lxitem_cnt.assign(nl, 0);
    c->xfront_off.assign(nl, 0); c->xfront_cnt.assign(nl, 0);
    c->aitem_off.assign(nl, 0); c->aitem_cnt.assign(nl, 0);
    c->raitem_off.assign(nl, 0); c->raitem_cnt.assign(nl, 0);
    std::vector<int4> aitems, smitems;
    c->smitem_off.assign(nl, 0); c->smitem_cnt.assign(nl, 0);
    auto strips = [&](int s, int rmax) {              // rmax: CTAs per front (k_reassemble loops)
        const int ns = kep::assembly_strips((int)S.forder[s]);
        const int r = std::min(ns, rmax);
        for (int x = 0; x < r; ++x) aitems.push_back(make_int4(s, x, ns, r));
    };
    c->uitem_off.assign(nl, 0); c->uitem_cnt.assign(nl, 0);
    c->small_off.assign(nl, 0); c->small_cnt.assign(nl, 0);
    c->small_cmax.assign(nl, 0); c->small_kmax.assign(nl, 0);
    c->fast_off.assign(nl, 0); c->fast_cnt.assign(nl, 0);
    c->ref_off.assign(nl, 0); c->ref_cnt.assign(nl, 0);
    c->item_off.assign(nl, 0); c->item_cnt.assign(nl, 0);
    c->level_qmax.assign(nl, 0);
    c->asm_red.assign(nl, 0);
    c->level_fmax.assign(nl, 0);
    c->fs_groups.clear();
    for (int L = 0; L < nl; ++L) {
        c->fast_off[L] = (int64_t)fast.size();
        c->ref_off[L] = (int64_t)ref.size();
        c->item_off[L] = (int64_t)items.size();
        c->litem_off[L] = (int64_t)litems.size();
        c->lsitem_off[L] = (int64_t)lsitems.size();
        c->lditem_off[L] = (int64_t)lditems.size();
        c->lxitem_off[L] = (int64_t)lxitems.size();
        c->xfront_off[L] = (int64_t)xfronts.size();
        int64_t xacc = 0;
        c->uitem_off[L] = (int64_t)uitems.size();
        c->small_off[L] = (int64_t)small.size();
        c->aitem_off[L] = (int64_t)aitems.size();
        {   // small-front levels: whole-front RED assembly (measured faster below ~700 at c4)
            double sf = 0.0;
            for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) sf += S.forder[S.level_fronts[k]];
            const int nlf = S.level_ptr[L + 1] - S.level_ptr[L];
            c->asm_red[L] = nlf > 0 && sf / nlf < 700.0;
            for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k)
                c->level_fmax[L] = std::max(c->level_fmax[L], (int)S.capacity[S.level_fronts[k]]);
        }
        for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) strips(S.level_fronts[k], INT_MAX);
        c->aitem_cnt[L] = (int64_t)aitems.size() - c->aitem_off[L];
        {   // shared-memory strip assembly where every front of the level is small enough
            bool ok = getenv("KEP_ASM_SMEM") != nullptr;       // opt-in: measured slower than the RED / gather
                                                               // kernels at c4 (137 vs 107 ms per 8 shifts)
            for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1] && ok; ++k)
                ok = S.capacity[S.level_fronts[k]] <= kAsmSmemCap;
            c->smitem_off[L] = (int64_t)smitems.size();
            if (ok)
                for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) {
                    const int s = S.level_fronts[k];
                    const int ns = kep::smem_strips(S.capacity[s]);
                    for (int x = 0; x < ns; ++x) smitems.push_back(make_int4(s, x, ns, 0));
                }
            c->smitem_cnt[L] = (int64_t)smitems.size() - c->smitem_off[L];
        }
        c->raitem_off[L] = (int64_t)aitems.size();
        for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k)
            if (is_fast(S.level_fronts[k])) {
                const int s = S.level_fronts[k];
                rd2[s].y = (int)aitems.size();
                strips(s, 8);
                rd2[s].z = (int)aitems.size() - rd2[s].y;
            }
        c->raitem_cnt[L] = (int64_t)aitems.size() - c->raitem_off[L];
        // k_small fronts in size classes (shared memory per launch = the class cap: occupancy).  The
        // class is chosen for kSmallPlan delayed-in columns; a front with more is handed to k_factor_ref.
        {
            static const int kCls[8] = {1536, 2048, 3072, 4096, 6144, 8192, 12288, (int)kSmallCap};
            int kTh[8] = {32, 64, 64, 128, 128, 256, 256, 256};
            if (const char* e = getenv("KEP_SMALL_TH"))         // tuning: threads per size class
                sscanf(e, "%d,%d,%d,%d,%d,%d,%d,%d", &kTh[0], &kTh[1], &kTh[2], &kTh[3], &kTh[4], &kTh[5], &kTh[6],
                       &kTh[7]);
            for (int cl = 0; cl < 8; ++cl) {
                kep_ctx::SmGroup g{(int64_t)smf.size(), 0, kCls[cl], kTh[cl]};
                for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) {
                    const int s = S.level_fronts[k];
                    if (!is_small(s) || is_big(s)) continue;     // a big front is factored by k_bigp only
                    const int64_t need = (int64_t)S.forder[s] * (S.npiv[s] + kSmallPlan);
                    if (need <= kCls[cl] && (cl == 0 || need > kCls[cl - 1])) smf.push_back(s);
                }
                g.cnt = (int64_t)smf.size() - g.off;
                if (g.cnt) c->sm_groups[L].push_back(g);
            }
        }
        {   // big-front groups of this level: shift-major, so the first nbig * m serve a batch of m
            std::vector<int> bl;
            for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k)
                if (is_big(S.level_fronts[k])) bl.push_back(S.level_fronts[k]);
            c->big_goff[L] = (int64_t)bgroups.size();
            c->big_nf[L] = (int64_t)bl.size();
            int64_t acc = 0;
            for (int sh = 0; sh < c->big_m; ++sh)
                for (int s : bl) {
                    bgroups.push_back(make_int2(s, sh));
                    bscr.push_back(acc);
                    acc += (int64_t)kep::big_scratch_doubles(S.capacity[s], kBigGroups);
                    c->big_qmax[L] = std::max(c->big_qmax[L], S.capacity[s] - S.ncb[s]);
                }
            bscr_max = std::max(bscr_max, acc);
            (void)bscr_acc;
        }
        // tile lists in the level's front order
        for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) {
            const int s = S.level_fronts[k];
            const int qcap = S.capacity[s] - S.ncb[s];            // p + slack
            if (is_big(s)) {                                       // k_bigp..k_bigfin, then the Schur tiles
                const int nt = (S.ncb[s] + 63) / 64;
                for (int I = 0; I < nt; ++I)
                    for (int J = 0; J <= I; ++J) items.push_back(make_int4(s, I, J, 0));
                c->item_flops[L] += (double)S.npiv[s] * (double)S.ncb[s] * (double)(S.ncb[s] + 1);
                continue;
            }
            if (is_small(s)) {                                     // k_small, then the Schur tiles
                const int qq = S.npiv[s] + kSmallDelay;
                if (kep::schur_small_ok(S.ncb[s], qq)) {
                    small.push_back(s);
                    c->small_cmax[L] = std::max(c->small_cmax[L], (int)S.ncb[s]);
                    c->small_kmax[L] = std::max(c->small_kmax[L], qq);
                } else {
                    const int nt = (S.ncb[s] + 63) / 64;
                    for (int I = 0; I < nt; ++I)
                        for (int J = 0; J <= I; ++J) items.push_back(make_int4(s, I, J, 0));
                }
                c->item_flops[L] += (double)S.npiv[s] * (double)S.ncb[s] * (double)(S.ncb[s] + 1);
                continue;
            }
            if (!is_fast(s)) {
                ref.push_back(s);
                continue;
            }
            c->level_qmax[L] = std::max(c->level_qmax[L], qcap);
            if (kep::schur_small_ok(S.ncb[s], qcap)) {
                small.push_back(s);                                  // whole CB in one CTA
                c->small_cmax[L] = std::max(c->small_cmax[L], (int)S.ncb[s]);
                c->small_kmax[L] = std::max(c->small_kmax[L], qcap);
            } else {
                const int nt = (S.ncb[s] + 63) / 64;
                for (int I = 0; I < nt; ++I)
                    for (int J = 0; J <= I; ++J) items.push_back(make_int4(s, I, J, 0));
            }
        }
        // fast fronts (and their k_fsu tiles) in increasing FS capacity: the k_fsp/k_fsu passes
        // run per size group
        std::vector<int> lf(S.level_fronts.begin() + S.level_ptr[L], S.level_fronts.begin() + S.level_ptr[L + 1]);
        std::stable_sort(lf.begin(), lf.end(), [&](int a, int b) {
            return S.capacity[a] - S.ncb[a] < S.capacity[b] - S.ncb[b];
        });
        std::vector<int64_t> fu;                                  // uitems offset of each fast front
        for (int s : lf) {
            const int qcap = S.capacity[s] - S.ncb[s];
            if (!is_fast(s)) continue;
            fast.push_back(s);
            {   // k_l21 row strips, in the same (sorted) order: a size group owns a contiguous range of
                // each mode's list, so its k_fsp -> k_l21 chain can run on the group's stream
                const int lmode = kep::l21_mode(qcap);
                auto& li = lmode == 1 ? lsitems : (lmode == 2 ? lxitems : (lmode == 3 ? lditems : litems));
                if (lmode == 2) {
                    xfronts.push_back(s);
                    xoff[s] = xacc;
                    xacc += kep::l21_x_doubles(qcap);
                }
                rd1[s].x = lmode;
                rd1[s].y = (int)li.size();
                for (int I = 0; I < (S.ncb[s] + 127) / 128; ++I) li.push_back(make_int4(s, I, 0, 0));   // k_l21: 128 CB rows
                rd1[s].z = (int)li.size() - rd1[s].y;
            }
            fu.push_back((int64_t)uitems.size());
            rd1[s].w = (int)uitems.size();
            for (int I = 0; I < (qcap + 63) / 64; ++I)
                for (int J = 0; J <= I; ++J) uitems.push_back(make_int4(s, I, J, 0));
            rd2[s].x = (int)uitems.size() - rd1[s].w;
        }
        c->fast_cnt[L] = (int64_t)fast.size() - c->fast_off[L];
        {   // size groups: at most three contiguous ranges of the sorted fast fronts, chosen by fs_cost
            const int64_t n = c->fast_cnt[L], f0 = c->fast_off[L];
            const int64_t mb = std::max(1, std::min(c->opts.max_batch, 8));
            fu.push_back((int64_t)uitems.size());
            auto qc = [&](int64_t x) { return S.capacity[fast[f0 + x]] - S.ncb[fast[f0 + x]]; };
            auto cost = [&](int64_t a, int64_t b) { return b > a ? kep::fs_cost(qc(b - 1), (b - a) * mb) : 0.0; };
            std::vector<int64_t> cuts;                             // candidate split points (qcap changes)
            for (int64_t x = 1; x < n; ++x)
                if (qc(x) != qc(x - 1)) cuts.push_back(x);
            double best = cost(0, n);
            int64_t b1 = n, b2 = n;
            for (size_t i = 0; i < cuts.size(); ++i) {
                const int64_t x = cuts[i];
                const double c2 = cost(0, x) + cost(x, n);
                if (c2 < best) { best = c2; b1 = x; b2 = n; }
                for (size_t j = i + 1; j < cuts.size(); ++j) {
                    const int64_t y = cuts[j];
                    const double c3 = cost(0, x) + cost(x, y) + cost(y, n);
                    if (c3 < best) { best = c3; b1 = x; b2 = y; }
                }
            }
            std::vector<kep_ctx::FsGroup> gs;
            std::vector<int64_t> bnd = {0, b1, b2, n};
            bnd.erase(std::unique(bnd.begin(), bnd.end()), bnd.end());
            // a level left with one group is cut into KEP_FS_SPLIT (default 2) equal parts, so that on
            // the forked streams one part's k_l21 (DMMA) overlaps another part's k_fsp (latency-bound);
            // measured at c4 per 8 shifts: one stream 500.1 ms, forked 492.3, split 2/3/4: 489.0/493.0/493.5
            static const int fs_split = [] { const char* x = getenv("KEP_FS_SPLIT"); return x ? atoi(x) : 2; }();
            if (bnd.size() == 2 && fs_split > 1 && n >= 2 * fs_split) {
                bnd.clear();
                for (int k2 = 0; k2 <= std::min(fs_split, 4); ++k2) bnd.push_back(n * k2 / std::min(fs_split, 4));
            }
            static const bool fs_split_all = [] { const char* x = getenv("KEP_FS_SPLIT_ALL"); return x && atoi(x) != 0; }();
            if (fs_split_all && bnd.size() > 2) {                  // tuning: every cost-model group cut in two
                std::vector<int64_t> b2;
                for (size_t k2 = 0; k2 + 1 < bnd.size(); ++k2) {
                    b2.push_back(bnd[k2]);
                    if (bnd[k2 + 1] - bnd[k2] >= 4) b2.push_back((bnd[k2] + bnd[k2 + 1]) / 2);
                }
                b2.push_back(n);
                bnd = b2;
            }
            for (size_t k2 = 0; k2 + 1 < bnd.size(); ++k2)
                if (bnd[k2 + 1] > bnd[k2]) {
                    kep_ctx::FsGroup g{f0 + bnd[k2], bnd[k2 + 1] - bnd[k2], fu[bnd[k2]], fu[bnd[k2 + 1]] - fu[bnd[k2]],
                                       (int)qc(bnd[k2 + 1] - 1), {-1, -1, -1, -1}, {0, 0, 0, 0}, -1, 0};
                    int64_t xi = c->xfront_off[L];               // xfronts index of the level's mode-2 fronts, in order
                    for (int64_t x = 0; x < bnd[k2]; ++x) xi += rd1[fast[f0 + x]].x == 2;
                    for (int64_t x = bnd[k2]; x < bnd[k2 + 1]; ++x) {
                        const int4 r = rd1[fast[f0 + x]];
                        if (g.loff[r.x] < 0) g.loff[r.x] = r.y;
                        g.lcnt[r.x] += r.z;
                        if (r.x == 2) { if (g.xoff < 0) g.xoff = xi; ++g.xcnt; ++xi; }
                    }
                    gs.push_back(g);
                }
            c->fs_groups.push_back(gs);
        }
        c->ref_cnt[L] = (int64_t)ref.size() - c->ref_off[L];
        c->item_cnt[L] = (int64_t)items.size() - c->item_off[L];
        c->litem_cnt[L] = (int64_t)litems.size() - c->litem_off[L];
        c->lsitem_cnt[L] = (int64_t)lsitems.size() - c->lsitem_off[L];
        c->lditem_cnt[L] = (int64_t)lditems.size() - c->lditem_off[L];
        c->lxitem_cnt[L] = (int64_t)lxitems.size() - c->lxitem_off[L];
        c->xfront_cnt[L] = (int64_t)xfronts.size() - c->xfront_off[L];
        xmax = std::max(xmax, xacc);
        mx_f = std::max(mx_f, c->fast_cnt[L]);
        mx_l[0] = std::max(mx_l[0], c->litem_cnt[L]);
        mx_l[1] = std::max(mx_l[1], c->lsitem_cnt[L]);
        mx_l[3] = std::max(mx_l[3], c->lditem_cnt[L]);
        mx_l[2] = std::max(mx_l[2], c->lxitem_cnt[L]);
        c->uitem_cnt[L] = (int64_t)uitems.size() - c->uitem_off[L];
        mx_u = std::max(mx_u, c->uitem_cnt[L]);
        mx_a = std::max(mx_a, c->raitem_cnt[L]);
        c->small_cnt[L] = (int64_t)small.size() - c->small_off[L];
    }
    // TMA-fed Schur tiles where K (the pivots of a front) is long: measured equal to the cp.async
    // kernel at K >= 128 and slower below (per-CTA barrier/tensor-map setup over few K chunks)
    c->tma_level.assign(nl, 0);
    for (int L = 0; L < nl; ++L) {
        double sp = 0.0, nfr = 0.0;
        for (int k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) { sp += S.npiv[S.level_fronts[k]]; nfr += 1.0; }
        c->tma_level[L] = nfr > 0.0 && sp / nfr >= 128.0;
    }
    for (int L = 0; L < nl; ++L)
        for (int64_t k = c->fast_off[L]; k < c->fast_off[L] + c->fast_cnt[L]; ++k) {
            const int s = fast[k];
            c->item_flops[L] += (double)S.npiv[s] * (double)S.ncb[s] * (double)(S.ncb[s] + 1);
        }
    std::vector<int32_t> lists(fast);
    lists.insert(lists.end(), ref.begin(), ref.end());
    const int64_t nfast = (int64_t)fast.size();
    for (int L = 0; L < nl; ++L) c->ref_off[L] += nfast;
    cudaFree(c->d_lists); c->d_lists = nullptr;
    cudaFree(c->d_items); c->d_items = nullptr;
    cudaFree(c->d_litems); c->d_litems = nullptr;
    cudaFree(c->d_uitems); c->d_uitems = nullptr;
    KEP_CUDA(c, upload(&c->d_uitems, uitems));
    cudaFree(c->d_small); c->d_small = nullptr;
    KEP_CUDA(c, upload(&c->d_small, small));
    cudaFree(c->d_smfronts); c->d_smfronts = nullptr;
    KEP_CUDA(c, upload(&c->d_smfronts, smf));
    cudaFree(c->d_aux_off); c->d_aux_off = nullptr;
    KEP_CUDA(c, upload(&c->d_litems, litems));
    cudaFree(c->d_lsitems); c->d_lsitems = nullptr;
    KEP_CUDA(c, upload(&c->d_lsitems, lsitems));
    cudaFree(c->d_lditems); c->d_lditems = nullptr;
    KEP_CUDA(c, upload(&c->d_lditems, lditems));
    cudaFree(c->d_lxitems); c->d_lxitems = nullptr;
    KEP_CUDA(c, upload(&c->d_lxitems, lxitems));
    cudaFree(c->d_xfronts); c->d_xfronts = nullptr;
    KEP_CUDA(c, upload(&c->d_xfronts, xfronts));
    cudaFree(c->d_xoff); c->d_xoff = nullptr;
    KEP_CUDA(c, upload(&c->d_xoff, xoff));
    c->xstride = xmax;
    {
        void* old[] = {c->d_rr_d1, c->d_rr_d2, c->d_rr_fr, c->d_rr_x, c->d_rr_cnt, c->d_rr_l[0], c->d_rr_l[1],
                       c->d_rr_l[2], c->d_rr_l[3], c->d_rr_u, c->d_rr_a};
        for (void* q : old) cudaFree(q);
        c->d_rr_d1 = c->d_rr_d2 = nullptr;
        KEP_CUDA(c, upload(&c->d_rr_d1, rd1));
        KEP_CUDA(c, upload(&c->d_rr_d2, rd2));
        KEP_CUDA(c, cudaMalloc(&c->d_rr_fr, sizeof(int32_t) * mx_f));
        KEP_CUDA(c, cudaMalloc(&c->d_rr_x, sizeof(int32_t) * mx_f));
        KEP_CUDA(c, cudaMalloc(&c->d_rr_cnt, sizeof(int32_t) * 8));
        for (int k = 0; k < 4; ++k) KEP_CUDA(c, cudaMalloc(&c->d_rr_l[k], sizeof(int4) * mx_l[k]));
        KEP_CUDA(c, cudaMalloc(&c->d_rr_u, sizeof(int4) * mx_u));
        KEP_CUDA(c, cudaMalloc(&c->d_rr_a, sizeof(int4) * mx_a));
    }
    cudaFree(c->d_aitems); c->d_aitems = nullptr;
    KEP_CUDA(c, upload(&c->d_aitems, aitems));
    cudaFree(c->d_smitems); c->d_smitems = nullptr;
    KEP_CUDA(c, upload(&c->d_smitems, smitems));
    // pivot-record offsets: Q_s = p_s + slack entries per front
    std::vector<int64_t> aoff(S.nf > 0 ? S.nf : 1, 0);
    int64_t acc = 0;
    for (int64_t f2 = 0; f2 < S.nf; ++f2) {
        aoff[f2] = acc;
        acc += S.capacity[f2] - S.ncb[f2];
    }
    c->aux_stride = std::max<int64_t>(acc, 1) * kep::AUX_W;
    KEP_CUDA(c, upload(&c->d_aux_off, aoff));
    // global scratch for the k_fsp block columns of levels whose FS blocks exceed shared memory
    std::vector<int64_t> goff(S.nf > 0 ? S.nf : 1, -1);
    int64_t gacc = 0;
    for (int L = 0; L < nl; ++L) {
        if (!c->fast_cnt[L] || !kep::fs_uses_gls(c->level_qmax[L])) continue;
        const int64_t per = (int64_t)kep::fs_gls_doubles(16, kep::fs_rows_pad(c->level_qmax[L]));
        for (int64_t x = c->fast_off[L]; x < c->fast_off[L] + c->fast_cnt[L]; ++x) {
            goff[fast[x]] = gacc;
            gacc += per;
        }
    }
    c->gscratch_stride = gacc;
    cudaFree(c->d_goff); c->d_goff = nullptr;
    KEP_CUDA(c, upload(&c->d_goff, goff));
    KEP_CUDA(c, upload(&c->d_lists, lists));
    KEP_CUDA(c, upload(&c->d_items, items));
    {
        void* old[] = {c->d_big_groups, c->d_big_scroff, c->d_big_scr, c->d_big_state, c->d_big_bars};
        for (void* q : old) cudaFree(q);
        c->d_big_groups = nullptr; c->d_big_scroff = nullptr; c->d_big_scr = nullptr;
        c->d_big_state = nullptr; c->d_big_bars = nullptr;
        KEP_CUDA(c, upload(&c->d_big_groups, bgroups));
        KEP_CUDA(c, upload(&c->d_big_scroff, bscr));
        KEP_CUDA(c, cudaMalloc(&c->d_big_scr, std::max<int64_t>(bscr_max, 1) * sizeof(double)));
        const size_t ng = std::max<size_t>(bgroups.size(), 1);
        KEP_CUDA(c, cudaMalloc(&c->d_big_state, ng * 16 * sizeof(int)));
        KEP_CUDA(c, cudaMalloc(&c->d_big_bars, ng * sizeof(unsigned)));
    }
    return KEP_OK;
}

// full symmetric CSR (both triangles) of the lower CSC pattern; src = lower entry index
void build_full_csr(int64_t n, const int64_t* colptr, const int32_t* rowidx, std::vector<int64_t>& rp,
                    std::vector<int32_t>& ci, std::vector<int64_t>& src) {
    rp.assign(n + 1, 0);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) {
            const int64_t i = rowidx[q];
            rp[i + 1]++;
            if (i != j) rp[j + 1]++;
        }
    for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
    ci.assign(rp[n], 0);
    src.assign(rp[n], 0);
    std::vector<int64_t> w(rp.begin(), rp.end() - 1);
    for (int64_t j = 0; j < n; ++j)                  // rows get their columns in increasing order
        for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) {
            const int64_t i = rowidx[q];
            ci[w[i]] = (int32_t)j; src[w[i]++] = q;
            if (i != j) { ci[w[j]] = (int32_t)i; src[w[j]++] = q; }
        }
}

kep_status upload_plan(kep_ctx* c, const int64_t* colptr, const int32_t* rowidx) {
    const Symbolic& S = c->sym;
    {
        std::vector<int64_t> rp, src;
        std::vector<int32_t> ci;
        build_full_csr(S.n, colptr, rowidx, rp, ci, src);
        c->csr_nnz = rp[S.n];
        KEP_CUDA(c, upload(&c->d_csr_rp, rp));
        KEP_CUDA(c, upload(&c->d_csr_ci, ci));
        KEP_CUDA(c, upload(&c->d_csr_src, src));
        KEP_CUDA(c, cudaMalloc(&c->d_csr_a, std::max<int64_t>(c->csr_nnz, 1) * sizeof(double)));
        KEP_CUDA(c, cudaMalloc(&c->d_csr_b, std::max<int64_t>(c->csr_nnz, 1) * sizeof(double)));
    }
    KEP_CUDA(c, upload(&c->d_forder, S.forder));
    KEP_CUDA(c, upload(&c->d_npiv, S.npiv));
    KEP_CUDA(c, upload(&c->d_ncb, S.ncb));
    KEP_CUDA(c, upload(&c->d_cap, S.capacity));
    KEP_CUDA(c, upload(&c->d_child_ptr, S.child_ptr));
    KEP_CUDA(c, upload(&c->d_child_list, S.child_list));
    KEP_CUDA(c, upload(&c->d_level_fronts, S.level_fronts));
    KEP_CUDA(c, upload(&c->d_arena_off, S.arena_off));
    KEP_CUDA(c, upload(&c->d_asm_ptr, S.asm_ptr));
    KEP_CUDA(c, upload(&c->d_asm_src, S.asm_src));
    KEP_CUDA(c, upload(&c->d_asm_rc, S.asm_rc));
    KEP_CUDA(c, upload(&c->d_rmap_ptr, S.rmap_ptr));
    KEP_CUDA(c, upload(&c->d_rmap, S.rmap));
    {
        std::vector<int32_t> pf(S.piv_first.begin(), S.piv_first.end());
        std::vector<int32_t> cp(S.cb_ptr.begin(), S.cb_ptr.end());
        std::vector<int32_t> cr(S.cb_rows.begin(), S.cb_rows.end());
        KEP_CUDA(c, upload(&c->d_piv_first, pf));
        std::vector<int32_t> acol;                       // per front: first entry of each local column
        acol.reserve((size_t)S.n + S.nf);
        for (int64_t f = 0; f < S.nf; ++f) {
            const int64_t a0 = S.asm_ptr[f], a1 = S.asm_ptr[f + 1];
            int64_t k = a0;
            for (int j = 0; j <= S.npiv[f]; ++j) {
                while (k < a1 && (int)(S.asm_rc[k] & 0xffffu) < j) ++k;
                acol.push_back((int32_t)(k - a0));
            }
        }
        KEP_CUDA(c, upload(&c->d_asm_col, acol));
        KEP_CUDA(c, upload(&c->d_cb_ptr, cp));
        KEP_CUDA(c, upload(&c->d_cb_rows, cr));
        KEP_CUDA(c, upload(&c->d_perm, S.perm));
        KEP_CUDA(c, upload(&c->d_iperm, S.iperm));
    }
    KEP_CUDA(c, cudaMalloc(&c->d_a, std::max<int64_t>(S.nnz, 1) * sizeof(double)));
    KEP_CUDA(c, cudaMalloc(&c->d_b, std::max<int64_t>(S.nnz, 1) * sizeof(double)));
    kep_status r = build_lists(c);
    if (r != KEP_OK) return r;
    r = alloc_batch(c);
    if (r != KEP_OK) return r;
    if (c->batch_cap < c->big_m) {                    // big-front levels are chosen for the batch that fits
        c->big_m = c->batch_cap;
        r = build_lists(c);
        if (r != KEP_OK) return r;
        r = alloc_batch(c);
    }
    return r;
}

// after a slack overflow: larger slack, new plan, re-upload the plan arrays that changed
kep_status replan(kep_ctx* c, int slack) {
    for (int64_t s = 0; s < c->sym.nf; ++s)                 // local positions are 16-bit (asm_rc, gather maps)
        if ((int64_t)c->sym.forder[s] + slack > 65535)
            return fail(c, KEP_ENOMEM, "delayed pivots grow a front beyond 65535 (16-bit local indices)");
    kep::plan_memory(c->sym, slack);
    cudaFree(c->d_cap);
    cudaFree(c->d_arena_off);
    c->d_cap = nullptr;
    c->d_arena_off = nullptr;
    KEP_CUDA(c, upload(&c->d_cap, c->sym.capacity));
    KEP_CUDA(c, upload(&c->d_arena_off, c->sym.arena_off));
    kep_status r = build_lists(c);
    if (r != KEP_OK) return r;
    return alloc_batch(c);
}

DevPlan make_plan(kep_ctx* c) {
    DevPlan P;
    P.nf = (int32_t)c->sym.nf;
    P.forder = c->d_forder;
    P.npiv = c->d_npiv;
    P.ncb = c->d_ncb;
    P.cap = c->d_cap;
    P.child_ptr = c->d_child_ptr;
    P.child_list = c->d_child_list;
    P.level_fronts = c->d_level_fronts;
    P.piv_first = c->d_piv_first;
    P.asm_col = c->d_asm_col;
    P.cb_ptr = c->d_cb_ptr;
    P.cb_rows = c->d_cb_rows;
    P.arena_off = c->d_arena_off;
    P.asm_ptr = c->d_asm_ptr;
    P.asm_rc = c->d_asm_rc;
    P.a = c->d_a;
    P.b = c->d_b;
    P.rmap_ptr = c->d_rmap_ptr;
    P.rmap = c->d_rmap;
    P.arena = c->d_arena;
    P.arena_stride = c->sym.arena_doubles;
    P.nd_in = c->d_nd_in;
    P.nd_out = c->d_nd_out;
    P.doff = c->d_doff;
    P.stats = c->d_stats;
    P.sigma = c->d_sigma;
    P.alpha = c->d_alpha;
    P.u = c->opts.pivot_u;
    P.aux = c->d_aux;
    P.aux_stride = c->aux_stride;
    P.aux_off = c->d_aux_off;
    P.flag = c->d_flag;
    P.forced = c->d_forced;
    P.fstate = c->d_fstate;
    P.pending = c->d_pending;
    P.gscratch = c->d_gscratch;
    P.gscratch_stride = c->gscratch_stride;
    P.goff = c->d_goff;
    P.xscr = c->d_xscr;
    P.xstride = c->xstride;
    P.xoff = c->d_xoff;
    P.debug = getenv("KEP_DEBUG") ? 1 : 0;
    P.tmaps = c->d_tmaps;
    P.tmap_idx = c->d_tmap_idx;
    P.ntmap = c->ntmap;
    return P;
}

void free_store(kep_factorization* k) {
    void* ptrs[] = {k->panel, k->lab, k->d, k->ds, k->kind, k->perm, k->hdr, k->poff, k->loff, k->qoff, k->yoff,
                    k->upd, k->ybuf, k->d_bigf};
    for (void* q : ptrs) cudaFree(q);
    k->panel = nullptr; k->lab = nullptr; k->d = nullptr; k->ds = nullptr; k->kind = nullptr; k->perm = nullptr;
    k->hdr = nullptr; k->poff = nullptr; k->loff = nullptr; k->qoff = nullptr; k->yoff = nullptr;
    k->upd = nullptr; k->ybuf = nullptr; k->d_bigf = nullptr;
}

// (Re)allocate the factor store for the current memory plan (capacities).
kep_status prepare_store(kep_ctx* c, kep_factorization* k) {
    free_store(k);
    const Symbolic& S = c->sym;
    k->h_poff.assign(S.nf, 0); k->h_loff.assign(S.nf, 0); k->h_qoff.assign(S.nf, 0);
    int64_t po = 0, lo = 0, qo = 0;
    for (int64_t s = 0; s < S.nf; ++s) {
        const int64_t cap = S.capacity[s], Q = cap - S.ncb[s];
        k->h_poff[s] = po; k->h_loff[s] = lo; k->h_qoff[s] = qo;
        po += cap * Q; lo += cap; qo += Q;
    }
    k->panel_doubles = po; k->lab_ints = lo; k->q_entries = qo;
    KEP_CUDA(c, cudaMalloc(&k->panel, std::max<int64_t>(po, 1) * sizeof(double)));
    KEP_CUDA(c, cudaMalloc(&k->lab, std::max<int64_t>(lo, 1) * sizeof(int32_t)));
    KEP_CUDA(c, cudaMalloc(&k->d, std::max<int64_t>(qo, 1) * sizeof(double)));
    KEP_CUDA(c, cudaMalloc(&k->ds, std::max<int64_t>(qo, 1) * sizeof(double)));
    KEP_CUDA(c, cudaMalloc(&k->kind, std::max<int64_t>(qo, 1) * sizeof(int32_t)));
    KEP_CUDA(c, cudaMalloc(&k->perm, std::max<int64_t>(qo, 1) * sizeof(int32_t)));
    KEP_CUDA(c, cudaMalloc(&k->upd, std::max<int64_t>(lo, 1) * sizeof(double)));
    KEP_CUDA(c, cudaMalloc(&k->hdr, std::max<int64_t>(S.nf, 1) * sizeof(int4)));
    {   // large fronts: blocked multi-CTA solves with global front vectors (2 f doubles each)
        k->h_yoff.assign(std::max<int64_t>(S.nf, 1), -1);
        int64_t yo = 0;
        for (int64_t s = 0; s < S.nf; ++s)
            if (S.capacity[s] > kep::solve_big_front()) { k->h_yoff[s] = yo; yo += 2 * (int64_t)S.capacity[s]; }
        KEP_CUDA(c, cudaMalloc(&k->ybuf, std::max<int64_t>(yo, 1) * sizeof(double)));
        KEP_CUDA(c, upload(&k->yoff, k->h_yoff));
        const int nlv = (int)S.level_ptr.size() - 1;
        std::vector<int32_t> bl;
        k->big_off.assign(nlv, 0); k->big_cnt.assign(nlv, 0); k->big_fmax.assign(nlv, 0); k->big_emax.assign(nlv, 0);
        for (int L = 0; L < nlv; ++L) {
            k->big_off[L] = (int64_t)bl.size();
            for (int x = S.level_ptr[L]; x < S.level_ptr[L + 1]; ++x) {
                const int s = S.level_fronts[x];
                if (k->h_yoff[s] < 0) continue;
                bl.push_back(s);
                k->big_fmax[L] = std::max(k->big_fmax[L], (int)S.capacity[s]);
                k->big_emax[L] = std::max(k->big_emax[L], (int)(S.capacity[s] - S.ncb[s]));
            }
            k->big_cnt[L] = (int64_t)bl.size() - k->big_off[L];
        }
        KEP_CUDA(c, upload(&k->d_bigf, bl));
    }
    KEP_CUDA(c, upload(&k->poff, k->h_poff));
    KEP_CUDA(c, upload(&k->loff, k->h_loff));
    KEP_CUDA(c, upload(&k->qoff, k->h_qoff));
    const int nl = (int)S.level_ptr.size() - 1;
    k->level_fmax.assign(nl, 0);
    for (int L = 0; L < nl; ++L)
        for (int x = S.level_ptr[L]; x < S.level_ptr[L + 1]; ++x)
            if (S.capacity[S.level_fronts[x]] <= kep::solve_big_front())       // large ones: blocked kernels
                k->level_fmax[L] = std::max(k->level_fmax[L], (int)S.capacity[S.level_fronts[x]]);
    return KEP_OK;
}

// One batch of `m` shifts through every level.  Fills c->h_stats[0..m).
// keep != NULL (m == 1): the factors are copied into keep's store level by level.
kep_status run_batch(kep_ctx* c, int m, const double* sigmas, kep_factorization* keep = nullptr,
                     double alpha = 1.0, bool resid = false) {
    for (int attempt = 0; attempt < 8; ++attempt) {
        if (m > c->batch_cap) return fail(c, KEP_EINVAL, "internal: batch larger than capacity");
        if (keep) {
            kep_status r = prepare_store(c, keep);
            if (r != KEP_OK) return r;
        }
        KEP_CUDA(c, cudaMemcpyAsync(c->d_sigma, sigmas, sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
        {
            std::vector<double> al(m, alpha);
            KEP_CUDA(c, cudaMemcpyAsync(c->d_alpha, al.data(), sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
            KEP_CUDA(c, cudaStreamSynchronize(c->stream));      // al is a local buffer
        }
        kep::launch_reset_stats(c->d_stats, m, c->stream);
        c->prof.other_launches += 1;
        if (const char* fill = getenv("KEP_DEBUG_FILL"))       // debug: poison the front arena
            cudaMemsetAsync(c->d_arena, atoi(fill) & 0xff, c->arena_alloc_doubles * sizeof(double), c->stream);
        DevPlan P = make_plan(c);
        const Symbolic& S = c->sym;
        const int nl = (int)S.level_ptr.size() - 1;
        const bool prof = c->opts.profile != 0;
        size_t nev = 0;
        int cur_level = 0;
        auto mark = [&](int cls, bool begin) {
            if (!prof) return;
            if (nev >= c->ev_pool.size()) {
                cudaEvent_t ev;
                cudaEventCreate(&ev);
                c->ev_pool.push_back(ev);
                c->ev_class.push_back(0);
                c->ev_level.push_back(0);
            }
            cudaEventRecord(c->ev_pool[nev], c->stream);
            c->ev_class[nev] = begin ? cls : -1;
            c->ev_level[nev] = cur_level;
            ++nev;
        };
        for (int L = 0; L < nl; ++L) {
            const int b = S.level_ptr[L], nfl = S.level_ptr[L + 1] - b;
            cur_level = L;
            mark(KEP_K_ASSEMBLE, true);
            if (c->smitem_cnt[L]) kep::launch_asm_smem(P, c->d_smitems + c->smitem_off[L], (int)c->smitem_cnt[L], m, c->stream);
            else if (c->asm_red[L]) kep::launch_assemble_red(P, c->d_level_fronts + b, nfl, m, c->level_fmax[L], c->stream);
            else kep::launch_assemble(P, c->d_aitems + c->aitem_off[L], (int)c->aitem_cnt[L], m, false, c->stream);
            mark(KEP_K_ASSEMBLE, false);
            if (resid) kep::launch_capture(P, c->d_level_fronts + b, nfl, c->d_f0, c->stream);
            if (c->big_nf[L] > 0) {                          // large fronts, all SMs (kernels_big.cu)
                const int ng = (int)(c->big_nf[L] * m);
                const int ncta = std::max(1, std::min(148 / ng, kBigGroups));
                const int2* gp = c->d_big_groups + c->big_goff[L];
                const int64_t* so = c->d_big_scroff + c->big_goff[L];
                int* sp = c->d_big_state + 16 * c->big_goff[L];
                unsigned* bp = c->d_big_bars + c->big_goff[L];
                kep::launch_big_init(P, gp, ng, so, c->d_big_scr, sp, bp, c->stream);
                const int nblk = kep::big_blocks(c->big_qmax[L]);
                for (int blk = 0; blk < nblk; ++blk) {
                    mark(KEP_K_PANEL, true);
                    kep::launch_big_panel(P, gp, ng, ncta, so, c->d_big_scr, sp, bp, c->stream);
                    mark(KEP_K_PANEL, false);
                    mark(KEP_K_FSU, true);                   // the FS trailing update (DMMA, K = 128)
                    kep::launch_big_update(P, gp, ng, so, c->d_big_scr, sp, bp, c->stream);
                    mark(KEP_K_FSU, false);
                }
                kep::launch_big_fin(P, gp, ng, so, c->d_big_scr, sp, bp, c->stream);
                c->prof.launches[KEP_K_PANEL] += nblk;
                c->prof.launches[KEP_K_FSU] += nblk;
                c->prof.other_launches += 2;
            }
            for (const auto& g : c->sm_groups[L]) {         // whole-panel fronts; overflow -> unblocked kernel
                mark(KEP_K_PANEL, true);
                kep::launch_small(P, c->d_smfronts + g.off, (int)g.cnt, m, g.cap, g.th, c->stream);
                mark(KEP_K_PANEL, false);
                mark(KEP_K_REF, true);
                kep::launch_factor_list(P, c->d_smfronts + g.off, (int)g.cnt, m, c->stream, true);
                mark(KEP_K_REF, false);
                c->prof.launches[KEP_K_PANEL]++;
                c->prof.launches[KEP_K_REF]++;
            }
            c->prof.launches[KEP_K_ASSEMBLE]++;
            if (c->fast_cnt[L]) {
                const int32_t* fl = c->d_lists + c->fast_off[L];
                const int nfl2 = (int)c->fast_cnt[L];
                // pass 0, then kReruns passes over the fronts whose full-column test failed
                // (each with one more forced delay), then the unblocked kernel for the rest
                const auto& groups = c->fs_groups[L];
                kep::RerunLists R;
                R.d1 = c->d_rr_d1; R.d2 = c->d_rr_d2;
                R.sl[0] = c->d_litems; R.sl[1] = c->d_lsitems; R.sl[2] = c->d_lxitems; R.sl[3] = c->d_lditems;
                R.su = c->d_uitems; R.sa = c->d_aitems;
                R.fr = c->d_rr_fr; R.x = c->d_rr_x; R.cnt = c->d_rr_cnt;
                for (int k = 0; k < 4; ++k) R.l[k] = c->d_rr_l[k];
                R.u = c->d_rr_u; R.a = c->d_rr_a;
                int32_t rc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                bool anyflag = false;                   // some pass flagged a front (rerun or unblocked kernel)
                int32_t pend[2] = {0, 0};
                KEP_CUDA(c, cudaMemsetAsync(c->d_pending, 0, 2 * sizeof(int32_t), c->stream));
                for (int pass = 0; pass <= kReruns; ++pass) {
                    if (pass == 0) {
                        static const bool fs_fork_on = [] { const char* x = getenv("KEP_FS_STREAMS"); return !x || atoi(x) != 0; }();
                        const bool forked = fs_fork_on && groups.size() > 1 && groups.size() <= 8;
                        if (forked) {                   // groups 1.. on forked streams, joined before k_l21
                            if (!c->fs_fork) {
                                KEP_CUDA(c, cudaEventCreateWithFlags(&c->fs_fork, cudaEventDisableTiming));
                                for (int x = 0; x < 7; ++x) {
                                    KEP_CUDA(c, cudaStreamCreateWithFlags(&c->fs_streams[x], cudaStreamNonBlocking));
                                    KEP_CUDA(c, cudaEventCreateWithFlags(&c->fs_join[x], cudaEventDisableTiming));
                                }
                            }
                            mark(KEP_K_PANEL, true);    // one interval for the whole fork-join region
                            KEP_CUDA(c, cudaEventRecord(c->fs_fork, c->stream));
                        }
                        for (size_t gi = 0; gi < groups.size(); ++gi) { // size groups of the level's fast fronts
                            const auto& gr = groups[gi];
                            cudaStream_t gst = (forked && gi > 0) ? c->fs_streams[gi - 1] : c->stream;
                            if (forked && gi > 0) KEP_CUDA(c, cudaStreamWaitEvent(gst, c->fs_fork, 0));
                            const int64_t nbk = gr.fcnt * m;
                            const int iters = kep::fs_iters(gr.qmax, nbk);
                            for (int itn = 0; itn < iters; ++itn) {
                                if (!forked) mark(KEP_K_PANEL, true);
                                kep::launch_fsp(P, c->d_lists + gr.foff, (int)gr.fcnt, m, gr.qmax, itn == 0 ? 0 : 2, gst);
                                if (!forked) mark(KEP_K_PANEL, false);
                                c->prof.launches[KEP_K_PANEL]++;
                                if (gr.ucnt) {
                                    if (!forked) mark(KEP_K_FSU, true);
                                    kep::launch_fsu(P, c->d_uitems + gr.uoff, (int)gr.ucnt, m, gst);
                                    if (!forked) mark(KEP_K_FSU, false);
                                    c->prof.launches[KEP_K_FSU]++;
                                }
                            }
                            if (forked) {               // the group's k_l21 launches follow on its stream
                                if (gr.xcnt) kep::launch_l21x_prep(P, c->d_xfronts + gr.xoff, (int)gr.xcnt, m, gst);
                                if (gr.lcnt[2]) kep::launch_l21(P, c->d_lxitems + gr.loff[2], (int)gr.lcnt[2], m, 2, gst);
                                if (gr.lcnt[0]) kep::launch_l21(P, c->d_litems + gr.loff[0], (int)gr.lcnt[0], m, 0, gst);
                                if (gr.lcnt[1]) kep::launch_l21(P, c->d_lsitems + gr.loff[1], (int)gr.lcnt[1], m, 1, gst);
                                if (gr.lcnt[3]) kep::launch_l21(P, c->d_lditems + gr.loff[3], (int)gr.lcnt[3], m, 3, gst);
                                c->prof.launches[KEP_K_L21] += (gr.xcnt > 0) + (gr.lcnt[0] > 0) + (gr.lcnt[1] > 0) +
                                                               (gr.lcnt[2] > 0) + (gr.lcnt[3] > 0);
                            }
                            if (forked && gi > 0) {
                                KEP_CUDA(c, cudaEventRecord(c->fs_join[gi - 1], gst));
                                KEP_CUDA(c, cudaStreamWaitEvent(c->stream, c->fs_join[gi - 1], 0));
                            }
                        }
                        if (forked) mark(KEP_K_PANEL, false);
                        if (!forked && (c->litem_cnt[L] || c->lsitem_cnt[L] || c->lxitem_cnt[L] || c->lditem_cnt[L])) {
                            mark(KEP_K_L21, true);
                            kep::launch_l21x_prep(P, c->d_xfronts + c->xfront_off[L], (int)c->xfront_cnt[L], m, c->stream);
                            kep::launch_l21(P, c->d_lxitems + c->lxitem_off[L], (int)c->lxitem_cnt[L], m, 2, c->stream);
                            kep::launch_l21(P, c->d_litems + c->litem_off[L], (int)c->litem_cnt[L], m, 0, c->stream);
                            kep::launch_l21(P, c->d_lsitems + c->lsitem_off[L], (int)c->lsitem_cnt[L], m, 1, c->stream);
                            kep::launch_l21(P, c->d_lditems + c->lditem_off[L], (int)c->lditem_cnt[L], m, 3, c->stream);
                            mark(KEP_K_L21, false);
                            c->prof.launches[KEP_K_L21] += 2 * (c->lxitem_cnt[L] > 0) + (c->litem_cnt[L] > 0) + (c->lsitem_cnt[L] > 0) +
                                                           (c->lditem_cnt[L] > 0);
                        }
                        mark(KEP_K_CHECK, true);
                        kep::launch_check(P, fl, nfl2, m, c->stream);
                        mark(KEP_K_CHECK, false);
                    } else {
                        // rerun pass: the flagged fronts only, one launch configuration for the largest
                        // flagged FS block
                        KEP_CUDA(c, cudaMemsetAsync(c->d_pending, 0, 2 * sizeof(int32_t), c->stream));
                        const int qr = std::min(pend[1], c->level_qmax[L]);
                        const int64_t nbk = (int64_t)rc[0] * m;
                        const int nbl = kep::front_nb_for(qr, nbk);
                        const int iters = std::min(kep::fs_iters(qr, nbk), (qr + nbl - 2) / (nbl - 1) + 1);
                        for (int itn = 0; itn < iters; ++itn) {
                            mark(KEP_K_PANEL, true);
                            kep::launch_fsp(P, c->d_rr_fr, rc[0], m, qr, itn == 0 ? 1 : 2, c->stream);
                            mark(KEP_K_PANEL, false);
                            c->prof.launches[KEP_K_PANEL]++;
                            if (rc[4]) {
                                mark(KEP_K_FSU, true);
                                kep::launch_fsu(P, c->d_rr_u, rc[4], m, c->stream);
                                mark(KEP_K_FSU, false);
                                c->prof.launches[KEP_K_FSU]++;
                            }
                        }
                        mark(KEP_K_L21, true);
                        kep::launch_l21x_prep(P, c->d_rr_x, rc[6], m, c->stream);
                        kep::launch_l21(P, c->d_rr_l[2], rc[3], m, 2, c->stream);
                        kep::launch_l21(P, c->d_rr_l[0], rc[1], m, 0, c->stream);
                        kep::launch_l21(P, c->d_rr_l[1], rc[2], m, 1, c->stream);
                        kep::launch_l21(P, c->d_rr_l[3], rc[7], m, 3, c->stream);
                        mark(KEP_K_L21, false);
                        c->prof.launches[KEP_K_L21] += 4;
                        mark(KEP_K_CHECK, true);
                        kep::launch_check(P, c->d_rr_fr, rc[0], m, c->stream);
                        mark(KEP_K_CHECK, false);
                    }
                    // fronts whose full-column test failed: compact lists, restore by re-assembly
                    mark(KEP_K_CHECK, true);
                    kep::launch_rerun_lists(P, fl, nfl2, m, R, c->stream);
                    mark(KEP_K_CHECK, false);
                    KEP_CUDA(c, cudaMemcpyAsync(pend, c->d_pending, sizeof(pend), cudaMemcpyDeviceToHost, c->stream));
                    KEP_CUDA(c, cudaMemcpyAsync(rc, c->d_rr_cnt, sizeof(rc), cudaMemcpyDeviceToHost, c->stream));
                    KEP_CUDA(c, cudaStreamSynchronize(c->stream));
                    c->prof.launches[KEP_K_CHECK] += 2;
                    if (rc[5] == 0) break;              // nothing flagged
                    anyflag = true;
                    mark(KEP_K_CHECK, true);
                    kep::launch_assemble(P, c->d_rr_a, rc[5], m, true, c->stream);
                    mark(KEP_K_CHECK, false);
                    c->prof.launches[KEP_K_CHECK]++;
                    if (rc[0] == 0) break;              // only fronts for the unblocked kernel
                }
                if (anyflag) {                          // fronts left for the unblocked kernel (flag != FL_OK)
                    mark(KEP_K_REF, true);
                    kep::launch_factor_list(P, fl, nfl2, m, c->stream, true);
                    mark(KEP_K_REF, false);
                    c->prof.launches[KEP_K_REF]++;
                }
            }
            if (c->ref_cnt[L]) {
                mark(KEP_K_REF, true);
                kep::launch_factor_list(P, c->d_lists + c->ref_off[L], (int)c->ref_cnt[L], m, c->stream);
                mark(KEP_K_REF, false);
                c->prof.launches[KEP_K_REF]++;
            }
            if (keep) kep::launch_store(P, keep->plan(), c->d_level_fronts + b, nfl, c->stream);
            if (c->item_cnt[L] || c->small_cnt[L]) {
                const bool tma = c->use_tma && c->tma_level[L];
                const int cls = tma ? KEP_K_SCHUR_TMA : KEP_K_SCHUR;
                mark(cls, true);
                if (tma) kep::launch_schur_tma(P, c->d_items + c->item_off[L], (int)c->item_cnt[L], m, c->stream);
                else kep::launch_schur(P, c->d_items + c->item_off[L], (int)c->item_cnt[L], m, c->stream);
                kep::launch_schur_small(P, c->d_small + c->small_off[L], (int)c->small_cnt[L], m, c->small_cmax[L],
                                        c->small_kmax[L], c->stream);
                mark(cls, false);
                c->prof.launches[cls] += (c->item_cnt[L] ? 1 : 0) + (c->small_cnt[L] ? 1 : 0);
                c->prof.schur_flops += c->item_flops[L] * m;
                if (tma) c->prof.schur_tma_flops += c->item_flops[L] * m;
            }
            if (resid)
                kep::launch_resid(P, keep->plan(), c->d_ritems + c->ritem_off[L], (int)c->ritem_cnt[L], c->d_f0,
                                  c->d_resid, c->stream);
        }
        KEP_CUDA(c, cudaGetLastError());
        KEP_CUDA(c, cudaMemcpyAsync(c->h_stats.data(), c->d_stats, sizeof(ShiftStat) * m, cudaMemcpyDeviceToHost, c->stream));
        KEP_CUDA(c, cudaStreamSynchronize(c->stream));
        for (size_t x = 0; x + 1 < nev; x += 2) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, c->ev_pool[x], c->ev_pool[x + 1]);
            c->prof.ms[c->ev_class[x]] += ms;
            if ((int)c->lvl_ms.size() <= c->ev_level[x]) c->lvl_ms.resize(c->ev_level[x] + 1, {});
            c->lvl_ms[c->ev_level[x]][c->ev_class[x]] += ms;
        }
        c->prof.shifts += m;
        c->prof.factor_flops += c->sym.flops * m;
        int need = 0;
        bool over = false;
        for (int i = 0; i < m; ++i)
            if (c->h_stats[i].flags & kep::FLAG_OVERFLOW) { over = true; need = std::max(need, c->h_stats[i].need_slack); }
        if (getenv("KEP_DEBUG"))
            fprintf(stderr, "[kep] batch m=%d attempt=%d overflow=%d need=%d slack=%d\n", m, attempt, (int)over, need,
                    c->sym.slack);
        if (!over) return KEP_OK;
        int slack = std::max(2 * c->sym.slack, need + 8);
        kep_status r = replan(c, slack);
        if (r != KEP_OK) return r;
        m = std::min(m, c->batch_cap);
    }
    return fail(c, KEP_ENOMEM, "delayed-pivot slack kept overflowing");
}

double bits_to_double(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof(d));
    return d;
}

}  // namespace

extern "C" {

void kep_default_opts(kep_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->ordering = KEP_ORDER_AUTO;
    o->user_perm = nullptr;
    o->amalgamate = 1;
    o->nrelax = 48;
    o->relax_frac = 0.05;
    o->pivot_u = 0.01;
    o->tau_sing = 1e-14;
    o->delay_slack = 16;
    o->max_batch = 16;
    o->device = -1;
    o->stream = nullptr;
    o->kernel_variant = 0;
    o->profile = 0;
}

const char* kep_version(void) { return "kep 0.1 sm_100a"; }

const char* kep_status_string(kep_status s) {
    switch (s) {
        case KEP_OK: return "KEP_OK";
        case KEP_EINVAL: return "KEP_EINVAL";
        case KEP_EPATTERN: return "KEP_EPATTERN";
        case KEP_ESINGULAR: return "KEP_ESINGULAR";
        case KEP_ENOTSPD: return "KEP_ENOTSPD";
        case KEP_ENOMEM: return "KEP_ENOMEM";
        case KEP_ECUDA: return "KEP_ECUDA";
        case KEP_EBREAKDOWN: return "KEP_EBREAKDOWN";
        case KEP_ENOCONV: return "KEP_ENOCONV";
        case KEP_ECLUSTER: return "KEP_ECLUSTER";
        case KEP_ENODEVICE: return "KEP_ENODEVICE";
    }
    return "KEP_UNKNOWN";
}

const char* kep_last_error(const kep_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

kep_status kep_analyze(int64_t n, const int64_t* colptr, const int32_t* rowidx, const kep_opts* opts, kep_ctx** out) {
    if (!out) return fail(nullptr, KEP_EINVAL, "out is NULL");
    *out = nullptr;
    kep_ctx* c = new (std::nothrow) kep_ctx();
    if (!c) return fail(nullptr, KEP_ENOMEM, "host allocation failed");
    std::memset(&c->prof, 0, sizeof(c->prof));
    if (opts) c->opts = *opts; else kep_default_opts(&c->opts);
    if (c->opts.pivot_u <= 0.0 || c->opts.pivot_u > 0.5) { delete c; return fail(nullptr, KEP_EINVAL, "pivot_u must be in (0, 0.5]"); }
    if (c->opts.max_batch < 1) c->opts.max_batch = 1;
    if (c->opts.delay_slack < 0) c->opts.delay_slack = 0;
    kep::SymbolicOptions so;
    so.ordering = (int)c->opts.ordering;
    so.user_perm = c->opts.user_perm;
    so.amalgamate = c->opts.amalgamate != 0;
    so.nrelax = c->opts.nrelax;
    so.relax_frac = c->opts.relax_frac;
    so.delay_slack = c->opts.delay_slack;
    std::string msg;
    try {
        msg = kep::analyze(n, colptr, rowidx, so, c->sym);
    } catch (const std::bad_alloc&) {
        delete c;
        return fail(nullptr, KEP_ENOMEM, "host allocation failed during analysis");
    } catch (const std::exception& e) {
        delete c;
        return fail(nullptr, KEP_EINVAL, e.what());
    }
    if (!msg.empty()) { delete c; return fail(nullptr, KEP_EINVAL, msg); }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        c->have_device = false;           // symbolic queries still work (CPU-only hosts)
        *out = c;
        return KEP_OK;
    }
    c->device = c->opts.device >= 0 ? c->opts.device : 0;
    if (c->opts.device < 0) cudaGetDevice(&c->device);
    if (cudaSetDevice(c->device) != cudaSuccess) { delete c; return fail(nullptr, KEP_ENODEVICE, "cudaSetDevice failed"); }
    c->have_device = true;
    if (c->opts.stream) c->stream = (cudaStream_t)c->opts.stream;
    else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) { delete c; return fail(nullptr, KEP_ECUDA, "stream creation failed"); }
        c->own_stream = true;
    }
    kep_status st = upload_plan(c, colptr, rowidx);
    if (st != KEP_OK) { std::string m = c->err; kep_destroy(c); return fail(nullptr, st, m); }
    *out = c;
    return KEP_OK;
}

kep_status kep_set_values_dev(kep_ctx* c, const double* a_dev, const double* b_dev) {
    if (!c || !a_dev || !b_dev) return fail(c, KEP_EINVAL, "null argument");
    if (!c->have_device) return fail(c, KEP_ENODEVICE, "no CUDA device");
    KEP_CUDA(c, cudaSetDevice(c->device));
    kep::launch_gather(a_dev, c->d_asm_src, c->d_a, c->sym.nnz, c->stream);
    kep::launch_gather(b_dev, c->d_asm_src, c->d_b, c->sym.nnz, c->stream);
    kep::launch_gather(a_dev, c->d_csr_src, c->d_csr_a, c->csr_nnz, c->stream);
    kep::launch_gather(b_dev, c->d_csr_src, c->d_csr_b, c->csr_nnz, c->stream);
    KEP_CUDA(c, cudaGetLastError());
    KEP_CUDA(c, cudaStreamSynchronize(c->stream));
    c->values_set = true;
    return KEP_OK;
}

kep_status kep_set_values(kep_ctx* c, const double* a, const double* b) {
    if (!c || !a || !b) return fail(c, KEP_EINVAL, "null argument");
    if (!c->have_device) return fail(c, KEP_ENODEVICE, "no CUDA device");
    KEP_CUDA(c, cudaSetDevice(c->device));
    const size_t bytes = (size_t)c->sym.nnz * sizeof(double);
    if (!c->d_stage) {                 // staging for the host values, kept for the next call
        cudaError_t e = cudaMalloc(&c->d_stage, 2 * std::max<size_t>(bytes, 8));
        if (e != cudaSuccess) { c->d_stage = nullptr; return fail(c, KEP_ENOMEM, "cudaMalloc failed"); }
    }
    double* ta = c->d_stage;
    double* tb = c->d_stage + std::max<size_t>(c->sym.nnz, 1);
    cudaError_t e = cudaMemcpyAsync(ta, a, bytes, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tb, b, bytes, cudaMemcpyHostToDevice, c->stream);
    kep_status st = KEP_OK;
    if (e != cudaSuccess) st = fail(c, KEP_ECUDA, cudaGetErrorString(e));
    else st = kep_set_values_dev(c, ta, tb);
    cudaStreamSynchronize(c->stream);    // the caller may reuse its host buffers on return
    return st;
}

kep_status kep_inertia_many(kep_ctx* c, int32_t m, const double* sigmas, int64_t* nus, kep_status* per_shift,
                            kep_inertia_info* infos) {
    if (!c || (m > 0 && (!sigmas || !nus || !per_shift))) return fail(c, KEP_EINVAL, "null argument");
    if (m < 0) return fail(c, KEP_EINVAL, "m < 0");
    if (!c->have_device) return fail(c, KEP_ENODEVICE, "no CUDA device");
    if (!c->values_set) return fail(c, KEP_EINVAL, "kep_set_values must precede kep_inertia");
    KEP_CUDA(c, cudaSetDevice(c->device));
    int done = 0;
    while (done < m) {
        // equal-sized batches (16 shifts at capacity 12 run as 8 + 8, not 12 + 4)
        const int left = m - done;
        const int nbat = (left + c->batch_cap - 1) / c->batch_cap;
        const int b = (left + nbat - 1) / nbat;
        kep_status st = run_batch(c, b, sigmas + done);
        if (st != KEP_OK) return st;
        const int got = std::min(b, c->batch_cap);     // a replan may shrink the batch
        for (int i = 0; i < got; ++i) {
            const ShiftStat& s = c->h_stats[i];
            const double minpiv = bits_to_double(s.minpiv_bits);
            const double smax = bits_to_double(s.smax_bits);
            const bool singular = s.n_zero > 0 || minpiv <= c->opts.tau_sing * smax;
            per_shift[done + i] = singular ? KEP_ESINGULAR : KEP_OK;
            if (!singular) nus[done + i] = (int64_t)s.n_neg;
            if (infos) {
                kep_inertia_info& I = infos[done + i];
                I.n_neg = (int64_t)s.n_neg;
                I.n_zero = (int64_t)s.n_zero;
                I.n_pos = (int64_t)s.n_pos;
                I.n_2x2 = (int64_t)s.n_2x2;
                I.n_delayed = (int64_t)s.n_delayed;
                I.min_abs_pivot = minpiv >= DBL_MAX ? 0.0 : minpiv;
                I.max_abs_entry = smax;
                I.n_redo = (int64_t)s.n_redo;
            }
        }
        done += got;
    }
    return KEP_OK;
}

kep_status kep_inertia(kep_ctx* c, double sigma, int64_t* nu, kep_inertia_info* info) {
    if (!nu) return fail(c, KEP_EINVAL, "nu is NULL");
    kep_status per = KEP_OK;
    int64_t v = 0;
    kep_status st = kep_inertia_many(c, 1, &sigma, &v, &per, info);
    if (st != KEP_OK) return st;
    if (per == KEP_OK) *nu = v;
    return per;
}

kep_status kep_factor(kep_ctx* c, double sigma, kep_factorization** out) {
    return kep_factor_pencil(c, 1.0, sigma, out);
}

kep_status kep_factor_pencil(kep_ctx* c, double alpha, double sigma, kep_factorization** out) {
    if (!c || !out) return fail(c, KEP_EINVAL, "null argument");
    *out = nullptr;
    if (!c->have_device) return fail(c, KEP_ENODEVICE, "no CUDA device");
    if (!c->values_set) return fail(c, KEP_EINVAL, "kep_set_values must precede kep_factor");
    KEP_CUDA(c, cudaSetDevice(c->device));
    kep_factorization* k = new (std::nothrow) kep_factorization();
    if (!k) return fail(c, KEP_ENOMEM, "host allocation failed");
    k->ctx = c;
    k->sigma = sigma;
    k->alpha = alpha;
    kep_status st = run_batch(c, 1, &sigma, k, alpha);
    if (st != KEP_OK) { kep_factor_destroy(k); return st; }
    const ShiftStat& S = c->h_stats[0];
    const double minpiv = bits_to_double(S.minpiv_bits), smax = bits_to_double(S.smax_bits);
    kep_inertia_info& I = k->info;
    I.n_neg = (int64_t)S.n_neg; I.n_zero = (int64_t)S.n_zero; I.n_pos = (int64_t)S.n_pos;
    I.n_2x2 = (int64_t)S.n_2x2; I.n_delayed = (int64_t)S.n_delayed;
    I.min_abs_pivot = minpiv >= DBL_MAX ? 0.0 : minpiv;
    I.max_abs_entry = smax;
    I.n_redo = (int64_t)S.n_redo;
    k->nu = I.n_neg;
    if (S.n_zero > 0 || minpiv <= c->opts.tau_sing * smax) {
        kep_factor_destroy(k);
        return fail(c, KEP_ESINGULAR, "A - sigma B is numerically singular at this shift");
    }
    const int64_t n = c->sym.n;
    cudaError_t e1 = cudaMalloc(&k->xw, std::max<int64_t>(n, 1) * sizeof(double));
    cudaError_t e2 = cudaMalloc(&k->bw, std::max<int64_t>(n, 1) * sizeof(double));
    if (e1 != cudaSuccess || e2 != cudaSuccess) { kep_factor_destroy(k); return fail(c, KEP_ENOMEM, "cudaMalloc failed"); }
    c->factors.push_back(k);
    *out = k;
    return KEP_OK;
}

kep_status kep_factor_residual(kep_ctx* c, double sigma, double* bound, double* max_front) {
    if (!c || !bound) return fail(c, KEP_EINVAL, "null argument");
    if (!c->have_device) return fail(c, KEP_ENODEVICE, "no CUDA device");
    if (!c->values_set) return fail(c, KEP_EINVAL, "kep_set_values must precede kep_factor_residual");
    KEP_CUDA(c, cudaSetDevice(c->device));
    const Symbolic& S = c->sym;
    const int nl = (int)S.level_ptr.size() - 1;
    kep_factorization* k = new (std::nothrow) kep_factorization();
    if (!k) return fail(c, KEP_ENOMEM, "host allocation failed");
    k->ctx = c;
    k->sigma = sigma;
    kep_status st = KEP_OK;
    for (int attempt = 0; attempt < 4; ++attempt) {
        // residual tiles (front, I, J) of every level, by capacity (fronts may grow by delays)
        std::vector<int4> it;
        c->ritem_off.assign(nl, 0);
        c->ritem_cnt.assign(nl, 0);
        const int RB = kep::resid_tile();
        for (int L = 0; L < nl; ++L) {
            c->ritem_off[L] = (int64_t)it.size();
            for (int x = S.level_ptr[L]; x < S.level_ptr[L + 1]; ++x) {
                const int s = S.level_fronts[x];
                const int nt = (S.capacity[s] + RB - 1) / RB;
                for (int I = 0; I < nt; ++I)
                    for (int J = 0; J <= I; ++J) it.push_back(make_int4(s, I, J, 0));
            }
            c->ritem_cnt[L] = (int64_t)it.size() - c->ritem_off[L];
        }
        cudaFree(c->d_ritems); c->d_ritems = nullptr;
        cudaFree(c->d_f0); c->d_f0 = nullptr;
        cudaFree(c->d_resid); c->d_resid = nullptr;
        KEP_CUDA(c, upload(&c->d_ritems, it));
        KEP_CUDA(c, cudaMalloc(&c->d_f0, std::max<int64_t>(S.arena_doubles, 1) * sizeof(double)));
        KEP_CUDA(c, cudaMalloc(&c->d_resid, std::max<int64_t>(S.nf, 1) * 4 * sizeof(double)));
        KEP_CUDA(c, cudaMemsetAsync(c->d_resid, 0, std::max<int64_t>(S.nf, 1) * 4 * sizeof(double), c->stream));
        const int32_t slack0 = S.slack;
        st = run_batch(c, 1, &sigma, k, 1.0, true);
        if (st != KEP_OK || S.slack == slack0) break;         // a replan changes capacities: redo the tiles
    }
    if (st == KEP_OK) {
        std::vector<double> r(std::max<int64_t>(S.nf, 1) * 4);
        KEP_CUDA(c, cudaMemcpy(r.data(), c->d_resid, sizeof(double) * r.size(), cudaMemcpyDeviceToHost));
        double sum = 0.0, mx = 0.0;
        const bool dbg = getenv("KEP_DEBUG_RESID") != nullptr;
        std::vector<int4> hdr;
        if (dbg) {
            hdr.resize(S.nf);
            KEP_CUDA(c, cudaMemcpy(hdr.data(), k->hdr, sizeof(int4) * S.nf, cudaMemcpyDeviceToHost));
        }
        if (const char* dump = getenv("KEP_DEBUG_DUMP")) {      // one front: F0, arena, perm, store
            const int64_t s2 = atoll(dump);
            const int4 h = hdr[s2];
            const int f = h.y, ld = kep::ldpad(S.capacity[s2]), q = h.z, e = h.x;
            std::vector<double> f0((size_t)f * ld), fa((size_t)f * ld), pan((size_t)f * e);
            std::vector<double> aux((size_t)(S.capacity[s2] - S.ncb[s2]) * kep::AUX_W);
            std::vector<int64_t> aoff(S.nf);
            cudaMemcpy(aoff.data(), c->d_aux_off, sizeof(int64_t) * S.nf, cudaMemcpyDeviceToHost);
            cudaMemcpy(f0.data(), c->d_f0 + S.arena_off[s2], f0.size() * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(fa.data(), c->d_arena + S.arena_off[s2], fa.size() * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(pan.data(), k->panel + k->h_poff[s2], pan.size() * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(aux.data(), c->d_aux + aoff[s2] * kep::AUX_W, aux.size() * 8, cudaMemcpyDeviceToHost);
            std::vector<int32_t> lab(f);
            cudaMemcpy(lab.data(), k->lab + k->h_loff[s2], f * 4, cudaMemcpyDeviceToHost);
            FILE* fp = fopen("gpurun_out/dump_front.bin", "wb");
            int hd[6] = {e, f, q, h.w, ld, S.capacity[s2] - S.ncb[s2]};
            fwrite(hd, 4, 6, fp);
            fwrite(f0.data(), 8, f0.size(), fp); fwrite(fa.data(), 8, fa.size(), fp); fwrite(pan.data(), 8, pan.size(), fp);
            fwrite(aux.data(), 8, aux.size(), fp); fwrite(lab.data(), 4, lab.size(), fp);
            fclose(fp);
        }
        for (int64_t s2 = 0; s2 < S.nf; ++s2) {
            const double v = std::sqrt(std::max(r[4 * s2], 0.0));
            sum += v;
            mx = std::max(mx, v);
            if (dbg && v > 1e-12)
                fprintf(stderr, "[resid] front %lld e=%d f=%d q=%d flag=%d p=%d c=%d |E|=%.3e FSxE=%.3e CBxE=%.3e TT=%.3e\n",
                        (long long)s2, hdr[s2].x, hdr[s2].y, hdr[s2].z, hdr[s2].w, (int)S.npiv[s2], (int)S.ncb[s2], v,
                        std::sqrt(r[4 * s2 + 1]), std::sqrt(r[4 * s2 + 2]), std::sqrt(r[4 * s2 + 3]));
        }
        *bound = sum;
        if (max_front) *max_front = mx;
    }
    cudaFree(c->d_ritems); c->d_ritems = nullptr;
    cudaFree(c->d_f0); c->d_f0 = nullptr;
    cudaFree(c->d_resid); c->d_resid = nullptr;
    free_store(k);
    delete k;
    return st;
}

kep_status kep_factor_info(const kep_factorization* k, kep_factor_stats* out) {
    if (!k || !out) return KEP_EINVAL;
    out->sigma = k->sigma;
    out->nu = k->nu;
    out->inertia = k->info;
    out->n = k->ctx->sym.n;
    std::vector<int4> hdr(k->ctx->sym.nf);
    if (cudaMemcpy(hdr.data(), k->hdr, sizeof(int4) * hdr.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        return KEP_ECUDA;
    int64_t nnz = 0;
    for (const int4& h : hdr)
        for (int t = 0; t < h.x; ++t) nnz += h.y - t - 1;
    out->nnz_L = nnz;
    out->store_bytes = k->panel_doubles * 8 + k->lab_ints * 4 + k->q_entries * 20;
    return KEP_OK;
}

// x = S^-1 b on the device, positions space: b_dev / x_dev in dof order (n doubles each).
kep_status kep_solve_dev(const kep_factorization* k, const double* b_dev, double* x_dev) {
    if (!k || !b_dev || !x_dev) return KEP_EINVAL;
    kep_ctx* c = k->ctx;
    KEP_CUDA(c, cudaSetDevice(c->device));
    const Symbolic& S = c->sym;
    const int nl = (int)S.level_ptr.size() - 1;
    kep::launch_gather(b_dev, c->d_perm, k->xw, S.n, c->stream);          // to elimination positions
    const kep::StorePlan T = k->plan();
    const DevPlan P = make_plan(c);
    for (int L = 0; L < nl; ++L) {
        kep::launch_fwd(P, T, c->d_level_fronts + S.level_ptr[L], S.level_ptr[L + 1] - S.level_ptr[L], k->level_fmax[L],
                        k->xw, c->stream);
        kep::launch_fwd_big(P, T, k->d_bigf + k->big_off[L], (int)k->big_cnt[L], k->big_fmax[L], k->big_emax[L], k->xw,
                            c->stream);
    }
    for (int L = nl - 1; L >= 0; --L) {
        kep::launch_bwd_big(T, k->d_bigf + k->big_off[L], (int)k->big_cnt[L], k->big_fmax[L], k->big_emax[L], k->xw,
                            c->stream);
        kep::launch_bwd(T, c->d_level_fronts + S.level_ptr[L], S.level_ptr[L + 1] - S.level_ptr[L], k->level_fmax[L],
                        k->xw, c->stream);
    }
    kep::launch_gather(k->xw, c->d_iperm, x_dev, S.n, c->stream);         // back to dofs
    KEP_CUDA(c, cudaGetLastError());
    return KEP_OK;
}

kep_status kep_solve(const kep_factorization* k, int32_t nrhs, const double* b, int64_t ldb, double* x, int64_t ldx) {
    if (!k || (nrhs > 0 && (!b || !x))) return KEP_EINVAL;
    kep_ctx* c = k->ctx;
    const int64_t n = c->sym.n;
    if (nrhs < 0 || ldb < n || ldx < n) return fail(c, KEP_EINVAL, "nrhs < 0 or leading dimension < n");
    KEP_CUDA(c, cudaSetDevice(c->device));
    for (int32_t r = 0; r < nrhs; ++r) {
        KEP_CUDA(c, cudaMemcpyAsync(k->bw, b + (size_t)r * ldb, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        kep_status st = kep_solve_dev(k, k->bw, k->bw);
        if (st != KEP_OK) return st;
        KEP_CUDA(c, cudaMemcpyAsync(x + (size_t)r * ldx, k->bw, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    }
    KEP_CUDA(c, cudaStreamSynchronize(c->stream));
    return KEP_OK;
}

kep_status kep_factor_export(const kep_factorization* k, int64_t* perm, double* d, double* dsub, int64_t* Lcolptr,
                             int32_t* Lrowidx, double* Lval) {
    if (!k || !perm || !d || !dsub || !Lcolptr) return KEP_EINVAL;
    kep_ctx* c = k->ctx;
    const Symbolic& S = c->sym;
    const int64_t n = S.n, nf = S.nf;
    std::vector<int4> hdr(nf);
    std::vector<int32_t> lab(k->lab_ints), kind(k->q_entries);
    std::vector<double> dd(k->q_entries), ds(k->q_entries);
    KEP_CUDA(c, cudaMemcpy(hdr.data(), k->hdr, sizeof(int4) * nf, cudaMemcpyDeviceToHost));
    KEP_CUDA(c, cudaMemcpy(lab.data(), k->lab, sizeof(int32_t) * lab.size(), cudaMemcpyDeviceToHost));
    KEP_CUDA(c, cudaMemcpy(kind.data(), k->kind, sizeof(int32_t) * kind.size(), cudaMemcpyDeviceToHost));
    KEP_CUDA(c, cudaMemcpy(dd.data(), k->d, sizeof(double) * dd.size(), cudaMemcpyDeviceToHost));
    KEP_CUDA(c, cudaMemcpy(ds.data(), k->ds, sizeof(double) * ds.size(), cudaMemcpyDeviceToHost));
    // elimination index of every variable (fronts in postorder, eliminated positions in order)
    std::vector<int64_t> elim_of(n, -1);
    int64_t kk = 0;
    for (int64_t s = 0; s < nf; ++s)
        for (int t = 0; t < hdr[s].x; ++t) {
            const int32_t v = lab[k->h_loff[s] + t];
            if (v < 0 || v >= n || elim_of[v] >= 0) return fail(c, KEP_ECUDA, "inconsistent factor labels");
            elim_of[v] = kk;
            perm[kk] = S.perm[v];
            const int64_t qi = k->h_qoff[s] + t;
            d[kk] = dd[qi];
            dsub[kk] = kind[qi] == kep::PK_2X2A ? ds[qi] : 0.0;
            ++kk;
        }
    if (kk != n) return fail(c, KEP_ECUDA, "factor does not eliminate every variable");
    // column counts, then entries (structural, rows sorted)
    Lcolptr[0] = 0;
    for (int64_t s = 0; s < nf; ++s)
        for (int t = 0; t < hdr[s].x; ++t) {
            const int64_t col = elim_of[lab[k->h_loff[s] + t]];
            Lcolptr[col + 1] = hdr[s].y - t - 1;
        }
    for (int64_t j = 0; j < n; ++j) Lcolptr[j + 1] += Lcolptr[j];
    if (!Lrowidx || !Lval) return KEP_OK;                    // sizes only
    std::vector<double> col;
    std::vector<std::pair<int64_t, double>> ent;
    for (int64_t s = 0; s < nf; ++s) {
        const int e = hdr[s].x, f = hdr[s].y;
        if (e == 0) continue;
        col.resize((size_t)f * e);
        KEP_CUDA(c, cudaMemcpy(col.data(), k->panel + k->h_poff[s], sizeof(double) * col.size(), cudaMemcpyDeviceToHost));
        for (int t = 0; t < e; ++t) {
            const int64_t j = elim_of[lab[k->h_loff[s] + t]];
            ent.clear();
            for (int i = t + 1; i < f; ++i) ent.emplace_back(elim_of[lab[k->h_loff[s] + i]], col[(size_t)t * f + i]);
            std::sort(ent.begin(), ent.end());
            int64_t w = Lcolptr[j];
            for (auto& pr : ent) {
                if (pr.first <= j) return fail(c, KEP_ECUDA, "factor entry above the diagonal");
                Lrowidx[w] = (int32_t)pr.first;
                Lval[w] = pr.second;
                ++w;
            }
        }
    }
    return KEP_OK;
}

void kep_factor_destroy(kep_factorization* k) {
    if (!k) return;
    if (k->ctx) {
        auto& v = k->ctx->factors;
        v.erase(std::remove(v.begin(), v.end(), k), v.end());
    }
    if (k->ctx && k->ctx->have_device) {
        cudaSetDevice(k->ctx->device);
        cudaStreamSynchronize(k->ctx->stream);
        free_store(k);
        cudaFree(k->xw);
        cudaFree(k->bw);
    }
    delete k;
}

void kep_default_kth_opts(kep_kth_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->m_max = 20;
    o->tau_res = 1e-10;
    o->tau_diff = 1e-10;
    o->max_lanczos = 64;
    o->max_bisect = 128;
    o->max_si = 500;
    o->shifts_per_round = 1;
    o->seed = 1;
    o->bisect_only = 0;
    o->bisect_rtol = 1e-14;
}

namespace {

// splitmix64 -> uniform(-1, 1)
void seeded_uniform(uint64_t seed, int64_t n, std::vector<double>& v) {
    v.resize(n);
    uint64_t x = seed;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t z = (x += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        v[i] = 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
    }
}

struct DevVec {
    double* p = nullptr;
    ~DevVec() { cudaFree(p); }
};

// Lanczos helpers on the ctx stream (dot products come back to the host)
struct Lz {
    kep_ctx* c;
    double* dtmp = nullptr;          // device scratch for reductions (>= 512 doubles)
    double dot(const double* x, const double* y) {
        kep::launch_gemv_t(x, 0, 1, y, c->sym.n, dtmp, c->stream);
        double v = 0.0;
        cudaMemcpyAsync(&v, dtmp, sizeof(double), cudaMemcpyDeviceToHost, c->stream);
        cudaStreamSynchronize(c->stream);
        return v;
    }
    void spmv(const double* x, double* ya, double* yb) {
        kep::launch_spmv2(c->d_csr_rp, c->d_csr_ci, c->d_csr_a, c->d_csr_b, x, ya, yb, c->sym.n, c->stream);
    }
    // r -= U (V^T r), twice (full reorthogonalisation in the B-inner product)
    void reorth(const double* V, const double* U, int j, double* r) {
        for (int pass = 0; pass < 2; ++pass) {
            kep::launch_gemv_t(V, c->sym.n, j, r, c->sym.n, dtmp, c->stream);
            kep::launch_combine(U, c->sym.n, j, dtmp, -1.0, 1.0, r, 0.0, nullptr, 0.0, nullptr, c->sym.n, c->stream);
        }
    }
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

kep_status kep_kth_eigenpair(kep_ctx* c, int64_t k, const kep_kth_opts* opts_in, double* lambda, double* x,
                             kep_kth_report* rep_out) {
    if (!c || !lambda) return fail(c, KEP_EINVAL, "null argument");
    if (!c->have_device) return fail(c, KEP_ENODEVICE, "no CUDA device");
    if (!c->values_set) return fail(c, KEP_EINVAL, "kep_set_values must precede kep_kth_eigenpair");
    const int64_t n = c->sym.n;
    if (k < 1 || k > n) return fail(c, KEP_EINVAL, "k out of range");
    kep_kth_opts o;
    if (opts_in) o = *opts_in; else kep_default_kth_opts(&o);
    if (o.m_max < 1 || o.m_max > 32) return fail(c, KEP_EINVAL, "m_max must be in [1, 32]");
    if (o.shifts_per_round < 1) o.shifts_per_round = 1;
    KEP_CUDA(c, cudaSetDevice(c->device));
    kep_kth_report R;
    std::memset(&R, 0, sizeof(R));
    R.status = KEP_OK;
    Lz L{c};
    DevVec tmp;
    KEP_CUDA(c, cudaMalloc(&tmp.p, sizeof(double) * 1024));
    L.dtmp = tmp.p;
    auto nu_at = [&](double& sig, int64_t& nu) -> kep_status {     // nu_sigma, perturbing an exact hit
        for (int t = 0; t < 8; ++t) {
            kep_status st = kep_inertia(c, sig, &nu, nullptr);
            if (st == KEP_OK) return KEP_OK;
            if (st != KEP_ESINGULAR) return st;
            sig += (std::fabs(sig) + 1e-300) * 1e-12 * (1 << t);
        }
        return fail(c, KEP_ESINGULAR, "shift stays singular after perturbation");
    };
    // ------------------------------------------------------------ stage 1 (Alg. 2)
    double t0 = now_s();
    const int J1 = std::max(2, o.max_lanczos);
    DevVec V, U, w, r, yb;
    KEP_CUDA(c, cudaMalloc(&V.p, sizeof(double) * n * (J1 + 1)));
    KEP_CUDA(c, cudaMalloc(&U.p, sizeof(double) * n * (J1 + 1)));
    KEP_CUDA(c, cudaMalloc(&w.p, sizeof(double) * n));
    KEP_CUDA(c, cudaMalloc(&r.p, sizeof(double) * n));
    KEP_CUDA(c, cudaMalloc(&yb.p, sizeof(double) * n));
    std::vector<double> h0;
    if (o.v0_stage1) h0.assign(o.v0_stage1, o.v0_stage1 + n); else seeded_uniform(o.seed, n, h0);
    KEP_CUDA(c, cudaMemcpyAsync(V.p, h0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    L.spmv(V.p, nullptr, yb.p);
    double nb = std::sqrt(L.dot(V.p, yb.p));
    kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 1.0 / nb, V.p, 0.0, nullptr, 0.0, nullptr, n, c->stream);
    kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 0.0, U.p, 1.0 / nb, yb.p, 0.0, nullptr, n, c->stream);
    kep_factorization* FB = nullptr;
    {
        kep_status st = kep_factor_pencil(c, 0.0, -1.0, &FB);            // B = 0 A - (-1) B
        if (st == KEP_ESINGULAR) return fail(c, KEP_ENOTSPD, "B is singular");
        if (st != KEP_OK) return st;
    }
    if (FB->info.n_neg != 0 || FB->info.n_zero != 0) {
        kep_factor_destroy(FB);
        return fail(c, KEP_ENOTSPD, "B is not positive definite (S:448)");
    }
    std::vector<double> al, be;
    double sig_prev = 0.0, sig = 0.0;
    int64_t nu_prev = 0, nu = 0;
    bool bracketed = false;
    for (int j = 1; j <= J1; ++j) {
        double* vj = V.p + (size_t)(j - 1) * n;
        double* uj = U.p + (size_t)(j - 1) * n;
        L.spmv(vj, w.p, nullptr);                                           // A v_j
        const double a = L.dot(vj, w.p);
        kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 1.0, w.p, -a, uj, j > 1 ? -be.back() : 0.0,
                            j > 1 ? uj - n : nullptr, n, c->stream);
        L.reorth(V.p, U.p, j, w.p);                                         // rh
        kep_status st = kep_solve_dev(FB, w.p, r.p);                         // r = B^-1 rh
        if (st != KEP_OK) { kep_factor_destroy(FB); return st; }
        const double b = std::sqrt(std::max(L.dot(w.p, r.p), 0.0));
        al.push_back(a);
        be.push_back(b);
        std::vector<double> d(al), Z;
        kep::tridiag_eigen(d, std::vector<double>(be.begin(), be.end() - 1), Z);   // Eq. (2.2)
        sig = (k <= nu_prev) ? d.front() : d.back();
        st = nu_at(sig, nu);
        if (st != KEP_OK) { kep_factor_destroy(FB); return st; }
        R.stage1_iters = j;
        if (j != 1 && ((nu < k && k <= nu_prev) || (nu_prev < k && k <= nu))) { bracketed = true; break; }
        sig_prev = sig;
        nu_prev = nu;
        if (b == 0.0) break;                                                 // invariant subspace
        kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 0.0, vj + n, 1.0 / b, r.p, 0.0, nullptr, n, c->stream);
        kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 0.0, uj + n, 1.0 / b, w.p, 0.0, nullptr, n, c->stream);
    }
    kep_factor_destroy(FB);
    if (!bracketed) return fail(c, KEP_ENOCONV, "stage 1 (Alg. 2) did not bracket lambda_k");
    double lo = std::min(sig_prev, sig), hi = std::max(sig_prev, sig);
    int64_t nlo = std::min(nu_prev, nu), nhi = std::max(nu_prev, nu);
    R.s1_lower = lo; R.s1_upper = hi; R.s1_nu_lower = nlo; R.s1_nu_upper = nhi;
    R.seconds[0] = now_s() - t0;
    // ------------------------------------------------------------ stage 2 (Alg. 1', P shifts per round)
    t0 = now_s();
    const int P = o.shifts_per_round;
    std::vector<double> sg(P);
    std::vector<int64_t> nv(P);
    std::vector<kep_status> ps(P);
    auto narrow_more = [&]() -> bool {
        if (o.bisect_only)                                                   // PAPER.md:674-676 footnote
            return (hi - lo) / std::max(std::fabs(lo), std::fabs(hi)) >= o.bisect_rtol;
        return nhi - nlo > o.m_max;                                          // Alg. 1' line 1
    };
    const int max_rounds = o.bisect_only ? std::max(o.max_bisect, 256) : o.max_bisect;
    auto trace = [&]() {                                                     // Fig. 4 / Table 5 analogue
        if (R.stage2_trace_len < 64) {
            R.stage2_trace_lower[R.stage2_trace_len] = lo;
            R.stage2_trace_upper[R.stage2_trace_len] = hi;
            R.stage2_trace_m[R.stage2_trace_len] = nhi - nlo;
            R.stage2_trace_len++;
        }
    };
    auto stalled = [&]() {
        if (R.stage2_rounds >= max_rounds ||
            (!o.bisect_only && hi - lo <= 4.0 * DBL_EPSILON * std::max(std::fabs(lo), std::fabs(hi)))) {
            R.status = o.bisect_only ? KEP_ENOCONV : KEP_ECLUSTER;
            return true;
        }
        return false;
    };
    if (o.root_finder == 1) {
        // Brent's method (zeroin) on g(sigma) = nu_sigma - k + 1/2: g < 0 at
        // the lower end, > 0 at the upper end; b is the latest iterate, [b, c] always brackets lambda_k,
        // a is the previous b.  Secant (a == c) or inverse quadratic interpolation, accepted only if it
        // falls well inside the bracket and shrinks faster than the step before last; else bisection.
        double a = lo, b = hi, c = lo;
        double fa = (double)(nlo - k) + 0.5, fb = (double)(nhi - k) + 0.5, fc = fa;
        int64_t na = nlo, nbb = nhi, nc = nlo;
        double d = b - a, e = d;
        for (;;) {
            if (std::fabs(fc) < std::fabs(fb)) {
                a = b; b = c; c = a;
                fa = fb; fb = fc; fc = fa;
                na = nbb; nbb = nc; nc = na;
            }
            lo = std::min(b, c); hi = std::max(b, c);
            nlo = b < c ? nbb : nc; nhi = b < c ? nc : nbb;
            if (R.stage2_rounds > 0) trace();
            if (!narrow_more() || stalled()) break;
            const double tol = 2.0 * DBL_EPSILON * std::fabs(b);
            const double mm = 0.5 * (c - b);
            if (std::fabs(e) >= tol && std::fabs(fa) > std::fabs(fb)) {
                double p, q;
                const double s = fb / fa;
                if (a == c) {                                                // secant
                    p = 2.0 * mm * s;
                    q = 1.0 - s;
                } else {                                                     // inverse quadratic
                    q = fa / fc;
                    const double r = fb / fc;
                    p = s * (2.0 * mm * q * (q - r) - (b - a) * (r - 1.0));
                    q = (q - 1.0) * (r - 1.0) * (s - 1.0);
                }
                if (p > 0.0) q = -q; else p = -p;
                if (2.0 * p < std::min(3.0 * mm * q - std::fabs(tol * q), std::fabs(e * q))) { e = d; d = p / q; }
                else { d = mm; e = mm; }
            } else {
                d = mm;
                e = mm;
            }
            a = b; fa = fb; na = nbb;
            b += std::fabs(d) > tol ? d : (mm > 0.0 ? tol : -tol);
            kep_status st = nu_at(b, nbb);
            if (st != KEP_OK) return st;
            fb = (double)(nbb - k) + 0.5;
            R.stage2_rounds++;
            R.stage2_shifts++;
            if ((fb > 0.0) == (fc > 0.0)) { c = a; fc = fa; nc = na; d = e = b - a; }
        }
    }
    while (o.root_finder != 1 && narrow_more()) {
        if (stalled()) break;
        for (int i = 0; i < P; ++i) sg[i] = lo + (hi - lo) * (double)(i + 1) / (double)(P + 1);
        kep_status st = kep_inertia_many(c, P, sg.data(), nv.data(), ps.data(), nullptr);
        if (st != KEP_OK) return st;
        for (int i = 0; i < P; ++i)
            if (ps[i] != KEP_OK) {                                           // perturb toward the wider side
                sg[i] += 1e-6 * (hi - lo);
                st = nu_at(sg[i], nv[i]);
                if (st != KEP_OK) return st;
            }
        R.stage2_rounds++;
        R.stage2_shifts += P;
        double l2 = lo, h2 = hi;
        int64_t nl2 = nlo, nh2 = nhi;
        for (int i = 0; i <= P; ++i) {                                       // first pair with nu_a < k <= nu_b
            const double sa = i == 0 ? lo : sg[i - 1], sb = i == P ? hi : sg[i];
            const int64_t na = i == 0 ? nlo : nv[i - 1], nbb = i == P ? nhi : nv[i];
            if (na < k && k <= nbb) { l2 = sa; h2 = sb; nl2 = na; nh2 = nbb; break; }
        }
        lo = l2; hi = h2; nlo = nl2; nhi = nh2;
        trace();
    }
    R.sigma_lower = lo; R.sigma_upper = hi; R.nu_lower = nlo; R.nu_upper = nhi;
    R.seconds[1] = now_s() - t0;
    if (R.status != KEP_OK) {
        if (rep_out) *rep_out = R;
        return KEP_OK;
    }
    if (o.bisect_only) {                                                     // lambda_k = midpoint, no stage 3
        *lambda = 0.5 * (lo + hi);
        R.eta = 0.5 * (hi - lo);
        if (rep_out) *rep_out = R;
        return KEP_OK;
    }
    // ------------------------------------------------------------ stage 3 (Alg. 3)
    t0 = now_s();
    const int64_t l = k - nlo, m = nhi - nlo;
    double sigma = 0.5 * (lo + hi);
    kep_factorization* F = nullptr;
    for (int t = 0; t < 8; ++t) {
        kep_status st = kep_factor(c, sigma, &F);
        if (st == KEP_OK) break;
        if (st != KEP_ESINGULAR) return st;
        sigma += 1e-6 * (hi - lo);
    }
    if (!F) return fail(c, KEP_ESINGULAR, "stage-3 shift stays singular");
    R.sigma_si = sigma;
    const int J3 = std::max<int>(o.max_si, (int)m);
    if ((size_t)(J3 + 1) * (size_t)m * sizeof(double) > 200 * 1024)        // k_ritz stages C (j x m) in shared memory
        return fail(c, KEP_EINVAL, "max_si * m_max too large for the Ritz-vector kernel");
    DevVec W, Vt, X, Xp, g, Cm, ta, tb;
    KEP_CUDA(c, cudaMalloc(&ta.p, sizeof(double) * n));                  // scratch of the convergence tests
    KEP_CUDA(c, cudaMalloc(&tb.p, sizeof(double) * n));
    KEP_CUDA(c, cudaMalloc(&W.p, sizeof(double) * n * (J3 + 1)));
    KEP_CUDA(c, cudaMalloc(&Vt.p, sizeof(double) * n * (J3 + 1)));
    KEP_CUDA(c, cudaMalloc(&X.p, sizeof(double) * n * m));
    KEP_CUDA(c, cudaMalloc(&Xp.p, sizeof(double) * n * m));
    KEP_CUDA(c, cudaMalloc(&g.p, sizeof(double) * 64));
    KEP_CUDA(c, cudaMalloc(&Cm.p, sizeof(double) * (size_t)(J3 + 1) * m));
    if (o.v0_stage3) h0.assign(o.v0_stage3, o.v0_stage3 + n); else seeded_uniform(o.seed + 0x5151, n, h0);
    KEP_CUDA(c, cudaMemcpyAsync(W.p, h0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    L.spmv(W.p, nullptr, yb.p);
    nb = std::sqrt(L.dot(W.p, yb.p));
    kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 1.0 / nb, W.p, 0.0, nullptr, 0.0, nullptr, n, c->stream);
    kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 0.0, Vt.p, 1.0 / nb, yb.p, 0.0, nullptr, n, c->stream);
    al.clear();
    be.clear();
    bool have_prev = false, done = false;
    double lam_k = 0.0;
    int iq_k = -1;
    std::vector<double> hres(m), hdif(m);
    for (int j = 1; j <= J3 && !done; ++j) {
        double* wj = W.p + (size_t)(j - 1) * n;
        double* vj = Vt.p + (size_t)(j - 1) * n;
        kep_status st = kep_solve_dev(F, vj, r.p);                           // z = (A - sigma B)^-1 v~_j
        if (st != KEP_OK) { kep_factor_destroy(F); return st; }
        const double a = L.dot(vj, r.p);
        kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 1.0, r.p, -a, wj, j > 1 ? -be.back() : 0.0,
                            j > 1 ? wj - n : nullptr, n, c->stream);
        L.reorth(Vt.p, W.p, j, r.p);
        L.spmv(r.p, nullptr, yb.p);                                          // u = B r
        const double b = std::sqrt(std::max(L.dot(r.p, yb.p), 0.0));
        al.push_back(a);
        be.push_back(b);
        R.stage3_iters = j;
        if (j >= m) {
            std::vector<double> th(al), Z;
            kep::tridiag_eigen(th, std::vector<double>(be.begin(), be.end() - 1), Z);   // Eq. (2.5)
            std::vector<int> ord(j);
            std::iota(ord.begin(), ord.end(), 0);
            std::stable_sort(ord.begin(), ord.end(), [&](int p1, int p2) { return std::fabs(th[p1]) > std::fabs(th[p2]); });
            std::vector<double> lam(m), eta(m), Ch((size_t)j * m), gh(m);
            for (int q = 0; q < m; ++q) {
                const int i = ord[q];
                const double yj = Z[(size_t)(j - 1) + (size_t)i * j];
                lam[q] = sigma + 1.0 / th[i];                                  // Eq. (2.6)
                const double rho = std::fabs(b * yj / th[i]);
                eta[q] = rho / std::fabs(th[i]) / std::sqrt(1.0 + rho * rho); // Eq. (3.1)
                for (int t = 0; t < j; ++t) Ch[t + (size_t)q * j] = th[i] * Z[t + (size_t)i * j];
                gh[q] = yj;                                                  // x = theta W y + r (e_j^T y)
            }
            bool inc = true, dis = true;
            for (int q = 0; q < m; ++q) inc = inc && lam[q] - eta[q] >= lo && lam[q] + eta[q] < hi;   // (3.3)
            std::vector<int> so(m);
            std::iota(so.begin(), so.end(), 0);
            std::sort(so.begin(), so.end(), [&](int p1, int p2) { return lam[p1] < lam[p2]; });
            for (int q = 0; q + 1 < m; ++q)                                                         // (3.4)
                dis = dis && lam[so[q]] + eta[so[q]] < lam[so[q + 1]] - eta[so[q + 1]];
            KEP_CUDA(c, cudaMemcpyAsync(Cm.p, Ch.data(), sizeof(double) * Ch.size(), cudaMemcpyHostToDevice, c->stream));
            KEP_CUDA(c, cudaMemcpyAsync(g.p, gh.data(), sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
            kep::launch_ritz(W.p, n, j, Cm.p, r.p, g.p, (int)m, X.p, n, n, c->stream);   // x_{i,2}, Eq. (2.7)
            KEP_CUDA(c, cudaGetLastError());
            if (inc && dis && !R.s3_iter_bound) R.s3_iter_bound = j;                // Table 6 "Bound"
            bool all_res = inc && dis, all_dif = inc && dis && have_prev;
            for (int q = 0; q < m && inc && dis; ++q) {                       // every pair: Table 6 columns
                double* xq = X.p + (size_t)q * n;
                const double xx = L.dot(xq, xq);
                L.spmv(xq, ta.p, tb.p);                                       // (A - lambda B) x
                kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 1.0, ta.p, -lam[q], tb.p, 0.0, nullptr, n, c->stream);
                hres[q] = std::sqrt(L.dot(ta.p, ta.p) / xx);
                all_res = all_res && hres[q] < o.tau_res;
                if (!have_prev) continue;
                double* xpq = Xp.p + (size_t)q * n;
                const double pp = L.dot(xpq, xpq), xp = L.dot(xq, xpq);
                const double sc = (xp < 0 ? -1.0 : 1.0) * std::sqrt(pp / xx);      // equal 2-norms, aligned signs
                kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 0.0, ta.p, sc, xq, -1.0, xpq, n, c->stream);
                hdif[q] = std::sqrt(L.dot(ta.p, ta.p) / pp);                       // Eq. (3.5)
                all_dif = all_dif && hdif[q] < o.tau_diff;
            }
            if (all_res && !R.s3_iter_residual) R.s3_iter_residual = j;
            if (all_dif && !R.s3_iter_difference) R.s3_iter_difference = j;
            const bool conv = inc && dis && have_prev && all_res && all_dif;
            KEP_CUDA(c, cudaMemcpyAsync(Xp.p, X.p, sizeof(double) * n * m, cudaMemcpyDeviceToDevice, c->stream));
            have_prev = true;
            if (conv) {
                const int q = so[l - 1];                                       // back to increasing order
                lam_k = lam[q];
                iq_k = q;
                R.eta = eta[q];
                R.rel_residual = hres[q];
                R.rel_diff = hdif[q];
                done = true;
                break;
            }
        }
        if (b == 0.0) break;
        kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 0.0, wj + n, 1.0 / b, r.p, 0.0, nullptr, n, c->stream);
        kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 0.0, vj + n, 1.0 / b, yb.p, 0.0, nullptr, n, c->stream);
    }
    kep_factor_destroy(F);
    R.seconds[2] = now_s() - t0;
    if (!done) {
        R.status = KEP_ENOCONV;
        if (rep_out) *rep_out = R;
        return KEP_OK;
    }
    *lambda = lam_k;
    if (x) {                                                                   // B-normalised eigenvector
        double* xq = X.p + (size_t)iq_k * n;
        L.spmv(xq, nullptr, yb.p);
        const double bn = std::sqrt(L.dot(xq, yb.p));
        kep::launch_combine(nullptr, 0, 0, nullptr, 0.0, 1.0 / bn, xq, 0.0, nullptr, 0.0, nullptr, n, c->stream);
        KEP_CUDA(c, cudaMemcpyAsync(x, xq, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        KEP_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    if (rep_out) *rep_out = R;
    return KEP_OK;
}

kep_status kep_get_analysis(const kep_ctx* c, kep_analysis_info* I) {
    if (!c || !I) return KEP_EINVAL;
    const Symbolic& S = c->sym;
    I->n = S.n;
    I->nnz_lower = S.nnz;
    I->n_supervariables = S.nsv;
    I->n_fronts = S.nf;
    I->n_levels = (int64_t)S.level_ptr.size() - 1;
    I->max_front = S.max_front;
    I->max_level_width = S.max_level_width;
    I->nzf = S.nzf;
    I->nzf_exec = S.nzf_exec;
    I->flops = S.flops;
    I->flops_exec = S.flops_exec;
    I->flops_schur = S.flops_schur;
    I->sum_cb = S.sum_cb;
    I->arena_bytes = S.arena_doubles * (int64_t)sizeof(double);
    I->delay_slack = S.slack;
    I->batch = c->batch_cap;
    return KEP_OK;
}

kep_status kep_get_profile(const kep_ctx* c, kep_profile* p) {
    if (!c || !p) return KEP_EINVAL;
    *p = c->prof;
    return KEP_OK;
}

kep_status kep_reset_profile(kep_ctx* c) {
    if (c) c->lvl_ms.clear();
    if (!c) return KEP_EINVAL;
    std::memset(&c->prof, 0, sizeof(c->prof));
    return KEP_OK;
}

kep_status kep_get_perm(const kep_ctx* c, int64_t* perm) {
    if (!c || !perm) return KEP_EINVAL;
    std::memcpy(perm, c->sym.perm.data(), sizeof(int64_t) * c->sym.n);
    return KEP_OK;
}

kep_status kep_get_fronts(const kep_ctx* c, int64_t* first, int64_t* parent, int64_t* forder) {
    if (!c) return KEP_EINVAL;
    const Symbolic& S = c->sym;
    for (int64_t s = 0; s < S.nf; ++s) {
        if (first) first[s] = S.piv_first[s];
        if (parent) parent[s] = S.parent[s];
        if (forder) forder[s] = S.forder[s];
    }
    if (first) first[S.nf] = S.n;
    return KEP_OK;
}

void kep_destroy(kep_ctx* c) {
    if (!c) return;
    if (getenv("KEP_PROFILE_LEVELS") && !c->lvl_ms.empty()) {
        fprintf(stderr, "[kep] per-level kernel ms (assemble fs ref schur l21 check fsu schur_tma) fronts maxf\n");
        for (size_t L = 0; L < c->lvl_ms.size(); ++L) {
            int mx = 0;
            for (int x = c->sym.level_ptr[L]; x < c->sym.level_ptr[L + 1]; ++x) mx = std::max(mx, (int)c->sym.forder[c->sym.level_fronts[x]]);
            fprintf(stderr, "[kep] L%2zu", L);
            for (int k = 0; k < KEP_K_NCLASS; ++k) fprintf(stderr, " %9.2f", c->lvl_ms[L][k]);
            fprintf(stderr, "  %6d %6d\n", c->sym.level_ptr[L + 1] - c->sym.level_ptr[L], mx);
        }
    }
    while (!c->factors.empty()) kep_factor_destroy(c->factors.back());
    if (c->have_device) {
        cudaSetDevice(c->device);
        if (c->stream) cudaStreamSynchronize(c->stream);
        free_batch(c);
        void* ptrs[] = {c->d_forder, c->d_npiv, c->d_ncb, c->d_cap, c->d_child_ptr, c->d_child_list,
                        c->d_level_fronts, c->d_arena_off, c->d_asm_ptr, c->d_asm_src, c->d_rmap_ptr,
                        c->d_asm_rc, c->d_rmap, c->d_a, c->d_b, c->d_lists, c->d_items,
                        c->d_litems, c->d_aux_off, c->d_uitems, c->d_piv_first, c->d_cb_ptr,
                        c->d_cb_rows, c->d_perm, c->d_iperm, c->d_csr_rp, c->d_csr_src, c->d_csr_ci, c->d_aitems, c->d_asm_col, c->d_stage, c->d_rr_d1, c->d_rr_d2, c->d_rr_fr, c->d_rr_x, c->d_rr_cnt, c->d_rr_l[0], c->d_rr_l[1], c->d_rr_l[2], c->d_rr_l[3], c->d_rr_u, c->d_rr_a, c->d_lsitems, c->d_lditems, c->d_lxitems, c->d_xfronts, c->d_xoff,
                        c->d_csr_a, c->d_csr_b, c->d_goff, c->d_small, c->d_f0, c->d_resid, c->d_ritems,
                        c->d_smfronts, c->d_tmaps, c->d_tmap_idx, c->d_big_groups, c->d_big_scroff, c->d_big_scr,
                        c->d_big_state, c->d_big_bars, c->d_smitems};
        for (void* p : ptrs) cudaFree(p);
        for (cudaEvent_t ev : c->ev_pool) cudaEventDestroy(ev);
        if (c->fs_fork) cudaEventDestroy(c->fs_fork);
        for (int x = 0; x < 7; ++x) {
            if (c->fs_join[x]) cudaEventDestroy(c->fs_join[x]);
            if (c->fs_streams[x]) cudaStreamDestroy(c->fs_streams[x]);
        }
        if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    }
    delete c;
}

}  // extern "C"
