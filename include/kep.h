/*
 * kep.h — C ABI of the B200-native nu_sigma(A, B) engine (arXiv 1710.05134).
 *
 * What it computes
 * ----------------
 * nu_sigma(A, B) = #{ i : lambda_i < sigma } for the symmetric-definite pencil
 * A x = lambda B x (Eq. 1.1; PAPER.md:45 definition of nu), via
 * a sparse symmetric-indefinite factorisation
 *     L D L^T = P Q (A - sigma B) Q^T P^T          (Alg. 1' line 3)
 * and Sylvester's law of inertia, nu = nu_0(D, I).
 * Q is a fill-reducing ordering computed once per sparsity pattern and recycled
 * for every shift (§3.3); P is the Bunch-Kaufman stability
 * permutation, chosen per shift inside each front with delayed
 * pivots (reading R1).  D has 1x1 and 2x2 blocks; a 2x2 block is
 * classified by the sign of its determinant (reading R2).
 *
 * Conventions (all entry points)
 * ------------------------------
 * - Real fp64 values, 0-based indices.  Matrices are given as the LOWER
 *   triangle (row >= col) in compressed sparse column form of the UNION
 *   pattern of A and B: colptr[n+1] (int64), rowidx
 *   (int32, sorted within each column, diagonal present).  A and B value
 *   arrays are aligned with rowidx; explicit zeros are allowed.
 * - Ownership: every pointer argument is owned by the caller and may be freed
 *   when the call returns; the library copies what it needs.  A kep_ctx owns
 *   all device memory it allocates; kep_destroy releases it.
 * - Errors: every function returns a kep_status and never aborts or throws
 *   across the ABI.  Outputs are written only on KEP_OK, except that
 *   kep_inertia fills `info` also on KEP_ESINGULAR.  kep_last_error gives a
 *   human-readable message for the last failing call on a context.
 * - Threading: one ctx = one CUDA device + one stream; calls on one ctx must be
 *   serialised by the caller; distinct ctxs may be used concurrently.
 * - Host pointers unless the name says `_dev`.
 */
#ifndef KEP_H
#define KEP_H

#include <stdint.h>
#include <stddef.h>

#if defined(__GNUC__)
#define KEP_API __attribute__((visibility("default")))
#else
#define KEP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KEP_OK = 0,
    KEP_EINVAL = 1,       /* bad argument (null pointer, n < 0, unsorted / upper entries, ...) */
    KEP_EPATTERN = 2,     /* values do not match the analysed pattern */
    KEP_ESINGULAR = 3,    /* some |pivot| <= tau_sing * max|A - sigma B|: sigma is
                             (numerically) an eigenvalue; perturb sigma and retry */
    KEP_ENOTSPD = 4,      /* B failed an all-positive-pivot check (kep_kth_eigenpair) */
    KEP_ENOMEM = 5,       /* host or device allocation failed */
    KEP_ECUDA = 6,        /* a CUDA runtime error (message in kep_last_error) */
    KEP_EBREAKDOWN = 7,   /* Lanczos breakdown (reserved; kep_kth_eigenpair restarts instead) */
    KEP_ENOCONV = 8,      /* stage 1 did not bracket lambda_k (kep_kth_eigenpair return), or, as a report
                             status, stage 3 did not converge within max_si */
    KEP_ECLUSTER = 9,     /* report status, not an error: stage 2 stopped on a cluster of
                             > m_max eigenvalues in a 4-ulp interval */
    KEP_ENODEVICE = 10    /* no usable CUDA device */
} kep_status;

typedef enum {
    KEP_ORDER_AUTO = 0,     /* METIS nested dissection (default) */
    KEP_ORDER_METIS = 1,    /* METIS_NodeND on the supervariable quotient graph */
    KEP_ORDER_NATURAL = 2,  /* identity (testing) */
    KEP_ORDER_USER = 3      /* caller-supplied permutation `user_perm` */
} kep_ordering;

typedef struct {
    kep_ordering ordering;      /* default KEP_ORDER_AUTO */
    const int64_t* user_perm;   /* KEP_ORDER_USER: user_perm[i] = dof placed i-th; length n */
    int32_t amalgamate;         /* relaxed supernode amalgamation on (1, default) / off (0) */
    int32_t nrelax;             /* merge child into parent if merged pivot count <= nrelax (default 48) */
    double relax_frac;          /* ... or if the added zeros are <= relax_frac of the merged L (default 0.05) */
    double pivot_u;             /* threshold for delayed pivots, u in (0, 0.5]; default 0.01 (DESIGN R1) */
    double tau_sing;            /* singularity tolerance relative to max|A - sigma B|; default 1e-14 */
    int32_t delay_slack;        /* initial per-front slack (columns) for delayed pivots; default 16 */
    int32_t max_batch;          /* max shifts factorised concurrently on the device; default 16 */
    int32_t device;             /* CUDA device ordinal; -1 = current (default) */
    void* stream;               /* cudaStream_t to run on; NULL = a stream owned by the ctx */
    int32_t kernel_variant;     /* 0 = default (fastest), 1 = reference unblocked kernels (testing) */
    int32_t profile;            /* 1 = time every kernel class with CUDA events on the ctx stream */
} kep_opts;

/* Kernel classes for kep_profile (rows of SURVEY.md §8(a)). */
enum { KEP_K_ASSEMBLE = 0,   /* a1 + a2: assembly + extend-add */
       KEP_K_PANEL = 1,      /* a3: blocked Bunch-Kaufman on the FS x FS block (k_fs) */
       KEP_K_REF = 2,        /* a3 + a4 + a5: reference unblocked front factorisation (variant 1, fronts
                                too large for the fast path, fronts that failed the full-column test) */
       KEP_K_SCHUR = 3,      /* a4: DMMA contribution-block update */
       KEP_K_L21 = 4,        /* a3: CB rows of the FS columns, G21 = W21 D^-1 M, W21 = A21 P^T L11^-T
                                (k_l21x_prep, k_l21) */
       KEP_K_CHECK = 5,      /* a3 + a5: full-column threshold tests, inertia, rerun lists, re-assembly of
                                fronts that failed them */
       KEP_K_FSU = 6,        /* a3: FS x FS trailing update after each pivot block (k_fsu) */
       KEP_K_SCHUR_TMA = 7,  /* a4 on the long-K levels: the TMA-fed k_schur_tma (+ k_schur_small) */
       KEP_K_NCLASS = 8 };

typedef struct {
    double ms[KEP_K_NCLASS];          /* summed CUDA-event time per class (profile = 1 only) */
    int64_t launches[KEP_K_NCLASS];   /* kernel launches per class (always counted) */
    double schur_flops;               /* algorithmic a4 flops p c (c + 1) summed over the fronts
                                         whose Schur update ran in KEP_K_SCHUR or KEP_K_SCHUR_TMA launches */
    double schur_tma_flops;           /* the part of schur_flops in KEP_K_SCHUR_TMA launches */
    double factor_flops;              /* algorithmic flops of all factorisations run (kep_analysis_info.flops each) */
    int64_t shifts;                   /* shifts factorised */
    int64_t other_launches;           /* bookkeeping kernels (stat reset) */
} kep_profile;

typedef struct {
    int64_t n_neg, n_zero, n_pos;   /* inertia of D; nu = n_neg */
    int64_t n_2x2;                  /* number of 2x2 pivot blocks */
    int64_t n_delayed;              /* columns delayed to a parent front (sum over fronts) */
    double min_abs_pivot;           /* min over blocks of the smallest |eigenvalue| */
    double max_abs_entry;           /* max |a_ij - sigma b_ij| */
    int64_t n_redo;                 /* fronts whose full-column threshold test failed on the fast
                                       path and were refactorised by the unblocked kernel */
} kep_inertia_info;

typedef struct {
    int64_t n;                  /* matrix order */
    int64_t nnz_lower;          /* stored lower entries of the union pattern */
    int64_t n_supervariables;   /* dof groups with identical structure (atoms) */
    int64_t n_fronts;           /* supernodes after amalgamation */
    int64_t n_levels;           /* elimination-tree levels (leaves = 0) */
    int64_t max_front;          /* largest front order f (no delays) */
    int64_t max_level_width;    /* largest number of fronts in one level */
    int64_t nzf;                /* entries of L (incl. diagonal) on fundamental supernodes (#nzf) */
    int64_t nzf_exec;           /* entries of L on the amalgamated fronts */
    double flops;               /* algorithmic factor flops per shift, fundamental supernodes, no delays */
    double flops_exec;          /* flops executed on the amalgamated fronts (no delays) */
    double flops_schur;         /* part of flops_exec in the contribution-block update (row a4) */
    int64_t sum_cb;             /* sum over fronts of lower CB entries c(c+1)/2 */
    int64_t arena_bytes;        /* device front arena per shift */
    int32_t delay_slack;        /* current per-front slack */
    int32_t batch;              /* shifts factorised concurrently */
} kep_analysis_info;

typedef struct kep_ctx kep_ctx;

/* Fill `opts` with the defaults listed above. */
KEP_API void kep_default_opts(kep_opts* opts);

/* Symbolic analysis of the union pattern (untimed setup, once per pattern;
 * PAPER.md:61, :400-403).  Validates the lower CSC, groups
 * identical-structure dofs into supervariables, orders the quotient graph with
 * nested dissection, builds the elimination tree, supernodes, front structures,
 * assembly and extend-add maps and the level schedule, and copies the static
 * maps to the device.  opts may be NULL (defaults).
 * Errors: KEP_EINVAL (malformed CSC, n <= 0, entry above the diagonal,
 * missing diagonal, front larger than 65535), KEP_ENOMEM, KEP_ECUDA,
 * KEP_ENODEVICE. */
KEP_API kep_status kep_analyze(int64_t n, const int64_t* colptr, const int32_t* rowidx,
                       const kep_opts* opts, kep_ctx** out);

/* Values of A and B aligned with the analysed rowidx (nnz_lower each, host).
 * Copied to the device in assembly order.  Must precede kep_inertia.  The
 * pattern is recycled: new values (another pencil on the same pattern, e.g.
 * the shifted pencils of PAPER.md:398-403 §3.3 "reuse the ordering and the
 * symbolic factorization") need no new analysis (SPEC.md:50-58 shifted_combine
 * on the union pattern).  Errors: KEP_EINVAL, KEP_ENODEVICE, KEP_ECUDA. */
KEP_API kep_status kep_set_values(kep_ctx* ctx, const double* a, const double* b);

/* Same, from device pointers (nnz_lower doubles each, on the ctx device). */
KEP_API kep_status kep_set_values_dev(kep_ctx* ctx, const double* a_dev, const double* b_dev);

/* nu_sigma(A, B) for one shift (the timed hot path: assembly, extend-add,
 * Bunch-Kaufman partial LDL^T with delayed pivots, Schur update, inertia).
 * Returns KEP_OK and *nu, or KEP_ESINGULAR (info filled, *nu untouched).
 * info may be NULL. */
KEP_API kep_status kep_inertia(kep_ctx* ctx, double sigma, int64_t* nu, kep_inertia_info* info);

/* nu for m shifts (batched on the device, max_batch at a time): the m
 * evaluations of one multisection round, i.e. Alg. 1' line 3-4 (PAPER.md:
 * 419-420) at P shifts at once (reading R12).
 * sigmas[m], nus[m], per_shift[m] host arrays.  nus[i] is written when
 * per_shift[i] == KEP_OK.  infos may be NULL.  Returns KEP_OK if the call ran
 * (individual shifts may be KEP_ESINGULAR), else the error. */
KEP_API kep_status kep_inertia_many(kep_ctx* ctx, int32_t m, const double* sigmas, int64_t* nus,
                            kep_status* per_shift, kep_inertia_info* infos);

/* ---------------------------------------------------------------------------
 * Retained factors and solves (SURVEY.md §8(f) row f1
 * "the same factors serve the shift-and-invert Lanczos solves of stage 3").
 * ------------------------------------------------------------------------- */
typedef struct kep_factorization kep_factorization;

typedef struct {
    double sigma;                   /* the shift factorised */
    int64_t nu;                     /* nu_sigma = n_neg of D */
    kep_inertia_info inertia;
    int64_t n;                      /* matrix order */
    int64_t nnz_L;                  /* stored strictly-lower entries of L (structural) */
    int64_t store_bytes;            /* device memory held by the factor */
} kep_factor_stats;

/* Factorise A - sigma B once and keep L, D and the permutation on the device:
 *     P (A - sigma B) P^T = L D L^T,
 * P = fill-reducing ordering composed with the Bunch-Kaufman / delayed-pivot
 * permutation (the same kernels as kep_inertia).  The factor is owned by the
 * caller, must not outlive ctx and is immutable (shareable for solves).
 * Errors: KEP_ESINGULAR (some |pivot| <= tau_sing max|A - sigma B|; no factor
 * is returned), KEP_ENOMEM, KEP_ECUDA, KEP_EINVAL (values not set). */
KEP_API kep_status kep_factor(kep_ctx* ctx, double sigma, kep_factorization** out);

/* Same for alpha A - sigma B (e.g. alpha = 0, sigma = -1 factorises B for the
 * B-solves of stage 1's generalized Lanczos). */
KEP_API kep_status kep_factor_pencil(kep_ctx* ctx, double alpha, double sigma, kep_factorization** out);

/* Front-local bound of the factor residual at sigma (SURVEY.md §8(c) item 13,
 * the P8 pin of the BASELINE north_star at sizes where the dense residual
 * cannot be formed).  Factorises A - sigma B exactly as kep_factor does and,
 * per front s, evaluates E_s = P_s F_s P_s^T - L_s D_s L_s^T - (0 (+) T_s)
 * (F_s the assembled front, T_s the trailing block its parent extend-adds);
 * these telescope over the assembly tree, so
 *     || P (A - sigma B) P^T - L D L^T ||_F <= *bound = sum_s ||E_s||_F.
 * *max_front (nullable) = max_s ||E_s||_F.  Diagnostics only: needs one extra
 * front arena of device memory; no factor is kept.  Errors: as kep_factor
 * (KEP_ESINGULAR is not raised: the bound is reported at any shift). */
KEP_API kep_status kep_factor_residual(kep_ctx* ctx, double sigma, double* bound, double* max_front);

/* Factor statistics (shift, nu, inertia, size of L). */
KEP_API kep_status kep_factor_info(const kep_factorization* f, kep_factor_stats* out);

/* x = (A - sigma B)^-1 b for nrhs right-hand sides (host, column-major,
 * leading dimensions ldb, ldx >= n; x may alias b).  Multifrontal forward
 * elimination, D^-1, back substitution: the shift-and-invert solves of Alg. 3
 * (Eq. 2.4 at PAPER.md:146-151) and the B-solves of Alg. 2
 * with the retained factor (SPEC.md:140-148 solve).
 * Errors: KEP_EINVAL (bad sizes or a front beyond the solve kernels). */
KEP_API kep_status kep_solve(const kep_factorization* f, int32_t nrhs, const double* b, int64_t ldb, double* x, int64_t ldx);

/* Same for one right-hand side in device memory (n doubles each, dof order,
 * may alias), enqueued on the ctx stream (not synchronised). */
KEP_API kep_status kep_solve_dev(const kep_factorization* f, const double* b_dev, double* x_dev);

/* Copy the factor to the host (testing, residual checks): perm[k] = dof
 * eliminated k-th; d[k] = D[k,k]; dsub[k] = D[k+1,k] (nonzero only for the
 * first column of a 2x2 block); L strictly lower in CSC (elimination order,
 * unit diagonal implied, rows sorted): Lcolptr[n+1], Lrowidx/Lval[nnz_L].
 * Lrowidx and Lval may be NULL to obtain Lcolptr (sizes) only. */
KEP_API kep_status kep_factor_export(const kep_factorization* f, int64_t* perm, double* d, double* dsub,
                                     int64_t* Lcolptr, int32_t* Lrowidx, double* Lval);

/* Release a factor.  kep_destroy(ctx) releases the factors still alive on ctx. */
KEP_API void kep_factor_destroy(kep_factorization* f);

/* ---------------------------------------------------------------------------
 * The three-stage k-th eigenpair method (Alg. 4; SURVEY.md
 * §8(f) rows f2, f3).
 * ------------------------------------------------------------------------- */
typedef struct {
    int32_t m_max;              /* stage 2 stops when nu_u - nu_l <= m_max (default 20); <= 32 */
    double tau_res;             /* relative residual 2-norm tolerance, test (3.3)-(3.5) line (default 1e-10) */
    double tau_diff;            /* relative difference 2-norm tolerance, Eq. (3.5) (default 1e-10) */
    int32_t max_lanczos;        /* stage-1 Lanczos steps cap (default 64) */
    int32_t max_bisect;         /* stage-2 rounds cap (default 128) */
    int32_t max_si;             /* stage-3 SI Lanczos steps cap (default 500) */
    int32_t shifts_per_round;   /* stage-2 multisection width P (1 = Alg. 1', default 1) */
    uint64_t seed;              /* seed of the start vectors (splitmix64, uniform(-1,1)) when v0s are NULL */
    const double* v0_stage1;    /* optional start vector of stage 1 (n, host) */
    const double* v0_stage3;    /* optional start vector of stage 3 (n, host) */
    int32_t bisect_only;        /* 1: "straightforward bisection":
                                   stage 2 stops when (sigma_u - sigma_l) / max(|sigma_l|, |sigma_u|) <
                                   bisect_rtol, lambda = the midpoint, no stage 3, x not written */
    double bisect_rtol;         /* default 1e-14 */
    int32_t root_finder;        /* stage 2: 0 = bisection / multisection (Alg. 1', default); 1 = Brent's method
                                   (zeroin: secant / inverse quadratic interpolation safeguarded by bisection)
                                   on g(sigma) = nu_sigma - k + 1/2, the derivative-free bracketing root finder
                                   of PAPER.md:110-115, :740-743 (one shift per iteration) */
} kep_kth_opts;

typedef struct {
    double s1_lower, s1_upper;          /* stage-1 interval [sigma_l, sigma_u) (Alg. 2) */
    int64_t s1_nu_lower, s1_nu_upper;
    double sigma_lower, sigma_upper;    /* stage-2 interval, nu_u - nu_l <= m_max */
    int64_t nu_lower, nu_upper;
    double sigma_si;                    /* stage-3 shift (interval midpoint) */
    int32_t stage1_iters, stage2_rounds, stage2_shifts, stage3_iters;
    double eta;                         /* error bound Eq. (3.1) of lambda_k */
    double rel_residual;                /* ||(A - lambda B) x||_2 / ||x||_2 */
    double rel_diff;                    /* Eq. (3.5) at the last step */
    double seconds[3];                  /* wall time per stage */
    kep_status status;                  /* KEP_OK, KEP_ECLUSTER (cluster suspected), KEP_ENOCONV */
    /* Table 6 analogue: first SI Lanczos iteration at which (3.3) and (3.4) held for
       all m pairs ("Bound"), at which every relative residual was < tau_res ("Residual"), and every
       relative difference (3.5) < tau_diff ("Difference"); 0 = never */
    int32_t s3_iter_bound, s3_iter_residual, s3_iter_difference;
    /* Fig. 4 / Table 5 analogue: the bracket after each stage-2 iteration (first 64) */
    int32_t stage2_trace_len;
    double stage2_trace_lower[64], stage2_trace_upper[64];
    int64_t stage2_trace_m[64];         /* eigenvalues in the bracket, nu_u - nu_l */
} kep_kth_report;

KEP_API void kep_default_kth_opts(kep_kth_opts* o);

/* lambda_k (1-based k, k-th smallest) and optionally its eigenvector x (n,
 * host; B-normalised) of A x = lambda B x with the index validated: stage 1
 * (Alg. 2) brackets lambda_k with Ritz values, stage 2 (Alg. 1') narrows the
 * bracket with nu_sigma until it holds <= m_max eigenvalues, stage 3 (Alg. 3)
 * runs SI Lanczos at its midpoint until the m error bounds (3.1) are inside the
 * interval and disjoint and every pair meets tau_res and tau_diff; lambda_k is
 * the (k - nu_l)-th of them.  Returns KEP_OK (report->status may be
 * KEP_ECLUSTER or KEP_ENOCONV: lambda not written), or an error.  report may
 * be NULL. */
KEP_API kep_status kep_kth_eigenpair(kep_ctx* ctx, int64_t k, const kep_kth_opts* opts, double* lambda, double* x,
                                     kep_kth_report* report);

/* Testing hook: the host tridiagonal eigensolver of the Lanczos stages (Eq. (2.2),
 * PAPER.md:129-134; Eq. (2.5)): T = tridiag(e, d, e) of order n
 * (d[n], e[n-1]) = Z diag(w) Z^T, w ascending, Z column-major n x n (caller-owned).
 * Implicit symmetric QR with the Wilkinson shift.  Errors: KEP_EINVAL, KEP_ENOCONV. */
KEP_API kep_status kep_tridiag_eigen(int32_t n, const double* d, const double* e, double* w, double* Z);

/* Analysis statistics (sizes, #nzf, flops per shift, memory). */
KEP_API kep_status kep_get_analysis(const kep_ctx* ctx, kep_analysis_info* info);

/* Accumulated kernel statistics since the last reset (see kep_opts.profile). */
KEP_API kep_status kep_get_profile(const kep_ctx* ctx, kep_profile* prof);
KEP_API kep_status kep_reset_profile(kep_ctx* ctx);

/* The fill-reducing permutation chosen: perm[i] = dof placed i-th (length n). */
KEP_API kep_status kep_get_perm(const kep_ctx* ctx, int64_t* perm);

/* Supernode partition and assembly tree (testing / diagnostics):
 * first[s] .. first[s+1]-1 are the pivot positions of front s (n_fronts+1
 * entries), parent[s] = parent front or -1, front_order[s] = f_s. */
KEP_API kep_status kep_get_fronts(const kep_ctx* ctx, int64_t* first, int64_t* parent, int64_t* front_order);

KEP_API void kep_destroy(kep_ctx* ctx);
KEP_API const char* kep_status_string(kep_status s);
KEP_API const char* kep_last_error(const kep_ctx* ctx);
/* Library version string, e.g. "kep 0.1 sm_100a". */
KEP_API const char* kep_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KEP_H */
