// device.cuh — device-side plan, per-shift state and shared helpers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kep {

// Per-shift counters (one per shift of a batch); reset before every batch.
struct ShiftStat {
    unsigned long long n_neg, n_zero, n_pos, n_2x2, n_delayed;
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
    const int64_t* arena_off;    // doubles, within one shift's arena
    const int64_t* asm_ptr;
    const uint32_t* asm_rc;      // (lrow << 16) | lcol
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
    double u;                    // threshold pivoting parameter
};

__device__ __forceinline__ void atomic_max_pos_double(unsigned long long* addr, double v) {
    atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_min_pos_double(unsigned long long* addr, double v) {
    atomicMin(addr, (unsigned long long)__double_as_longlong(v));
}

// Launchers (kernels.cu)
void launch_assemble(const DevPlan& P, int lvl_begin, int nfronts, int batch, cudaStream_t st);
void launch_panel(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, int max_f, cudaStream_t st);
void launch_schur(const DevPlan& P, const int4* items, int nitems, int batch, cudaStream_t st);
int panel_max_front();
void launch_factor_list(const DevPlan& P, const int32_t* fronts, int nfronts, int batch, cudaStream_t st);
void launch_gather(const double* src, const int64_t* idx, double* dst, int64_t n, cudaStream_t st);
void launch_reset_stats(ShiftStat* st, int batch, cudaStream_t s);

}  // namespace kep
