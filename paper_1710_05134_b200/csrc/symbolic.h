// symbolic.h — host-side symbolic analysis (row a0 of SURVEY.md §8, untimed).
//
// Pattern-only work done once per sparsity pattern and recycled for every
// shift (§3.3 "once ordering and symbolic
// factorization are obtained ... they can be recycled").
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace kep {

struct SymbolicOptions {
    int ordering = 0;              // kep_ordering
    const int64_t* user_perm = nullptr;
    bool amalgamate = true;
    int nrelax = 16;
    double relax_frac = 0.05;
    int delay_slack = 16;
};

// Result of the analysis.  "position" = place in the elimination order.
struct Symbolic {
    int64_t n = 0, nnz = 0;
    std::vector<int64_t> perm;     // perm[pos] = dof
    std::vector<int64_t> iperm;    // iperm[dof] = pos
    int64_t nsv = 0;               // supervariables

    // fronts (supernodes after amalgamation), in postorder (children before parents)
    int64_t nf = 0;
    std::vector<int64_t> piv_first;     // [nf+1] first pivot position of each front
    std::vector<int32_t> npiv, ncb, forder, parent, level;
    std::vector<int64_t> cb_ptr;        // [nf+1] CB row positions of each front
    std::vector<int64_t> cb_rows;       // positions (ascending)
    std::vector<int32_t> child_ptr, child_list;    // children of each front, ascending
    std::vector<int32_t> level_ptr, level_fronts;  // fronts of each level, ascending
    std::vector<int32_t> level_child_ptr;          // not used by kernels; diagnostics

    // assembly map: entries grouped by front, (lrow << 16 | lcol) local indices
    std::vector<int64_t> asm_ptr;       // [nf+1]
    std::vector<int64_t> asm_src;       // [nnz] original entry index
    std::vector<uint32_t> asm_rc;       // [nnz]

    // extend-add map: CB row t of front c -> local index in parent (no delays)
    std::vector<int64_t> rmap_ptr;      // [nf+1] == cb_ptr
    std::vector<int32_t> rmap;

    // memory plan (doubles), per shift
    int32_t slack = 16;
    std::vector<int64_t> arena_off;     // [nf]
    std::vector<int32_t> capacity;      // [nf] f + slack
    int64_t arena_doubles = 0;

    // statistics
    int64_t nzf = 0, nzf_exec = 0, sum_cb = 0, max_front = 0, max_level_width = 0;
    double flops = 0, flops_exec = 0, flops_schur = 0;
};

// Returns empty string on success, else an error message.
std::string analyze(int64_t n, const int64_t* colptr, const int32_t* rowidx,
                    const SymbolicOptions& opt, Symbolic& out);

// Recompute the memory plan for a new slack.
void plan_memory(Symbolic& s, int slack);

}  // namespace kep
