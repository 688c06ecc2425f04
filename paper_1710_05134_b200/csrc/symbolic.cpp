// symbolic.cpp — host symbolic analysis (untimed).
//
// Steps (SURVEY.md §3 call stack 1):
//   1. validate the lower CSC of pattern(A) U pattern(B)
//   2. group dofs with identical closed adjacency into supervariables (atoms,
//      o orbitals per atom share one pattern)
//   3. fill-reducing nested dissection of the quotient graph with METIS
//      ("METIS"; ordering Q of Alg. 1' line 3)
//   4. elimination tree (Liu), postorder, column counts (row subtrees)
//   5. fundamental supernodes + relaxed amalgamation
//   6. front row structures, extend-add relative maps, assembly maps
//   7. level schedule (leaves = level 0) and the per-shift front memory plan
// Everything here depends on the pattern only and is recycled for every shift
// (PAPER.md:400-403).
#include "symbolic.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <string>

extern "C" int METIS_SetDefaultOptions(int64_t* options);
extern "C" int METIS_NodeND(int64_t* nvtxs, int64_t* xadj, int64_t* adjncy, int64_t* vwgt,
                            int64_t* options, int64_t* perm, int64_t* iperm);

namespace kep {

namespace {

const int kOrderAuto = 0, kOrderMetis = 1, kOrderNatural = 2, kOrderUser = 3;

std::string fmt(const char* what, int64_t a, int64_t b = -1) {
    std::string s(what);
    s += " (" + std::to_string(a);
    if (b >= 0) s += ", " + std::to_string(b);
    return s + ")";
}

}  // namespace

void plan_memory(Symbolic& S, int slack) {
    S.slack = slack;
    const int64_t nf = S.nf;
    S.capacity.assign(nf, 0);
    S.arena_off.assign(nf, 0);
    std::vector<int64_t> need(nf), align(nf);
    for (int64_t s = 0; s < nf; ++s) {
        int64_t cap = (int64_t)S.forder[s] + slack;
        S.capacity[s] = (int32_t)cap;
        const int64_t ldc = (cap + 1) & ~int64_t(1);  // fronts use an even leading dimension ldpad(capacity)
        need[s] = ldc * cap;
        // a front starts at a multiple of its leading dimension, so one 2-D TMA tensor map per distinct
        // leading dimension (rows of ld doubles over the whole arena) addresses every front with it
        align[s] = ldc;
    }
    std::map<int64_t, int64_t> freel;                 // offset -> size
    int64_t top = 0;
    auto alloc = [&](int64_t sz, int64_t al) -> int64_t {
        for (auto it = freel.begin(); it != freel.end(); ++it) {
            const int64_t off = it->first, end = it->first + it->second;
            const int64_t a = (off + al - 1) / al * al;
            if (a + sz <= end) {
                freel.erase(it);
                if (a > off) freel[off] = a - off;
                if (end > a + sz) freel[a + sz] = end - (a + sz);
                return a;
            }
        }
        const int64_t a = (top + al - 1) / al * al;
        if (a > top) freel[top] = a - top;            // alignment gap: reusable
        top = a + sz;
        return a;
    };
    auto release = [&](int64_t off, int64_t sz) {
        auto it = freel.emplace(off, sz).first;
        auto nx = std::next(it);
        if (nx != freel.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            freel.erase(nx);
        }
        if (it != freel.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                freel.erase(it);
                it = pv;
            }
        }
        if (it->first + it->second == top) {          // shrink the top
            top = it->first;
            freel.erase(it);
        }
    };
    int64_t peak = 0;
    const int64_t nl = (int64_t)S.level_ptr.size() - 1;
    for (int64_t L = 0; L < nl; ++L) {
        for (int32_t k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) {
            int32_t s = S.level_fronts[k];
            S.arena_off[s] = alloc(need[s], align[s]);
        }
        peak = std::max(peak, top);
        for (int32_t k = S.level_ptr[L]; k < S.level_ptr[L + 1]; ++k) {
            int32_t s = S.level_fronts[k];
            for (int32_t q = S.child_ptr[s]; q < S.child_ptr[s + 1]; ++q) {
                int32_t c = S.child_list[q];
                release(S.arena_off[c], need[c]);
            }
        }
    }
    S.arena_doubles = std::max<int64_t>(peak, 32);
}

std::string analyze(int64_t n, const int64_t* colptr, const int32_t* rowidx,
                    const SymbolicOptions& opt, Symbolic& S) {
    // ------------------------------------------------------------ 1. validate
    if (n <= 0) return "n must be positive";
    if (!colptr || !rowidx) return "null colptr/rowidx";
    if (colptr[0] != 0) return "colptr[0] must be 0";
    for (int64_t j = 0; j < n; ++j) {
        int64_t b = colptr[j], e = colptr[j + 1];
        if (e <= b) return fmt("column without a diagonal entry", j);
        if (rowidx[b] != j) return fmt("first entry of a column must be its diagonal (lower CSC)", j, rowidx[b]);
        for (int64_t q = b + 1; q < e; ++q) {
            if (rowidx[q] <= rowidx[q - 1]) return fmt("row indices must be strictly increasing in a column", j);
            if (rowidx[q] >= n) return fmt("row index out of range", j, rowidx[q]);
        }
    }
    const int64_t nnz = colptr[n];
    S = Symbolic();
    S.n = n;
    S.nnz = nnz;

    // ------------------------------------------------------------ 2. full adjacency (no diagonal)
    std::vector<int64_t> xadj(n + 1, 0);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t q = colptr[j] + 1; q < colptr[j + 1]; ++q) {
            xadj[rowidx[q] + 1]++;
            xadj[j + 1]++;
        }
    for (int64_t i = 0; i < n; ++i) xadj[i + 1] += xadj[i];
    std::vector<int32_t> adj(xadj[n]);
    {
        std::vector<int64_t> nx(xadj.begin(), xadj.end() - 1);
        for (int64_t j = 0; j < n; ++j)
            for (int64_t q = colptr[j] + 1; q < colptr[j + 1]; ++q) {
                int32_t i = rowidx[q];
                adj[nx[j]++] = i;
                adj[nx[i]++] = (int32_t)j;
            }
    }   // each adjacency list is ascending

    // ------------------------------------------------------------ 3. supervariables
    std::vector<int64_t> sv_first;           // original dof of each sv start
    std::vector<int32_t> sv_of(n);
    sv_first.push_back(0);
    sv_of[0] = 0;
    for (int64_t i = 1; i < n; ++i) {
        bool same = false;
        int64_t da = xadj[i] - xadj[i - 1], db = xadj[i + 1] - xadj[i];
        if (da == db && da > 0) {
            // closed neighbourhoods N[i-1] == N[i]  <=>  adj(i-1)\{i} == adj(i)\{i-1}, both contain each other
            const int32_t* A = &adj[xadj[i - 1]];
            const int32_t* B = &adj[xadj[i]];
            int64_t p = 0, q = 0;
            bool has_i = false, has_im1 = false;
            same = true;
            while (p < da || q < db) {
                if (p < da && A[p] == i) { has_i = true; ++p; continue; }
                if (q < db && B[q] == i - 1) { has_im1 = true; ++q; continue; }
                if (p >= da || q >= db || A[p] != B[q]) { same = false; break; }
                ++p; ++q;
            }
            same = same && has_i && has_im1;
        }
        if (!same) sv_first.push_back(i);
        sv_of[i] = (int32_t)(sv_first.size() - 1);
    }
    const int64_t nsv = (int64_t)sv_first.size();
    sv_first.push_back(n);
    S.nsv = nsv;
    std::vector<int64_t> svsize(nsv);
    for (int64_t s = 0; s < nsv; ++s) svsize[s] = sv_first[s + 1] - sv_first[s];

    // quotient graph
    std::vector<int64_t> qx(nsv + 1, 0), qa;
    qa.reserve(xadj[n] / 4 + 16);
    for (int64_t s = 0; s < nsv; ++s) {
        int64_t d = sv_first[s];
        int64_t last = -1;
        for (int64_t q = xadj[d]; q < xadj[d + 1]; ++q) {
            int64_t t = sv_of[adj[q]];
            if (t != s && t != last) { qa.push_back(t); last = t; }
        }
        qx[s + 1] = (int64_t)qa.size();
    }
    std::vector<int32_t>().swap(adj);
    std::vector<int64_t>().swap(xadj);

    // ------------------------------------------------------------ 4. ordering (new -> old sv)
    std::vector<int64_t> svperm(nsv);
    std::iota(svperm.begin(), svperm.end(), 0);
    int ord = opt.ordering == kOrderAuto ? kOrderMetis : opt.ordering;
    if (ord == kOrderUser) {
        if (!opt.user_perm) return "KEP_ORDER_USER needs user_perm";
        std::vector<char> seen(nsv, 0), dseen(n, 0);
        int64_t k = 0;
        for (int64_t i = 0; i < n; ++i) {
            int64_t d = opt.user_perm[i];
            if (d < 0 || d >= n || dseen[d]) return "user_perm is not a permutation";
            dseen[d] = 1;
            int32_t s = sv_of[d];
            if (!seen[s]) { seen[s] = 1; svperm[k++] = s; }
        }
    } else if (ord == kOrderMetis) {
        if (nsv >= 3 && qx[nsv] > 0) {
            int64_t opts[40];
            METIS_SetDefaultOptions(opts);
            int64_t nv = nsv;
            std::vector<int64_t> iperm(nsv);
            std::vector<int64_t> vw(svsize);
            int rc = METIS_NodeND(&nv, qx.data(), qa.data(), vw.data(), opts, svperm.data(), iperm.data());
            if (rc != 1) return fmt("METIS_NodeND failed", rc);
        }
    } else if (ord != kOrderNatural) {
        return "unknown ordering";
    }
    std::vector<int64_t> spos(nsv);
    for (int64_t k = 0; k < nsv; ++k) spos[svperm[k]] = k;

    // ------------------------------------------------------------ 5. etree (Liu) + postorder
    std::vector<int64_t> par(nsv, -1), anc(nsv, -1);
    for (int64_t k = 0; k < nsv; ++k) {
        int64_t old = svperm[k];
        for (int64_t q = qx[old]; q < qx[old + 1]; ++q) {
            int64_t j = spos[qa[q]];
            if (j >= k) continue;
            int64_t r = j;
            while (anc[r] != -1 && anc[r] != k) {
                int64_t nx = anc[r];
                anc[r] = k;
                r = nx;
            }
            if (anc[r] == -1) { anc[r] = k; par[r] = k; }
        }
    }
    std::vector<int64_t> head(nsv, -1), nxt(nsv, -1), post(nsv);
    for (int64_t k = nsv - 1; k >= 0; --k)
        if (par[k] >= 0) { nxt[k] = head[par[k]]; head[par[k]] = k; }
    {
        int64_t cnt = 0;
        std::vector<int64_t> stack;
        for (int64_t r = 0; r < nsv; ++r) {
            if (par[r] != -1) continue;
            stack.push_back(r);
            while (!stack.empty()) {
                int64_t v = stack.back();
                if (head[v] != -1) {            // descend into first unvisited child
                    int64_t c = head[v];
                    head[v] = nxt[c];
                    stack.push_back(c);
                } else {
                    post[v] = cnt++;
                    stack.pop_back();
                }
            }
        }
    }
    {   // relabel by postorder
        std::vector<int64_t> sp2(nsv), par2(nsv, -1);
        for (int64_t k = 0; k < nsv; ++k) {
            sp2[post[k]] = svperm[k];
            par2[post[k]] = par[k] >= 0 ? post[par[k]] : -1;
        }
        svperm.swap(sp2);
        par.swap(par2);
        for (int64_t k = 0; k < nsv; ++k) spos[svperm[k]] = k;
    }
    // quotient adjacency in new numbering
    std::vector<int64_t> nx_(nsv + 1, 0), na_(qa.size());
    for (int64_t k = 0; k < nsv; ++k) nx_[k + 1] = nx_[k] + (qx[svperm[k] + 1] - qx[svperm[k]]);
    for (int64_t k = 0; k < nsv; ++k) {
        int64_t old = svperm[k], w = nx_[k];
        for (int64_t q = qx[old]; q < qx[old + 1]; ++q) na_[w++] = spos[qa[q]];
        std::sort(na_.begin() + nx_[k], na_.begin() + nx_[k + 1]);
    }
    std::vector<int64_t>().swap(qa);
    std::vector<int64_t> wsz(nsv);
    for (int64_t k = 0; k < nsv; ++k) wsz[k] = svsize[svperm[k]];

    // ------------------------------------------------------------ 6. column counts (row subtrees)
    std::vector<int64_t> cnt(nsv, 0), wcnt(nsv, 0), mark(nsv, -1);
    for (int64_t i = 0; i < nsv; ++i) {
        mark[i] = i;
        for (int64_t q = nx_[i]; q < nx_[i + 1]; ++q) {
            int64_t k = na_[q];
            if (k >= i) break;
            while (mark[k] != i) {
                mark[k] = i;
                cnt[k]++;
                wcnt[k] += wsz[i];
                k = par[k];
            }
        }
    }
    // algorithmic nzf / flops on fundamental supernodes (no padding, no delays)
    {
        double fl = 0;
        int64_t nzf = 0;
        for (int64_t k = 0; k < nsv; ++k) {
            int64_t w = wsz[k], W = wcnt[k];
            nzf += w * W + w * (w + 1) / 2;
            for (int64_t t = 0; t < w; ++t) {
                double m = (double)(W + w - 1 - t);
                fl += m * m + 2.0 * m;
            }
        }
        S.nzf = nzf;
        S.flops = fl;
    }

    // ------------------------------------------------------------ 7. supernodes + amalgamation
    std::vector<int64_t> nchild(nsv, 0);
    for (int64_t k = 0; k < nsv; ++k)
        if (par[k] >= 0) nchild[par[k]]++;
    std::vector<int64_t> sn_first, sn_last;
    for (int64_t k = 0; k < nsv; ++k) {
        bool join = k > 0 && par[k - 1] == k && nchild[k] == 1 && cnt[k - 1] == cnt[k] + 1;
        if (!join) sn_first.push_back(k);
    }
    int64_t nsn = (int64_t)sn_first.size();
    sn_last.resize(nsn);
    for (int64_t s = 0; s < nsn; ++s) sn_last[s] = (s + 1 < nsn ? sn_first[s + 1] : nsv) - 1;
    std::vector<int64_t> sn_of(nsv);
    for (int64_t s = 0; s < nsn; ++s)
        for (int64_t k = sn_first[s]; k <= sn_last[s]; ++k) sn_of[k] = s;
    std::vector<int64_t> snp(nsn), sncb(nsn), snz(nsn, 0), snpar(nsn);
    std::vector<char> live(nsn, 1);
    for (int64_t s = 0; s < nsn; ++s) {
        int64_t np = 0;
        for (int64_t k = sn_first[s]; k <= sn_last[s]; ++k) np += wsz[k];
        snp[s] = np;
        sncb[s] = wcnt[sn_last[s]];
        snpar[s] = par[sn_last[s]] >= 0 ? sn_of[par[sn_last[s]]] : -1;
    }
    if (opt.amalgamate && nsn > 1) {
        std::vector<int64_t> ending(nsv, -1), into(nsn);
        std::iota(into.begin(), into.end(), 0);
        auto find = [&](int64_t s) {
            int64_t r = s;
            while (into[r] != r) r = into[r];
            while (into[s] != r) { int64_t t = into[s]; into[s] = r; s = t; }
            return r;
        };
        for (int64_t s = 0; s < nsn; ++s) ending[sn_last[s]] = s;
        for (int64_t P = 0; P < nsn; ++P) {
            while (sn_first[P] > 0) {
                int64_t C = ending[sn_first[P] - 1];
                if (C < 0 || !live[C] || snpar[C] < 0 || find(snpar[C]) != P) break;
                int64_t npm = snp[C] + snp[P];
                double added = (double)snp[C] * (double)(snp[P] + sncb[P] - sncb[C]);
                double zm = (double)snz[C] + (double)snz[P] + added;
                double Lm = 0.5 * (double)npm * (double)(npm + 1) + (double)npm * (double)sncb[P];
                bool ok = npm <= opt.nrelax || zm <= opt.relax_frac * Lm;
                if (!ok) break;
                live[C] = 0;
                into[C] = P;
                ending[sn_last[C]] = -1;
                sn_first[P] = sn_first[C];
                snp[P] = npm;
                snz[P] = (int64_t)zm;
            }
        }
    }
    // fronts = live supernodes (postorder kept: merges are contiguous)
    std::vector<int64_t> ffirst, flast;
    for (int64_t s = 0; s < nsn; ++s)
        if (live[s]) { ffirst.push_back(sn_first[s]); flast.push_back(sn_last[s]); }
    const int64_t nf = (int64_t)ffirst.size();
    S.nf = nf;
    std::vector<int32_t> fr_of_sv(nsv);
    for (int64_t f = 0; f < nf; ++f)
        for (int64_t k = ffirst[f]; k <= flast[f]; ++k) fr_of_sv[k] = (int32_t)f;

    // ------------------------------------------------------------ 8. dof positions, perm
    std::vector<int64_t> sv_pos0(nsv + 1, 0);
    for (int64_t k = 0; k < nsv; ++k) sv_pos0[k + 1] = sv_pos0[k] + wsz[k];
    S.perm.resize(n);
    S.iperm.resize(n);
    for (int64_t k = 0; k < nsv; ++k) {
        int64_t d0 = sv_first[svperm[k]];
        for (int64_t t = 0; t < wsz[k]; ++t) {
            S.perm[sv_pos0[k] + t] = d0 + t;
            S.iperm[d0 + t] = sv_pos0[k] + t;
        }
    }

    // ------------------------------------------------------------ 9. front structures
    S.piv_first.resize(nf + 1);
    S.npiv.resize(nf);
    S.ncb.resize(nf);
    S.forder.resize(nf);
    S.parent.assign(nf, -1);
    S.cb_ptr.assign(nf + 1, 0);
    std::vector<int64_t> cbsv_ptr(nf + 1, 0), cbsv;
    std::vector<std::vector<int32_t>> kids(nf);
    std::fill(mark.begin(), mark.end(), -1);
    for (int64_t f = 0; f < nf; ++f) {
        int64_t lo = ffirst[f], hi = flast[f];
        std::vector<int64_t> lst;
        for (int64_t k = lo; k <= hi; ++k)
            for (int64_t q = nx_[k]; q < nx_[k + 1]; ++q) {
                int64_t t = na_[q];
                if (t > hi && mark[t] != f) { mark[t] = f; lst.push_back(t); }
            }
        for (int32_t c : kids[f])
            for (int64_t q = cbsv_ptr[c]; q < cbsv_ptr[c + 1]; ++q) {
                int64_t t = cbsv[q];
                if (t > hi && mark[t] != f) { mark[t] = f; lst.push_back(t); }
            }
        std::sort(lst.begin(), lst.end());
        cbsv.insert(cbsv.end(), lst.begin(), lst.end());
        cbsv_ptr[f + 1] = (int64_t)cbsv.size();
        if (!lst.empty()) {
            int32_t pf = fr_of_sv[lst[0]];
            S.parent[f] = pf;
            kids[pf].push_back((int32_t)f);
        }
        int64_t np = sv_pos0[hi + 1] - sv_pos0[lo], nc = 0;
        for (int64_t t : lst) nc += wsz[t];
        S.piv_first[f] = sv_pos0[lo];
        S.npiv[f] = (int32_t)np;
        S.ncb[f] = (int32_t)nc;
        if (np + nc + opt.delay_slack > 65535) return fmt("front too large for 16-bit local indices", np + nc);
        S.forder[f] = (int32_t)(np + nc);
        S.cb_ptr[f + 1] = S.cb_ptr[f] + nc;
    }
    S.piv_first[nf] = n;
    S.cb_rows.resize(S.cb_ptr[nf]);
    for (int64_t f = 0; f < nf; ++f) {
        int64_t w = S.cb_ptr[f];
        for (int64_t q = cbsv_ptr[f]; q < cbsv_ptr[f + 1]; ++q) {
            int64_t t = cbsv[q];
            for (int64_t d = 0; d < wsz[t]; ++d) S.cb_rows[w++] = sv_pos0[t] + d;
        }
    }
    S.child_ptr.assign(nf + 1, 0);
    for (int64_t f = 0; f < nf; ++f) S.child_ptr[f + 1] = S.child_ptr[f] + (int32_t)kids[f].size();
    S.child_list.resize(S.child_ptr[nf]);
    for (int64_t f = 0; f < nf; ++f)
        std::copy(kids[f].begin(), kids[f].end(), S.child_list.begin() + S.child_ptr[f]);

    // ------------------------------------------------------------ 10. extend-add relative maps
    std::vector<int32_t> local(n, -1);
    S.rmap_ptr = S.cb_ptr;
    S.rmap.assign(S.cb_ptr[nf], -1);
    auto set_local = [&](int64_t f, bool on) {
        int64_t p0 = S.piv_first[f];
        for (int32_t t = 0; t < S.npiv[f]; ++t) local[p0 + t] = on ? t : -1;
        for (int64_t q = S.cb_ptr[f]; q < S.cb_ptr[f + 1]; ++q)
            local[S.cb_rows[q]] = on ? (int32_t)(S.npiv[f] + (q - S.cb_ptr[f])) : -1;
    };
    for (int64_t f = 0; f < nf; ++f) {
        if (S.child_ptr[f] == S.child_ptr[f + 1]) continue;
        set_local(f, true);
        for (int32_t q = S.child_ptr[f]; q < S.child_ptr[f + 1]; ++q) {
            int32_t c = S.child_list[q];
            for (int64_t t = S.cb_ptr[c]; t < S.cb_ptr[c + 1]; ++t) {
                int32_t l = local[S.cb_rows[t]];
                if (l < 0) return "internal: child CB row missing from parent front";
                S.rmap[t] = l;
            }
        }
        set_local(f, false);
    }

    // ------------------------------------------------------------ 11. assembly map
    std::vector<int32_t> fr_of_pos(n);
    for (int64_t f = 0; f < nf; ++f)
        for (int64_t p = S.piv_first[f]; p < S.piv_first[f + 1]; ++p) fr_of_pos[p] = (int32_t)f;
    S.asm_ptr.assign(nf + 1, 0);
    std::vector<int32_t> efront(nnz);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) {
            int64_t pi = S.iperm[rowidx[q]], pj = S.iperm[j];
            int32_t f = fr_of_pos[std::min(pi, pj)];
            efront[q] = f;
            S.asm_ptr[f + 1]++;
        }
    for (int64_t f = 0; f < nf; ++f) S.asm_ptr[f + 1] += S.asm_ptr[f];
    S.asm_src.resize(nnz);
    S.asm_rc.resize(nnz);
    {
        std::vector<int64_t> w(S.asm_ptr.begin(), S.asm_ptr.end() - 1);
        for (int64_t j = 0; j < n; ++j)
            for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) S.asm_src[w[efront[q]]++] = q;
    }
    std::vector<int32_t>().swap(efront);
    // original entry -> column (for the source index)
    std::vector<int32_t> ecol(nnz);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) ecol[q] = (int32_t)j;
    for (int64_t f = 0; f < nf; ++f) {
        set_local(f, true);
        std::vector<std::pair<uint32_t, int64_t>> tmp;
        tmp.reserve(S.asm_ptr[f + 1] - S.asm_ptr[f]);
        for (int64_t k = S.asm_ptr[f]; k < S.asm_ptr[f + 1]; ++k) {
            int64_t q = S.asm_src[k];
            int64_t pi = S.iperm[rowidx[q]], pj = S.iperm[ecol[q]];
            int64_t lo = std::min(pi, pj), hi = std::max(pi, pj);
            int32_t lc = local[lo], lr = local[hi];
            if (lc < 0 || lr < 0 || lc >= S.npiv[f]) return "internal: entry outside its front";
            tmp.emplace_back(((uint32_t)lc << 16) | (uint32_t)lr, q);
        }
        std::sort(tmp.begin(), tmp.end());
        for (size_t t = 0; t < tmp.size(); ++t) {
            uint32_t key = tmp[t].first;       // (lc << 16 | lr) -> store (lr << 16 | lc)
            uint32_t lc = key >> 16, lr = key & 0xffffu;
            S.asm_rc[S.asm_ptr[f] + t] = (lr << 16) | lc;
            S.asm_src[S.asm_ptr[f] + t] = tmp[t].second;
        }
        set_local(f, false);
    }

    // ------------------------------------------------------------ 12. levels
    S.level.assign(nf, 0);
    int32_t nlev = 0;
    for (int64_t f = 0; f < nf; ++f) {            // children precede parents
        int32_t L = 0;
        for (int32_t q = S.child_ptr[f]; q < S.child_ptr[f + 1]; ++q)
            L = std::max(L, S.level[S.child_list[q]] + 1);
        S.level[f] = L;
        nlev = std::max(nlev, L + 1);
    }
    S.level_ptr.assign(nlev + 1, 0);
    for (int64_t f = 0; f < nf; ++f) S.level_ptr[S.level[f] + 1]++;
    for (int32_t L = 0; L < nlev; ++L) S.level_ptr[L + 1] += S.level_ptr[L];
    S.level_fronts.resize(nf);
    {
        std::vector<int32_t> w(S.level_ptr.begin(), S.level_ptr.end() - 1);
        for (int64_t f = 0; f < nf; ++f) S.level_fronts[w[S.level[f]]++] = (int32_t)f;
    }

    // ------------------------------------------------------------ 13. statistics
    S.max_front = 0;
    S.nzf_exec = 0;
    S.flops_exec = 0;
    S.flops_schur = 0;
    S.sum_cb = 0;
    for (int64_t f = 0; f < nf; ++f) {
        int64_t p = S.npiv[f], c = S.ncb[f], fo = p + c;
        S.max_front = std::max(S.max_front, fo);
        S.nzf_exec += p * fo - p * (p - 1) / 2;
        for (int64_t m = c; m < fo; ++m) S.flops_exec += (double)m * m + 2.0 * m;
        S.flops_schur += (double)p * (double)c * (double)(c + 1);
        S.sum_cb += c * (c + 1) / 2;
    }
    S.max_level_width = 0;
    for (int32_t L = 0; L < nlev; ++L)
        S.max_level_width = std::max<int64_t>(S.max_level_width, S.level_ptr[L + 1] - S.level_ptr[L]);

    plan_memory(S, opt.delay_slack);
    return "";
}

}  // namespace kep
