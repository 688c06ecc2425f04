"""O-sparse: a plain multifrontal LDL^T of A - sigma B, inertia only.

Follows Alg. 1' line 3: L D L^T <- P Q (A - sigma B) Q^T P^T,
with a fill-reducing ordering Q that depends on the pattern only and is
recycled across shifts (§3.3), and a stability permutation
P.  nu = nu_0(D, I) (Sylvester PAPER.md:87).

The paper hands the factorisation to MUMPS and says nothing
about its internals; this oracle takes the readings listed in DESIGN.md:

* Q (reading R6): geometric nested dissection on the atom coordinates:
  split a region at the median of its longest axis, the separator is the
  side's atoms adjacent to the other side (the smaller such set), recurse,
  separator ordered last; regions of <= LEAF atoms are leaves.  Pencils
  without coordinates use reverse Cuthill-McKee with one atom per front.
* fronts: one per ND node (leaf or separator); front structure by the
  symbolic rule struct(s) = piv(s) U adj_later(piv(s)) U (U_children
  struct(c) minus piv(c)); parent(s) = owner of min(struct(s) minus piv(s)).
* pivoting (reading R1): in a front with a contribution block, Bunch-Kaufman
  restricted to the fully-summed (FS) candidates, accepted only if the
  threshold test with u = 0.01 holds against the whole current column (1x1:
  |d| >= u max_i |a_ij|; 2x2: Duff-Reid |D^-1| [g_k; g_r] <= [1/u; 1/u]);
  otherwise the column is delayed to the parent.  A front without a
  contribution block (a root) runs textbook Bunch-Kaufman on everything.
* after the FS columns are eliminated the contribution block is the Schur
  complement C - L21 D L21^T (one matmul), passed to the parent together
  with the delayed rows/columns.

Plain numpy, fp64, full symmetric dense fronts; the pivot loop is unblocked
(_partial_fs_bk, the default) or, for the large configurations, the same rule
with nb-column panels and a BLAS3 update of the remaining FS columns
(_partial_fs_bk_blocked, pinned against the unblocked loop and eigh in
tests/test_oracle.py).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

from .dense_bk import ALPHA, Inertia, block_inertia_1x1, block_inertia_2x2

U_THRESHOLD = 0.01
LEAF = 16
_CHUNK = 2048           # column chunk of the blocked path's large products (bounds temporaries only)


# ----------------------------------------------------------------------------- ordering
def _atom_graph(p) -> sp.csr_matrix:
    o = p.o
    col = p.colidx()
    ra = p.rowidx.astype(np.int64) // o
    ca = col // o
    na = p.n // o
    G = sp.coo_matrix((np.ones(ra.shape[0]), (ra, ca)), shape=(na, na)).tocsr()
    G = ((G + G.T) > 0).astype(np.float64).tocsr()
    G.setdiag(0)
    G.eliminate_zeros()
    return G


def geometric_nd(G: sp.csr_matrix, coords: np.ndarray, leaf: int = LEAF):
    """Atom order and front blocks (list of (start, end) in the order)."""
    na = G.shape[0]
    order = np.empty(na, dtype=np.int64)
    blocks = []
    # explicit stack of tasks: ('region', ids, slot_start) ; fills order[slot:slot+len]
    stack = [(np.arange(na, dtype=np.int64), 0)]
    mark = np.zeros(na, dtype=np.float64)
    while stack:
        ids, start = stack.pop()
        m = ids.shape[0]
        if m == 0:
            continue
        if m <= leaf:
            order[start:start + m] = ids
            blocks.append((start, start + m))
            continue
        c = coords[ids]
        axis = int(np.argmax(c.max(axis=0) - c.min(axis=0)))
        srt = np.argsort(c[:, axis], kind="stable")
        Lh, Rh = ids[srt[: m // 2]], ids[srt[m // 2:]]
        mark[Rh] = 1.0
        bl = (G[Lh] @ mark) > 0                      # L atoms adjacent to R
        mark[Rh] = 0.0
        mark[Lh] = 1.0
        br = (G[Rh] @ mark) > 0                      # R atoms adjacent to L
        mark[Lh] = 0.0
        if bl.sum() <= br.sum():
            S, A1, A2 = Lh[bl], Lh[~bl], Rh
        else:
            S, A1, A2 = Rh[br], Lh, Rh[~br]
        if S.shape[0]:
            s0 = start + A1.shape[0] + A2.shape[0]
            order[s0:s0 + S.shape[0]] = np.sort(S)
            blocks.append((s0, s0 + S.shape[0]))
        stack.append((A1, start))
        stack.append((A2, start + A1.shape[0]))
    blocks.sort()
    return order, blocks


def rcm_order(G: sp.csr_matrix):
    na = G.shape[0]
    order = np.asarray(reverse_cuthill_mckee(G, symmetric_mode=True), dtype=np.int64)
    return order, [(i, i + 1) for i in range(na)]


# ----------------------------------------------------------------------------- symbolic
class SparseOracle:
    """Symbolic analysis of one pattern (recycled across shifts)."""

    def __init__(self, p, ordering: str = "auto", leaf: int = LEAF):
        self.p = p
        o = p.o
        G = _atom_graph(p)
        if ordering == "auto":
            ordering = "nd" if p.coords is not None else "rcm"
        if ordering == "nd":
            aorder, blocks = geometric_nd(G, p.coords, leaf)
        elif ordering == "rcm":
            aorder, blocks = rcm_order(G)
        elif ordering == "natural":
            aorder = np.arange(G.shape[0], dtype=np.int64)
            blocks = [(i, i + 1) for i in range(G.shape[0])]
        else:
            raise ValueError(ordering)
        assert np.array_equal(np.sort(aorder), np.arange(G.shape[0]))
        self.ordering = ordering
        apos = np.empty_like(aorder)
        apos[aorder] = np.arange(aorder.shape[0])
        # dof-level permutation: position of dof (atom*o + r) = apos[atom]*o + r
        dpos = (apos[:, None] * o + np.arange(o)[None, :]).ravel()
        self.dpos = dpos
        nb = len(blocks)
        owner = np.empty(aorder.shape[0], dtype=np.int64)   # atom position -> block
        for b, (s, e) in enumerate(blocks):
            owner[s:e] = b
        # symbolic: per block, atom-position structure
        Gp = G[aorder][:, aorder].tocsr()
        struct = [None] * nb
        parent = np.full(nb, -1, dtype=np.int64)
        pending = [[] for _ in range(nb)]
        children = [[] for _ in range(nb)]
        for b, (s, e) in enumerate(blocks):
            nbrs = Gp.indices[Gp.indptr[s]:Gp.indptr[e]]
            later = nbrs[nbrs >= e]
            parts = [np.arange(s, e), later] + pending[b]
            st = np.unique(np.concatenate(parts))
            struct[b] = st
            pending[b] = None
            cb = st[st >= e]
            if cb.shape[0]:
                par = int(owner[cb[0]])
                parent[b] = par
                children[par].append(b)
                pending[par].append(cb)
        self.blocks = blocks
        self.struct = struct
        self.parent = parent
        self.children = children
        # permuted lower CSC of the pattern, entry map (col-position, row-position, original index)
        col = p.colidx()
        pr = dpos[p.rowidx.astype(np.int64)]
        pc = dpos[col]
        lo = np.minimum(pr, pc)
        hi = np.maximum(pr, pc)
        srt = np.lexsort((hi, lo))
        self.e_col = lo[srt]
        self.e_row = hi[srt]
        self.e_src = srt
        n = p.n
        self.e_colptr = np.zeros(n + 1, dtype=np.int64)
        self.e_colptr[1:] = np.cumsum(np.bincount(self.e_col, minlength=n))
        # dofs of a block / struct in position space
        self.o = o

    def _dofs(self, atom_positions: np.ndarray) -> np.ndarray:
        o = self.o
        return (atom_positions[:, None] * o + np.arange(o)[None, :]).ravel()

    def front_sizes(self):
        return [(self.blocks[b][1] - self.blocks[b][0]) * self.o for b in range(len(self.blocks))], \
               [self.struct[b].shape[0] * self.o for b in range(len(self.blocks))]

    # ------------------------------------------------------------------------- numeric
    def inertia(self, sigma: float, u: float = U_THRESHOLD, nb: int = 0) -> Inertia:
        """Inertia of D.  nb = 0: the unblocked pivot loop (_partial_fs_bk);
        nb >= 1: the same pivot rule with nb-column panels and a BLAS3 update of
        the remaining FS columns after each panel (_partial_fs_bk_blocked)."""
        p = self.p
        vals = (p.a - sigma * p.b)[self.e_src]
        total = Inertia(smax=float(np.max(np.abs(vals))) if vals.shape[0] else 0.0)
        n = p.n
        pos = np.full(n, -1, dtype=np.int64)
        cbs = {}                                  # block -> (dof positions list, CB matrix)
        for b, (s, e) in enumerate(self.blocks):
            piv = self._dofs(np.arange(s, e))
            rest = self._dofs(self.struct[b][self.struct[b] >= e])
            delayed = []
            for c in self.children[b]:
                idx, _ = cbs[c]
                delayed.extend([x for x in idx if x < piv[0]])     # delayed dofs come from earlier blocks
            delayed = np.array(sorted(delayed), dtype=np.int64)
            fs = np.concatenate([piv, delayed])
            idx = np.concatenate([fs, rest])
            f = idx.shape[0]
            pos[idx] = np.arange(f)
            F = np.zeros((f, f), order="F" if nb > 0 else "C")
            # assemble original entries of the pivot columns (lower part, rows >= col)
            lo, hi = self.e_colptr[piv[0]], self.e_colptr[piv[-1] + 1]
            r = pos[self.e_row[lo:hi]]
            cc = pos[self.e_col[lo:hi]]
            assert np.all(r >= 0) and np.all(cc >= 0)
            v = vals[lo:hi]
            np.add.at(F, (r, cc), v)
            off = r != cc
            np.add.at(F, (cc[off], r[off]), v[off])
            # extend-add children contribution blocks (with their delayed rows/cols)
            for c in self.children[b]:
                cidx, C = cbs.pop(c)
                li = pos[np.asarray(cidx)]
                assert np.all(li >= 0)
                for j0 in range(0, li.shape[0], _CHUNK):    # column chunks (memory only)
                    j1 = min(li.shape[0], j0 + _CHUNK)
                    F[np.ix_(li, li[j0:j1])] += C[:, j0:j1]
                del C
            root = rest.shape[0] == 0
            if nb > 0:
                inert, order, e_cnt = _partial_fs_bk_blocked(F, fs.shape[0], u=u, root=root, nb=nb)
            else:
                inert, order, e_cnt = _partial_fs_bk(F, fs.shape[0], u=u, root=root)
            total.add(inert)
            if not root:
                loc = order[e_cnt:]
                cbs[b] = (idx[loc].tolist(), np.array(F[e_cnt:, e_cnt:], order="F"))   # a copy: F is freed
            pos[idx] = -1
            del F
        return total


# ----------------------------------------------------------------------------- front kernel
def _partial_fs_bk(F: np.ndarray, nfs: int, u: float, root: bool):
    """Eliminate FS columns 0..nfs-1 of the dense symmetric front F in place.

    Returns (Inertia, order, e): ``order`` is the local permutation applied
    (position -> original local index), e = number eliminated; on return
    F[e:, e:] holds the contribution block (delayed columns first, then the
    non-FS rows in their original order), symmetric.
    """
    f = F.shape[0]
    q = nfs
    res = Inertia()
    order = np.arange(f)
    Lfac = np.zeros((f, q))                 # multipliers L (rows x eliminated pivots)
    Dblocks = []                            # (k, size, Dk)
    e = 0
    qe = q                                  # candidates e..qe-1 ; delayed qe..q-1

    def swap(i, j):
        if i == j:
            return
        F[[i, j], :] = F[[j, i], :]
        F[:, [i, j]] = F[:, [j, i]]
        Lfac[[i, j], :] = Lfac[[j, i], :]
        order[[i, j]] = order[[j, i]]

    while e < qe:
        k = e
        akk = abs(F[k, k])
        candC = np.abs(F[k + 1:qe, k])
        if candC.shape[0]:
            r = k + 1 + int(np.argmax(candC))
            gC = float(candC[r - k - 1])
        else:
            r, gC = k, 0.0
        allR = np.abs(F[k + 1:, k])
        gR = float(np.max(allR)) if allR.shape[0] else 0.0
        if akk == 0.0 and gR == 0.0:
            res.n_zero += 1                   # zero column: exact zero pivot
            res.min_abs_pivot = 0.0
            Dblocks.append((k, 1, np.zeros((1, 1))))
            e += 1
            continue
        # Bunch-Kaufman choice among the FS candidates
        if akk >= ALPHA * gC:
            kind, j = 1, k
        else:
            rowr = np.abs(F[k:qe, r])
            rowr[r - k] = 0.0
            rho = float(np.max(rowr))
            if akk * rho >= ALPHA * gC * gC:
                kind, j = 1, k
            elif abs(F[r, r]) >= ALPHA * rho:
                kind, j = 1, r
            else:
                kind, j = 2, r
        if not root:
            if kind == 1:
                colj = np.abs(F[k:, j])
                colj[j - k] = 0.0
                ok = abs(F[j, j]) >= u * float(np.max(colj))
            else:
                det = F[k, k] * F[r, r] - F[r, k] * F[r, k]
                if det == 0.0:
                    ok = False
                else:
                    gk = np.abs(F[k:, k]); gk[0] = 0.0; gk[r - k] = 0.0
                    gr = np.abs(F[k:, r]); gr[0] = 0.0; gr[r - k] = 0.0
                    Dinv = np.abs(np.array([[F[r, r], -F[r, k]], [-F[r, k], F[k, k]]]) / det)
                    t = Dinv @ np.array([float(np.max(gk)), float(np.max(gr))])
                    ok = bool(np.all(t <= 1.0 / u))
            if not ok:
                swap(k, qe - 1)             # delay column k to the parent
                qe -= 1
                res.n_delayed += 1
                continue
        if kind == 1:
            swap(k, j)
            d = F[k, k]
            v = F[k + 1:, k].copy()
            # update the remaining FS columns (all rows); CB x CB is done at the end
            F[k + 1:, k + 1:q] -= np.outer(v, v[: q - k - 1]) / d
            Lfac[k + 1:, k] = v / d
            Dblocks.append((k, 1, np.array([[d]])))
            neg, zer, pos, mn = block_inertia_1x1(d)
            e += 1
        else:
            swap(k + 1, r)
            Dk = F[k:k + 2, k:k + 2].copy()
            V = F[k + 2:, k:k + 2].copy()
            W = V @ np.linalg.inv(Dk)
            F[k + 2:, k + 2:q] -= W @ V[: q - k - 2].T
            Lfac[k + 2:, k:k + 2] = W
            Dblocks.append((k, 2, Dk))
            neg, zer, pos, mn = block_inertia_2x2(Dk[0, 0], Dk[1, 0], Dk[1, 1])
            res.n_2x2 += 1
            e += 2
        res.n_neg += neg
        res.n_zero += zer
        res.n_pos += pos
        res.min_abs_pivot = min(res.min_abs_pivot, mn)
    if q < f and e > 0:
        # Schur complement of the non-FS block: C -= L21 D L21^T
        L21 = Lfac[q:, :e]
        W = np.zeros_like(L21)
        for (k, sz, Dk) in Dblocks:
            W[:, k:k + sz] = L21[:, k:k + sz] @ Dk
        F[q:, q:] -= W @ L21.T
    if e < f:
        T = F[e:, e:]
        lowT = np.tril(T)
        F[e:, e:] = lowT + np.tril(lowT, -1).T
    return res, order, e


def _partial_fs_bk_blocked(F: np.ndarray, nfs: int, u: float, root: bool, nb: int = 64):
    """The pivot rule of _partial_fs_bk with the FS columns eliminated in panels.

    Same contract and the same pivot sequence in exact arithmetic (SURVEY.md
    §8(c) O-sparse step 3: "nb-column BK panels with a BLAS3 update of the
    remaining FS columns"; the LAPACK dsytf2 -> dlasyf idea).  Inside a panel
    F is not updated: the current value of column j is formed on demand as
        F[:, j] - Lp[:, :t] Wp[j, :t]^T,     Lp = L columns, Wp = L D columns
    of the t pivots eliminated since the panel started (a 1x1 pivot d with
    updated column v contributes L = v / d, W = v; a 2x2 block Dk with updated
    columns V contributes L = V Dk^-1, W = V).  Every decision (BK choice,
    threshold test, delay) reads only such on-demand columns, exactly the
    values the unblocked loop holds at that step.  When the panel holds >= nb
    pivots (or no candidate is left) the remaining FS columns are updated at
    once: F[e:, e:q] -= Lp[e:] Wp[e:q]^T.  Rows and columns are swapped in F,
    Lp and Wp together, so swaps commute with the pending update.  With nb = 1
    every panel holds one pivot and this is the unblocked loop.

    Only the CB rows (>= q, never swapped) of L are kept for the final Schur
    complement, so a root front needs no L storage.
    """
    f = F.shape[0]
    q = nfs
    res = Inertia()
    order = np.arange(f)
    L21 = np.zeros((f - q, q))              # multipliers of the CB rows (rows >= q)
    Dblocks = []
    e = 0
    qe = q
    width = nb + 1                          # a 2x2 pivot may overfill the panel by one column
    Lp = np.zeros((f, width), order="F")
    Wp = np.zeros((f, width), order="F")
    t = 0

    def col(j):                             # current column j, rows e..f-1
        c = F[e:, j].copy()
        if t:
            c -= Lp[e:, :t] @ Wp[j, :t]
        return c

    def swap(i, j):
        if i == j:
            return
        F[[i, j], :] = F[[j, i], :]
        F[:, [i, j]] = F[:, [j, i]]
        Lp[[i, j], :t] = Lp[[j, i], :t]
        Wp[[i, j], :t] = Wp[[j, i], :t]
        order[[i, j]] = order[[j, i]]

    def flush():
        nonlocal t
        if t and e < q:
            for j0 in range(e, q, _CHUNK):          # column chunks: bounded temporaries (memory only)
                j1 = min(q, j0 + _CHUNK)
                F[e:, j0:j1] -= Lp[e:, :t] @ Wp[j0:j1, :t].T
        t = 0

    while e < qe:
        k = e
        ck = col(k)                          # ck[i - k] = current F[i, k]
        akk = abs(ck[0])
        candC = np.abs(ck[1:qe - k])
        if candC.shape[0]:
            r = k + 1 + int(np.argmax(candC))
            gC = float(candC[r - k - 1])
        else:
            r, gC = k, 0.0
        gR = float(np.max(np.abs(ck[1:]))) if f - k > 1 else 0.0
        if akk == 0.0 and gR == 0.0:
            res.n_zero += 1                   # zero column: exact zero pivot, nothing to update
            res.min_abs_pivot = 0.0
            Dblocks.append((k, 1, np.zeros((1, 1))))
            e += 1
            if e >= qe:
                flush()
            continue
        cr = None
        if akk >= ALPHA * gC:
            kind, j = 1, k
        else:
            cr = col(r)                       # cr[i - k] = current F[i, r]
            rowr = np.abs(cr[0:qe - k])
            rowr[r - k] = 0.0
            rho = float(np.max(rowr))
            if akk * rho >= ALPHA * gC * gC:
                kind, j = 1, k
            elif abs(cr[r - k]) >= ALPHA * rho:
                kind, j = 1, r
            else:
                kind, j = 2, r
        if not root:
            if kind == 1:
                cj = ck if j == k else cr
                colj = np.abs(cj)
                colj[j - k] = 0.0
                ok = abs(cj[j - k]) >= u * float(np.max(colj))
            else:
                fkk, frr, frk = ck[0], cr[r - k], ck[r - k]
                det = fkk * frr - frk * frk
                if det == 0.0:
                    ok = False
                else:
                    gk = np.abs(ck); gk[0] = 0.0; gk[r - k] = 0.0
                    gr = np.abs(cr); gr[0] = 0.0; gr[r - k] = 0.0
                    Dinv = np.abs(np.array([[frr, -frk], [-frk, fkk]]) / det)
                    tt = Dinv @ np.array([float(np.max(gk)), float(np.max(gr))])
                    ok = bool(np.all(tt <= 1.0 / u))
            if not ok:
                swap(k, qe - 1)             # delay column k to the parent
                qe -= 1
                res.n_delayed += 1
                if e >= qe:
                    flush()
                continue
        if kind == 1:
            swap(k, j)
            ck = col(k)
            d = ck[0]
            v = ck[1:]
            Lp[k + 1:, t] = v / d
            Wp[k + 1:, t] = v
            Lp[:k + 1, t] = 0.0
            Wp[:k + 1, t] = 0.0
            if q < f:
                L21[:, k] = v[q - k - 1:] / d
            Dblocks.append((k, 1, np.array([[d]])))
            neg, zer, pos, mn = block_inertia_1x1(d)
            t += 1
            e += 1
        else:
            swap(k + 1, r)
            c0 = col(k)
            c1 = col(k + 1)
            Dk = np.array([[c0[0], c1[0]], [c1[0], c1[1]]])
            V = np.stack([c0[2:], c1[2:]], axis=1)
            W = V @ np.linalg.inv(Dk)
            Lp[k + 2:, t:t + 2] = W
            Wp[k + 2:, t:t + 2] = V
            Lp[:k + 2, t:t + 2] = 0.0
            Wp[:k + 2, t:t + 2] = 0.0
            if q < f:
                L21[:, k:k + 2] = W[q - k - 2:]
            Dblocks.append((k, 2, Dk))
            neg, zer, pos, mn = block_inertia_2x2(Dk[0, 0], Dk[1, 0], Dk[1, 1])
            res.n_2x2 += 1
            t += 2
            e += 2
        res.n_neg += neg
        res.n_zero += zer
        res.n_pos += pos
        res.min_abs_pivot = min(res.min_abs_pivot, mn)
        if t >= nb or e >= qe:
            flush()
    flush()
    if q < f and e > 0:
        # Schur complement of the non-FS block: C -= L21 D L21^T
        L = L21[:, :e]
        W = np.zeros_like(L)
        for (k, sz, Dk) in Dblocks:
            W[:, k:k + sz] = L[:, k:k + sz] @ Dk
        for j0 in range(q, f, _CHUNK):              # column chunks (memory only)
            j1 = min(f, j0 + _CHUNK)
            F[q:, j0:j1] -= W @ L[j0 - q:j1 - q].T
    if e < f:                                       # symmetric trailing block: upper <- lower, in place
        for j0 in range(e, f, _CHUNK):
            j1 = min(f, j0 + _CHUNK)
            B = F[j0:j1, j0:j1]
            B[:] = np.tril(B) + np.tril(B, -1).T
            if j1 < f:
                F[j0:j1, j1:] = F[j1:, j0:j1].T
    return res, order, e


def nu_sparse(p, sigma: float, oracle: SparseOracle | None = None, u: float = U_THRESHOLD) -> Inertia:
    """Inertia of D from the multifrontal LDL^T of A - sigma B; nu = .n_neg."""
    so = oracle if oracle is not None else SparseOracle(p)
    return so.inertia(sigma, u=u)
