"""Host-side checks of the C-ABI library (no GPU): exports, validation, symbolic.

The symbolic analysis (kep_analyze) is pinned against
brute-force boolean elimination in the oracle (pin P9).
"""
import ctypes
import os
import re

import numpy as np
import pytest

import kepgen
from oracle.symbolic import brute_symbolic, factor_flops
from paper_1710_05134_b200 import Kep, KepError, lib
from paper_1710_05134_b200.kep import KEP_EINVAL, KEP_ENODEVICE

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    h = open(os.path.join(ROOT, "include", "kep.h")).read()
    return sorted(set(re.findall(r"KEP_API\s+[\w\s\*]+?\b(kep_\w+)\s*\(", h)))


def test_library_exports_every_declared_symbol():
    L = lib()
    names = _declared_symbols()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
    assert L.kep_version().decode().startswith("kep")


def test_analyze_rejects_bad_patterns():
    # entry above the diagonal / missing diagonal / unsorted rows -> KEP_EINVAL
    bad = [
        (2, [0, 1, 2], [1, 1]),          # column 0 lacks its diagonal
        (2, [0, 2, 3], [0, 1, 0]),       # column 1 holds row 0 (upper)
        (3, [0, 3, 4, 5], [0, 2, 1, 1, 2]),  # unsorted
    ]
    for n, cp, ri in bad:
        with pytest.raises(KepError) as e:
            Kep(n, np.array(cp), np.array(ri))
        assert e.value.status == KEP_EINVAL


@pytest.mark.parametrize("shape,o,seed,amal", [((2, 3, 3), 2, 5, False), ((3, 3, 3), 1, 6, False),
                                               ((2, 2, 4), 3, 7, True)])
def test_symbolic_vs_bruteforce(shape, o, seed, amal):
    p = kepgen.tb_pencil(shape=shape, o=o, seed=seed)
    k = Kep.from_pencil(p, amalgamate=amal)
    perm = k.perm()
    assert np.array_equal(np.sort(perm), np.arange(p.n))
    pos = np.empty(p.n, dtype=np.int64)
    pos[perm] = np.arange(p.n)
    counts, parent = brute_symbolic(p.n, p.colptr, p.rowidx, pos)
    a = k.analysis()
    assert a["nzf"] == counts.sum()
    assert a["flops"] == factor_flops(counts)
    assert a["nzf_exec"] >= a["nzf"] and a["flops_exec"] >= a["flops"]
    # front structure: every column's true structure fits in its front, and the
    # assembly tree is consistent with the elimination tree
    first, fparent, forder = k.fronts()
    nf = len(fparent)
    front_of = np.repeat(np.arange(nf), np.diff(first))
    for j in range(p.n):
        f = front_of[j]
        # column count of pivot j cannot exceed what its front holds below it
        assert counts[j] <= forder[f] - (j - first[f])
        if parent[j] >= 0:
            pf = front_of[parent[j]]
            assert pf == f or fparent[f] == pf or pf > f


def test_natural_and_user_orderings():
    p = kepgen.tb_pencil(shape=(2, 2, 3), o=2, seed=8)
    kn = Kep.from_pencil(p, ordering="natural")
    assert np.array_equal(kn.perm(), np.arange(p.n))
    rp = np.random.default_rng(0).permutation(p.n)
    ku = Kep.from_pencil(p, user_perm=rp)
    pu = ku.perm()
    assert np.array_equal(np.sort(pu), np.arange(p.n))
    # user order is coarsened to supervariables (atoms): first atom placed first
    assert pu[0] // 2 == rp[0] // 2


def test_no_device_is_reported_not_faked():
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    p = kepgen.tb_pencil(shape=(2, 2, 2), o=1, seed=1)
    k = Kep.from_pencil(p)
    with pytest.raises(KepError) as e:
        k.set_values(p.a, p.b)
    assert e.value.status == KEP_ENODEVICE
