"""Multisection driver (host logic) — single process and world_size 2 over gloo on CPU.

The nu callable here is a stand-in with a known spectrum (counts by
searchsorted), so the driver logic is tested without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1710_05134_b200.multisection import Bracket, Multisection


def _spectrum(n=1000, seed=0):
    return np.sort(np.random.default_rng(seed).uniform(-5, 5, n))


def _nu_factory(w, singular_at=None):
    def nu_many(sig):
        sig = np.asarray(sig)
        st = np.zeros(sig.shape[0], dtype=np.int32)
        if singular_at is not None:
            st[np.isin(sig, singular_at)] = 3
        return np.searchsorted(w, sig, side="left").astype(np.int64), st
    return nu_many


def test_single_process_reaches_m_max():
    w = _spectrum()
    k = 300
    ms = Multisection(_nu_factory(w), k=k, shifts_per_rank=4, m_max=20)
    b = ms.run(Bracket(-6.0, 6.0, 0, len(w)))
    assert b.nu_lo < k <= b.nu_hi and b.count <= 20
    assert b.lo < w[k - 1] < b.hi
    # P = 1 is exactly Alg. 1': halving the bracket each round
    ms1 = Multisection(_nu_factory(w), k=k, shifts_per_rank=1, m_max=20)
    b0 = Bracket(-6.0, 6.0, 0, len(w))
    b1 = ms1.round(b0)
    assert b1.hi - b1.lo == pytest.approx((b0.hi - b0.lo) / 2)


def _with_eig_at(w, x):
    return np.sort(np.concatenate([w, [x]]))


@pytest.mark.parametrize("end", ["hi", "lo"])
def test_singular_shift_is_perturbed(end):
    """A singular shift sits on an eigenvalue: the bracket must pair the count with the
    perturbed shift it was evaluated at (nu(sigma + delta) was paired with sigma)."""
    P = 4
    b = Bracket(-6.0, 6.0, 0, 201)
    bad = Multisection(None, k=1, shifts_per_rank=P).shifts(b)[1]
    w = _with_eig_at(_spectrum(200, 1), bad)
    kb = int(np.searchsorted(w, bad, side="left"))      # w[kb] == bad
    k = kb + 1 if end == "hi" else kb + 2               # bracket ends (hi) / starts (lo) at the bad shift
    ms = Multisection(_nu_factory(w, singular_at=[bad]), k=k, shifts_per_rank=P)
    nb = ms.round(b)
    assert nb.nu_lo < k <= nb.nu_hi
    assert np.searchsorted(w, nb.lo, side="left") == nb.nu_lo
    assert np.searchsorted(w, nb.hi, side="left") == nb.nu_hi
    moved = nb.hi if end == "hi" else nb.lo
    assert moved != bad and abs(moved - bad) <= 4e-6 * (b.hi - b.lo)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = _spectrum(2000, 3)
    ms = Multisection(_nu_factory(w), k=k, shifts_per_rank=3, rank=rank, world=world)
    b = ms.run(Bracket(-6.0, 6.0, 0, len(w)))
    out[rank] = (b.lo, b.hi, b.nu_lo, b.nu_hi, len(ms.trace))
    dist.destroy_process_group()


def _worker_singular(rank, world, port, out):
    """The singular shift is rank 1's: rank 0 must learn the perturbed shift too."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = Bracket(-6.0, 6.0, 0, 201)
    bad = Multisection(None, k=1, shifts_per_rank=2, world=world).shifts(b)[1]   # global shift 1 -> rank 1
    w = _with_eig_at(_spectrum(200, 1), bad)
    k = int(np.searchsorted(w, bad, side="left"))
    ms = Multisection(_nu_factory(w, singular_at=[bad]), k=k, shifts_per_rank=2, rank=rank, world=world)
    nb = ms.round(b)
    out[rank] = (nb.lo, nb.hi, nb.nu_lo, nb.nu_hi, int(np.searchsorted(w, nb.hi, side="left")), bad)
    dist.destroy_process_group()


def test_two_ranks_gloo_singular_shift_shared():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_singular, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == out[1]
    lo, hi, nlo, nhi, nu_at_hi, bad = out[0]
    assert nhi == nu_at_hi and hi != bad


def test_two_ranks_gloo_agree_with_single():
    world, k = 2, 777
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), k, out), nprocs=world, join=True)
    assert out[0] == out[1]
    w = _spectrum(2000, 3)
    single = Multisection(_nu_factory(w), k=k, shifts_per_rank=6)          # same P = 6 shifts per round
    b = single.run(Bracket(-6.0, 6.0, 0, len(w)))
    assert out[0][:4] == (b.lo, b.hi, b.nu_lo, b.nu_hi)
    assert out[0][2] < k <= out[0][3]
