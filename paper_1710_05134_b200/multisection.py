"""Stage 2 driver: spectral multisection over shifts and GPUs.

Alg. 1' halves [sigma_l, sigma_u) with one nu evaluation
per iteration until nu_u - nu_l <= m_max (m_max = 20).  With P
devices the natural B200 generalisation (reading R12) evaluates P
interior shifts per round,

    sigma_i = sigma_l + i (sigma_u - sigma_l) / (P + 1),   i = 1..P,

and keeps the first consecutive pair with nu_a < k <= nu_b (for P = 1 this is
exactly Alg. 1' line 5).  Every rank evaluates its own shifts through the C ABI
(kep_inertia_many); the int64 counts are all-gathered over torch.distributed
(NCCL on GPUs, gloo in CPU tests) — the only exchange step — and every rank
applies the same deterministic update.  A shift reported singular
(KEP_ESINGULAR) is perturbed by 1e-6 (sigma_u - sigma_l) and re-evaluated
(R3).  Host logic only: no arithmetic of the
factorisation happens here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import numpy as np

KEP_OK = 0


@dataclass
class Bracket:
    lo: float
    hi: float
    nu_lo: int
    nu_hi: int

    @property
    def count(self) -> int:
        return self.nu_hi - self.nu_lo


@dataclass
class RoundTrace:
    shifts: List[float]
    nus: List[int]
    bracket: Tuple[float, float, int, int]


@dataclass
class Multisection:
    nu_many: Callable[[np.ndarray], Tuple[np.ndarray, np.ndarray]]   # sigmas -> (nus, status)
    k: int
    shifts_per_rank: int = 16
    m_max: int = 20
    group: object = None               # torch.distributed process group (None = default / single)
    rank: int = 0
    world: int = 1
    device: Optional[object] = None    # torch device for the all-gather buffer (cuda for NCCL)
    trace: List[RoundTrace] = field(default_factory=list)

    def shifts(self, b: Bracket) -> np.ndarray:
        P = self.world * self.shifts_per_rank
        return b.lo + (np.arange(P, dtype=np.float64) + 1.0) * (b.hi - b.lo) / (P + 1)

    def _local(self, sig: np.ndarray, width: float):
        """nu at this rank's shifts; a singular shift is moved by attempt * 1e-6 * width
        and re-evaluated (R3).  Returns (nus, shifts actually evaluated)."""
        sig = np.asarray(sig, dtype=np.float64).copy()
        nus, st = self.nu_many(sig)
        nus = np.asarray(nus, dtype=np.int64).copy()
        st = np.asarray(st)
        for i in np.nonzero(st != KEP_OK)[0]:
            s = float(sig[i])
            for attempt in range(1, 5):                      # perturb and retry (R3)
                s2 = s + attempt * 1e-6 * width
                v, st2 = self.nu_many(np.array([s2]))
                if st2[0] == KEP_OK:
                    nus[i] = v[0]
                    sig[i] = s2
                    break
            else:
                raise RuntimeError(f"shift {s} stays singular after perturbation")
        return nus, sig

    def _allgather(self, nus: np.ndarray, sig: np.ndarray):
        """All ranks' (nu, sigma) in global shift order.  One collective: the int64 counts
        and the float64 shifts (bit-cast to int64) travel in one int64 tensor."""
        if self.world == 1:
            return nus, sig
        import torch
        import torch.distributed as dist
        packed = np.concatenate([nus.astype(np.int64), sig.astype(np.float64).view(np.int64)])
        t = torch.from_numpy(packed)
        if self.device is not None:
            t = t.to(self.device)
        out = torch.empty(self.world * packed.shape[0], dtype=torch.int64, device=t.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        g = out.cpu().numpy().reshape(self.world, 2, -1)
        # rank r holds shifts r, r+world, ... ; restore shift order
        nu_all = g[:, 0, :].T.reshape(-1).copy()
        sig_all = g[:, 1, :].copy().view(np.float64).T.reshape(-1).copy()
        return nu_all, sig_all

    def round(self, b: Bracket) -> Bracket:
        sig_plan = self.shifts(b)
        mine = sig_plan[self.rank::self.world]
        nus_loc, sig_loc = self._local(mine, b.hi - b.lo)
        nus, sig_all = self._allgather(nus_loc, sig_loc)
        # the bracket pairs every count with the shift it was evaluated at (a perturbed
        # singular shift included), so nu(sigma) = #{lambda < sigma} holds for both ends
        sig_full = np.concatenate([[b.lo], sig_all, [b.hi]])
        nu_full = np.concatenate([[b.nu_lo], nus, [b.nu_hi]])
        if np.any(np.diff(sig_full) <= 0):
            raise RuntimeError("perturbed shifts are not increasing")
        if np.any(np.diff(nu_full) < 0):
            raise RuntimeError("nu is not monotone in sigma: inconsistent counts")
        j = int(np.searchsorted(nu_full, self.k, side="left")) - 1     # first pair nu_a < k <= nu_b
        j = min(max(j, 0), len(sig_full) - 2)
        nb = Bracket(float(sig_full[j]), float(sig_full[j + 1]), int(nu_full[j]), int(nu_full[j + 1]))
        self.trace.append(RoundTrace(sig_all.tolist(), nus.tolist(), (nb.lo, nb.hi, nb.nu_lo, nb.nu_hi)))
        return nb

    def run(self, b: Bracket, max_rounds: int = 64) -> Bracket:
        if not (b.nu_lo < self.k <= b.nu_hi):
            raise ValueError("bracket does not contain the k-th eigenvalue")
        for _ in range(max_rounds):
            if b.count <= self.m_max:
                break
            b = self.round(b)
        return b

    def step(self, b: Bracket, initial: Bracket) -> Tuple[Bracket, bool]:
        """One round of a repeated stage 2 (the benchmark step): returns the new bracket,
        or `initial` again (restart) once the bracket holds <= m_max eigenvalues."""
        nb = self.round(b)
        if nb.count <= self.m_max:
            return initial, True
        return nb, False
