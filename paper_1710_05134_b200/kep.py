"""Thin ctypes binding of libkep.so (include/kep.h) — argument marshalling only.

Every step of the numeric path runs in the CUDA kernels behind the C ABI;
this module never computes anything itself and has no CPU fallback: if the
shared library is missing it raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libkep.so")

KEP_OK, KEP_EINVAL, KEP_EPATTERN, KEP_ESINGULAR, KEP_ENOTSPD, KEP_ENOMEM, KEP_ECUDA = range(7)
KEP_ENODEVICE = 10
ORDER = {"auto": 0, "metis": 1, "natural": 2, "user": 3}


class KepError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class _Opts(C.Structure):
    _fields_ = [("ordering", C.c_int), ("user_perm", C.POINTER(C.c_int64)), ("amalgamate", C.c_int32),
                ("nrelax", C.c_int32), ("relax_frac", C.c_double), ("pivot_u", C.c_double),
                ("tau_sing", C.c_double), ("delay_slack", C.c_int32), ("max_batch", C.c_int32),
                ("device", C.c_int32), ("stream", C.c_void_p), ("kernel_variant", C.c_int32),
                ("profile", C.c_int32)]


class _Profile(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_int64 * 8), ("schur_flops", C.c_double),
                ("schur_tma_flops", C.c_double), ("factor_flops", C.c_double), ("shifts", C.c_int64),
                ("other_launches", C.c_int64)]


KERNEL_CLASSES = ("assemble", "fs", "ref", "schur", "l21", "check", "fsu", "schur_tma")


class _Info(C.Structure):
    _fields_ = [("n_neg", C.c_int64), ("n_zero", C.c_int64), ("n_pos", C.c_int64), ("n_2x2", C.c_int64),
                ("n_delayed", C.c_int64), ("min_abs_pivot", C.c_double), ("max_abs_entry", C.c_double),
                ("n_redo", C.c_int64)]


class _Analysis(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz_lower", C.c_int64), ("n_supervariables", C.c_int64),
                ("n_fronts", C.c_int64), ("n_levels", C.c_int64), ("max_front", C.c_int64),
                ("max_level_width", C.c_int64), ("nzf", C.c_int64), ("nzf_exec", C.c_int64),
                ("flops", C.c_double), ("flops_exec", C.c_double), ("flops_schur", C.c_double),
                ("sum_cb", C.c_int64), ("arena_bytes", C.c_int64), ("delay_slack", C.c_int32),
                ("batch", C.c_int32)]


class _FStats(C.Structure):
    _fields_ = [("sigma", C.c_double), ("nu", C.c_int64), ("inertia", _Info), ("n", C.c_int64),
                ("nnz_L", C.c_int64), ("store_bytes", C.c_int64)]


class _KthOpts(C.Structure):
    _fields_ = [("m_max", C.c_int32), ("tau_res", C.c_double), ("tau_diff", C.c_double),
                ("max_lanczos", C.c_int32), ("max_bisect", C.c_int32), ("max_si", C.c_int32),
                ("shifts_per_round", C.c_int32), ("seed", C.c_uint64),
                ("v0_stage1", C.POINTER(C.c_double)), ("v0_stage3", C.POINTER(C.c_double)),
                ("bisect_only", C.c_int32), ("bisect_rtol", C.c_double), ("root_finder", C.c_int32)]


class _KthReport(C.Structure):
    _fields_ = [("s1_lower", C.c_double), ("s1_upper", C.c_double), ("s1_nu_lower", C.c_int64),
                ("s1_nu_upper", C.c_int64), ("sigma_lower", C.c_double), ("sigma_upper", C.c_double),
                ("nu_lower", C.c_int64), ("nu_upper", C.c_int64), ("sigma_si", C.c_double),
                ("stage1_iters", C.c_int32), ("stage2_rounds", C.c_int32), ("stage2_shifts", C.c_int32),
                ("stage3_iters", C.c_int32), ("eta", C.c_double), ("rel_residual", C.c_double),
                ("rel_diff", C.c_double), ("seconds", C.c_double * 3), ("status", C.c_int),
                ("s3_iter_bound", C.c_int32), ("s3_iter_residual", C.c_int32), ("s3_iter_difference", C.c_int32),
                ("stage2_trace_len", C.c_int32), ("stage2_trace_lower", C.c_double * 64),
                ("stage2_trace_upper", C.c_double * 64), ("stage2_trace_m", C.c_int64 * 64)]


_lib = None


def lib():
    """Load libkep.so (raises if it has not been built: no silent fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing — run __graft_entry__.build() "
                              "(python -m paper_1710_05134_b200.build)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.kep_default_opts.argtypes = [P(_Opts)]
        L.kep_analyze.argtypes = [C.c_int64, P(C.c_int64), P(C.c_int32), P(_Opts), P(C.c_void_p)]
        L.kep_set_values.argtypes = [C.c_void_p, P(C.c_double), P(C.c_double)]
        L.kep_set_values_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.kep_inertia.argtypes = [C.c_void_p, C.c_double, P(C.c_int64), P(_Info)]
        L.kep_inertia_many.argtypes = [C.c_void_p, C.c_int32, P(C.c_double), P(C.c_int64), P(C.c_int), P(_Info)]
        L.kep_get_analysis.argtypes = [C.c_void_p, P(_Analysis)]
        L.kep_get_perm.argtypes = [C.c_void_p, P(C.c_int64)]
        L.kep_get_fronts.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64)]
        L.kep_destroy.argtypes = [C.c_void_p]
        L.kep_get_profile.argtypes = [C.c_void_p, P(_Profile)]
        L.kep_reset_profile.argtypes = [C.c_void_p]
        L.kep_status_string.argtypes = [C.c_int]
        L.kep_status_string.restype = C.c_char_p
        L.kep_last_error.argtypes = [C.c_void_p]
        L.kep_last_error.restype = C.c_char_p
        L.kep_version.restype = C.c_char_p
        L.kep_factor.argtypes = [C.c_void_p, C.c_double, P(C.c_void_p)]
        L.kep_factor_pencil.argtypes = [C.c_void_p, C.c_double, C.c_double, P(C.c_void_p)]
        L.kep_factor_pencil.restype = C.c_int
        L.kep_default_kth_opts.argtypes = [P(_KthOpts)]
        L.kep_default_kth_opts.restype = None
        L.kep_kth_eigenpair.argtypes = [C.c_void_p, C.c_int64, P(_KthOpts), P(C.c_double), P(C.c_double),
                                        P(_KthReport)]
        L.kep_kth_eigenpair.restype = C.c_int
        L.kep_factor_info.argtypes = [C.c_void_p, P(_FStats)]
        L.kep_solve.argtypes = [C.c_void_p, C.c_int32, P(C.c_double), C.c_int64, P(C.c_double), C.c_int64]
        L.kep_solve_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.kep_factor_export.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_double), P(C.c_double), P(C.c_int64),
                                        P(C.c_int32), P(C.c_double)]
        L.kep_tridiag_eigen.argtypes = [C.c_int32, P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double)]
        L.kep_tridiag_eigen.restype = C.c_int
        L.kep_factor_residual.argtypes = [C.c_void_p, C.c_double, P(C.c_double), P(C.c_double)]
        L.kep_factor_residual.restype = C.c_int
        L.kep_factor_destroy.argtypes = [C.c_void_p]
        L.kep_factor_destroy.restype = None
        for f in ("kep_factor", "kep_factor_info", "kep_solve", "kep_solve_dev", "kep_factor_export"):
            getattr(L, f).restype = C.c_int
        for f in ("kep_analyze", "kep_set_values", "kep_set_values_dev", "kep_inertia", "kep_inertia_many",
                  "kep_get_analysis", "kep_get_perm", "kep_get_fronts", "kep_get_profile", "kep_reset_profile"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _status_name(s: int) -> str:
    try:
        return lib().kep_status_string(s).decode()
    except Exception:
        return str(s)


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class InertiaInfo:
    n_neg: int
    n_zero: int
    n_pos: int
    n_2x2: int
    n_delayed: int
    min_abs_pivot: float
    max_abs_entry: float
    n_redo: int


class Kep:
    """One analysed pattern on one device (kep_ctx)."""

    def __init__(self, n, colptr, rowidx, ordering="auto", user_perm=None, amalgamate=True, nrelax=48,
                 relax_frac=0.05, pivot_u=0.01, tau_sing=1e-14, delay_slack=16, max_batch=16, device=-1,
                 stream=None, kernel_variant=0, profile=False):
        L = lib()
        o = _Opts()
        L.kep_default_opts(C.byref(o))
        o.ordering = ORDER[ordering]
        self._perm_keep = None
        if user_perm is not None:
            self._perm_keep = np.ascontiguousarray(user_perm, dtype=np.int64)
            o.user_perm = _ptr(self._perm_keep, C.c_int64)
            o.ordering = ORDER["user"]
        o.amalgamate = int(bool(amalgamate))
        o.nrelax = int(nrelax)
        o.relax_frac = float(relax_frac)
        o.pivot_u = float(pivot_u)
        o.tau_sing = float(tau_sing)
        o.delay_slack = int(delay_slack)
        o.max_batch = int(max_batch)
        o.device = int(device)
        o.stream = stream
        o.kernel_variant = int(kernel_variant)
        o.profile = int(bool(profile))
        self.n = int(n)
        cp = np.ascontiguousarray(colptr, dtype=np.int64)
        ri = np.ascontiguousarray(rowidx, dtype=np.int32)
        self.nnz = int(cp[-1])
        h = C.c_void_p()
        st = L.kep_analyze(self.n, _ptr(cp, C.c_int64), _ptr(ri, C.c_int32), C.byref(o), C.byref(h))
        if st != KEP_OK:
            raise KepError(st, L.kep_last_error(None).decode())
        self._h = h

    @classmethod
    def from_pencil(cls, p, **kw):
        k = cls(p.n, p.colptr, p.rowidx, **kw)
        return k

    def _check(self, st):
        if st != KEP_OK:
            raise KepError(st, lib().kep_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            lib().kep_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_values(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        if a.shape != (self.nnz,) or b.shape != (self.nnz,):
            raise KepError(KEP_EPATTERN, "values do not match the analysed pattern")
        self._check(lib().kep_set_values(self._h, _ptr(a, C.c_double), _ptr(b, C.c_double)))

    def set_values_dev(self, a_ptr: int, b_ptr: int):
        self._check(lib().kep_set_values_dev(self._h, C.c_void_p(a_ptr), C.c_void_p(b_ptr)))

    def inertia(self, sigma: float):
        """Returns (status, nu, InertiaInfo); status KEP_OK or KEP_ESINGULAR."""
        nu = C.c_int64(-1)
        info = _Info()
        st = lib().kep_inertia(self._h, float(sigma), C.byref(nu), C.byref(info))
        if st not in (KEP_OK, KEP_ESINGULAR):
            self._check(st)
        return st, (int(nu.value) if st == KEP_OK else None), InertiaInfo(*[getattr(info, f) for f, _ in _Info._fields_])

    def inertia_many(self, sigmas, with_info=False):
        s = np.ascontiguousarray(sigmas, dtype=np.float64)
        m = s.shape[0]
        nus = np.full(m, -1, dtype=np.int64)
        per = np.zeros(m, dtype=np.int32)
        infos = (_Info * max(m, 1))()
        self._check(lib().kep_inertia_many(self._h, m, _ptr(s, C.c_double), _ptr(nus, C.c_int64),
                                           _ptr(per, C.c_int), infos if with_info else None))
        if with_info:
            return nus, per, [InertiaInfo(*[getattr(infos[i], f) for f, _ in _Info._fields_]) for i in range(m)]
        return nus, per

    def analysis(self) -> dict:
        a = _Analysis()
        self._check(lib().kep_get_analysis(self._h, C.byref(a)))
        return {f: getattr(a, f) for f, _ in _Analysis._fields_}

    def profile(self) -> dict:
        pr = _Profile()
        self._check(lib().kep_get_profile(self._h, C.byref(pr)))
        return dict(ms={n: pr.ms[i] for i, n in enumerate(KERNEL_CLASSES)},
                    launches={n: pr.launches[i] for i, n in enumerate(KERNEL_CLASSES)},
                    schur_flops=pr.schur_flops, schur_tma_flops=pr.schur_tma_flops, factor_flops=pr.factor_flops,
                    shifts=pr.shifts,
                    other_launches=pr.other_launches)

    def reset_profile(self):
        self._check(lib().kep_reset_profile(self._h))

    def factor(self, sigma: float) -> "Factor":
        """kep_factor: retained LDL^T of A - sigma B (raises KepError, e.g. KEP_ESINGULAR)."""
        h = C.c_void_p()
        self._check(lib().kep_factor(self._h, float(sigma), C.byref(h)))
        return Factor(self, h)

    def factor_pencil(self, alpha: float, sigma: float) -> "Factor":
        """Retained LDL^T of alpha A - sigma B (alpha = 0, sigma = -1: B)."""
        h = C.c_void_p()
        self._check(lib().kep_factor_pencil(self._h, float(alpha), float(sigma), C.byref(h)))
        return Factor(self, h)

    def factor_residual(self, sigma: float):
        """kep_factor_residual: (sum_s ||E_s||_F, max_s ||E_s||_F), the front-local bound of
        ||P (A - sigma B) P^T - L D L^T||_F."""
        bound, mx = C.c_double(np.nan), C.c_double(np.nan)
        self._check(lib().kep_factor_residual(self._h, float(sigma), C.byref(bound), C.byref(mx)))
        return bound.value, mx.value

    def kth_eigenpair(self, k: int, m_max=20, tau_res=1e-10, tau_diff=1e-10, max_lanczos=64, max_bisect=128,
                      max_si=500, shifts_per_round=1, seed=1, v0_stage1=None, v0_stage3=None, want_x=True,
                      bisect_only=False, bisect_rtol=1e-14, root_finder="bisection"):
        """kep_kth_eigenpair: (lambda_k or None, x or None, report dict)."""
        o = _KthOpts()
        lib().kep_default_kth_opts(C.byref(o))
        o.m_max, o.tau_res, o.tau_diff = int(m_max), float(tau_res), float(tau_diff)
        o.max_lanczos, o.max_bisect, o.max_si = int(max_lanczos), int(max_bisect), int(max_si)
        o.shifts_per_round, o.seed = int(shifts_per_round), int(seed)
        o.bisect_only, o.bisect_rtol = int(bool(bisect_only)), float(bisect_rtol)
        o.root_finder = {"bisection": 0, "brent": 1}[root_finder]
        keep = []
        for name, v in (("v0_stage1", v0_stage1), ("v0_stage3", v0_stage3)):
            if v is not None:
                arr = np.ascontiguousarray(v, dtype=np.float64)
                assert arr.shape == (self.n,)
                keep.append(arr)
                setattr(o, name, _ptr(arr, C.c_double))
        lam = C.c_double(np.nan)
        x = np.empty(self.n) if want_x else None
        rp = _KthReport()
        st = lib().kep_kth_eigenpair(self._h, int(k), C.byref(o), C.byref(lam),
                                     _ptr(x, C.c_double) if want_x else C.cast(None, C.POINTER(C.c_double)),
                                     C.byref(rp))
        self._check(st)
        arrays = ("seconds", "stage2_trace_lower", "stage2_trace_upper", "stage2_trace_m")
        rep = {f: getattr(rp, f) for f, _ in _KthReport._fields_ if f not in arrays}
        rep["seconds"] = list(rp.seconds)
        nt = rp.stage2_trace_len
        rep["stage2_trace"] = [(rp.stage2_trace_lower[i], rp.stage2_trace_upper[i], rp.stage2_trace_m[i])
                               for i in range(nt)]
        # Table 4 / Table 5 analogues: length, index range, m, gap
        for tag, a, b, na, nb in (("table4", rp.s1_lower, rp.s1_upper, rp.s1_nu_lower, rp.s1_nu_upper),
                                  ("table5", rp.sigma_lower, rp.sigma_upper, rp.nu_lower, rp.nu_upper)):
            m = nb - na
            rep[tag] = dict(interval=(a, b), length=b - a, index_range=(na + 1, nb), m=m,
                            gap=(b - a) / m if m > 0 else None)
        rep["table6"] = dict(m=rp.nu_upper - rp.nu_lower, bound=rp.s3_iter_bound, residual=rp.s3_iter_residual,
                             difference=rp.s3_iter_difference)
        ok = rp.status == KEP_OK
        return (lam.value if ok else None), (x if ok and not bisect_only else None), rep

    def perm(self) -> np.ndarray:
        p = np.empty(self.n, dtype=np.int64)
        self._check(lib().kep_get_perm(self._h, _ptr(p, C.c_int64)))
        return p

    def fronts(self):
        nf = self.analysis()["n_fronts"]
        first = np.empty(nf + 1, dtype=np.int64)
        parent = np.empty(nf, dtype=np.int64)
        order = np.empty(nf, dtype=np.int64)
        self._check(lib().kep_get_fronts(self._h, _ptr(first, C.c_int64), _ptr(parent, C.c_int64), _ptr(order, C.c_int64)))
        return first, parent, order


def tridiag_eigen(d, e):
    """kep_tridiag_eigen (testing hook): eigenvalues (ascending) and eigenvectors of tridiag(e, d, e)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    e = np.ascontiguousarray(e, dtype=np.float64)
    n = d.shape[0]
    assert e.shape == (max(n - 1, 0),)
    w = np.empty(n)
    Z = np.empty((n, n), order="F")
    ee = e if n > 1 else np.zeros(1)
    st = lib().kep_tridiag_eigen(n, _ptr(d, C.c_double), _ptr(ee, C.c_double), _ptr(w, C.c_double),
                                 _ptr(Z, C.c_double))
    if st != KEP_OK:
        raise KepError(st, "kep_tridiag_eigen")
    return w, Z


def version() -> str:
    return lib().kep_version().decode()


class Factor:
    """A kep_factorization: P (A - sigma B) P^T = L D L^T kept on the device."""

    def __init__(self, owner: Kep, handle):
        self._owner = owner            # keeps the ctx alive
        self._h = handle
        self.n = owner.n

    def close(self):
        if getattr(self, "_h", None):
            if getattr(self._owner, "_h", None):       # kep_destroy already released it otherwise
                lib().kep_factor_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        st = _FStats()
        r = lib().kep_factor_info(self._h, C.byref(st))
        if r != KEP_OK:
            raise KepError(r, "kep_factor_info")
        inf = InertiaInfo(*[getattr(st.inertia, f) for f, _ in _Info._fields_])
        return dict(sigma=st.sigma, nu=st.nu, inertia=inf, n=st.n, nnz_L=st.nnz_L, store_bytes=st.store_bytes)

    def solve(self, b):
        """x = (A - sigma B)^-1 b for b of shape (n,) or (n, nrhs) (host arrays)."""
        b = np.asarray(b, dtype=np.float64)
        one = b.ndim == 1
        B = np.asfortranarray(b.reshape(self.n, -1))
        X = np.empty_like(B, order="F")
        r = lib().kep_solve(self._h, B.shape[1], _ptr(B, C.c_double), self.n, _ptr(X, C.c_double), self.n)
        if r != KEP_OK:
            raise KepError(r, lib().kep_last_error(self._owner._h).decode())
        return X[:, 0] if one else X

    def solve_dev(self, b_ptr: int, x_ptr: int):
        """One right-hand side in device memory (enqueued on the ctx stream)."""
        r = lib().kep_solve_dev(self._h, C.c_void_p(b_ptr), C.c_void_p(x_ptr))
        if r != KEP_OK:
            raise KepError(r, lib().kep_last_error(self._owner._h).decode())

    def export(self):
        """(perm, d, dsub, Lcolptr, Lrowidx, Lval): P S P^T = L D L^T, L unit lower in CSC."""
        n = self.n
        perm = np.empty(n, np.int64)
        d = np.empty(n)
        ds = np.empty(n)
        cp = np.zeros(n + 1, np.int64)
        P = C.POINTER
        r = lib().kep_factor_export(self._h, _ptr(perm, C.c_int64), _ptr(d, C.c_double), _ptr(ds, C.c_double),
                                    _ptr(cp, C.c_int64), C.cast(None, P(C.c_int32)), C.cast(None, P(C.c_double)))
        if r != KEP_OK:
            raise KepError(r, lib().kep_last_error(self._owner._h).decode())
        ri = np.empty(int(cp[-1]), np.int32)
        vals = np.empty(int(cp[-1]))
        r = lib().kep_factor_export(self._h, _ptr(perm, C.c_int64), _ptr(d, C.c_double), _ptr(ds, C.c_double),
                                    _ptr(cp, C.c_int64), _ptr(ri, C.c_int32), _ptr(vals, C.c_double))
        if r != KEP_OK:
            raise KepError(r, lib().kep_last_error(self._owner._h).decode())
        return perm, d, ds, cp, ri, vals
