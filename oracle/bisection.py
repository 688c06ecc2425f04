"""Spectral bisection, Alg. 1 and Alg. 1'.

Alg. 1: repeat until sigma_u - sigma_l < tau:
          sigma := (sigma_l + sigma_u)/2 ; nu := nu_sigma(A, B) ;
          if k <= nu: sigma_u := sigma else sigma_l := sigma
        return (sigma_l + sigma_u)/2, |lambda_hat - lambda_k| < tau/2.
Alg. 1': same step, stop when nu_u - nu_l <= m_max (nu_u, nu_l tracked).

``nu`` is any callable sigma -> nu_sigma(A, B).  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations


def bisect_alg1(nu, k: int, lo: float, hi: float, tau: float):
    it = 0
    while not (hi - lo < tau):
        sigma = (lo + hi) / 2.0
        if k <= nu(sigma):
            hi = sigma
        else:
            lo = sigma
        it += 1
    return (lo + hi) / 2.0, it, (lo, hi)


def bisect_alg1p(nu, k: int, lo: float, hi: float, nu_lo: int, nu_hi: int, m_max: int = 20,
                 max_iter: int = 128):
    it = 0
    trace = []
    while not (nu_hi - nu_lo <= m_max) and it < max_iter:
        sigma = (lo + hi) / 2.0
        v = nu(sigma)
        if k <= v:
            hi, nu_hi = sigma, v
        else:
            lo, nu_lo = sigma, v
        it += 1
        trace.append((sigma, v))
    return (lo, hi, nu_lo, nu_hi), it, trace


def brent_nu(nu, k: int, lo: float, hi: float, nu_lo: int, nu_hi: int, m_max: int = 20,
             max_iter: int = 128):
    """Brent's method on the step function nu ("as long as the
    algorithms are derivative-free and a root is bracketed ... Brent's method").

    The root of g(sigma) = nu_sigma - k + 1/2 is lambda_k: g < 0 for sigma <= lambda_k, g > 0 above
    (nu counts eigenvalues strictly below sigma).  Brent's "zero" algorithm as published
    (R. P. Brent, Algorithms for Minimization without Derivatives, 1973, ch. 4): b is the latest
    iterate and [b, c] brackets the root; the step is the secant (a == c) or inverse quadratic
    interpolation through (a, b, c), accepted only when it lands inside 3/4 of the way to c and
    shrinks faster than the step before last, otherwise the midpoint (bisection).  The stopping rule
    is Alg. 1' line 1: nu_u - nu_l <= m_max.  Returns ((lo, hi, nu_lo, nu_hi),
    iterations, trace of (sigma, nu))."""
    eps = 2.0 ** -52
    a, b, c = lo, hi, lo
    fa, fb = nu_lo - k + 0.5, nu_hi - k + 0.5
    fc = fa
    na, nb, nc = nu_lo, nu_hi, nu_lo
    d = e = b - a
    it = 0
    trace = []
    while True:
        if abs(fc) < abs(fb):
            a, b, c = b, c, b
            fa, fb, fc = fb, fc, fb
            na, nb, nc = nb, nc, nb
        lo, hi = min(b, c), max(b, c)
        nu_lo, nu_hi = (nb, nc) if b < c else (nc, nb)
        if nu_hi - nu_lo <= m_max or it >= max_iter:
            break
        tol = 2.0 * eps * abs(b)
        m = 0.5 * (c - b)
        if abs(e) >= tol and abs(fa) > abs(fb):
            s = fb / fa
            if a == c:
                p = 2.0 * m * s
                q = 1.0 - s
            else:
                q = fa / fc
                r = fb / fc
                p = s * (2.0 * m * q * (q - r) - (b - a) * (r - 1.0))
                q = (q - 1.0) * (r - 1.0) * (s - 1.0)
            if p > 0.0:
                q = -q
            else:
                p = -p
            if 2.0 * p < min(3.0 * m * q - abs(tol * q), abs(e * q)):
                e = d
                d = p / q
            else:
                d = e = m
        else:
            d = e = m
        a, fa, na = b, fb, nb
        b = b + (d if abs(d) > tol else (tol if m > 0.0 else -tol))
        nb = nu(b)
        fb = nb - k + 0.5
        it += 1
        trace.append((b, nb))
        if (fb > 0.0) == (fc > 0.0):
            c, fc, nc = a, fa, na
            d = e = b - a
    return (lo, hi, nu_lo, nu_hi), it, trace
