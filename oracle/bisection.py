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
