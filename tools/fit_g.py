"""Fits the polynomial used by the verify kernel for g(w) = exp(-w) - 1 + w.

g(w) = u^2 h(u), u = -w, h(u) = (e^u - 1 - u) / u^2 on u in [-1, 1]. A degree-7
Chebyshev interpolant (near-minimax) is converted to monomial form, rounded to
fp32, and checked with fp32 Horner evaluation against an fp64 reference.
Prints the coefficients (lowest degree first) and the max relative error.
"""
import numpy as np
from numpy.polynomial import chebyshev as Ch


def h(u):
    u = np.asarray(u, dtype=np.float64)
    out = np.empty_like(u)
    small = np.abs(u) < 1e-3
    us = u[small]
    out[small] = 0.5 + us / 6 + us ** 2 / 24 + us ** 3 / 120 + us ** 4 / 720
    ul = u[~small]
    out[~small] = (np.expm1(ul) - ul) / ul ** 2
    return out


def fit(deg=7, n=200):
    x = np.cos(np.pi * (np.arange(n) + 0.5) / n)
    mono = Ch.cheb2poly(Ch.chebfit(x, h(x), deg)).astype(np.float32)
    xs = np.linspace(-1, 1, 200001)
    u = xs.astype(np.float32)
    p = np.float32(mono[-1])
    for c in mono[-2::-1]:
        p = (p * u + c).astype(np.float32)
    err = np.max(np.abs(p.astype(np.float64) - h(xs)) / h(xs))
    return mono, err


if __name__ == "__main__":
    mono, err = fit()
    print("coefficients (u^0 .. u^7):", [repr(float(c)) for c in mono])
    print("max relative error (fp32 Horner):", err)
