"""Fits the polynomials used by the kernels for g(w) = exp(-w) - 1 + w.

g(w) = u^2 h(u), u = -w, h(u) = (e^u - 1 - u) / u^2 on |u| <= R. A Chebyshev
interpolant (degree 5 on R = 1/2 for the stream kernel, degree 7 on R = 1 for
the sampling kernel) (near-minimax) is converted to monomial form, rounded to
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


def fit(deg=7, R=1.0, n=200):
    x = R * np.cos(np.pi * (np.arange(n) + 0.5) / n)
    mono = Ch.cheb2poly(Ch.chebfit(x / R, h(x), deg))
    mono = (mono / R ** np.arange(deg + 1)).astype(np.float32)
    xs = np.linspace(-R, R, 200001)
    u = xs.astype(np.float32)
    p = np.float32(mono[-1])
    for c in mono[-2::-1]:
        p = (p * u + c).astype(np.float32)
    err = np.max(np.abs(p.astype(np.float64) - h(xs)) / h(xs))
    return mono, err


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--deg", type=int, default=7)
    ap.add_argument("--range", type=float, default=1.0)
    args = ap.parse_args()
    mono, err = fit(args.deg, args.range)
    print(f"coefficients (u^0 .. u^{args.deg}) on |u| <= {args.range}:", [repr(float(c)) for c in mono])
    print("max relative error (fp32 Horner):", err)
