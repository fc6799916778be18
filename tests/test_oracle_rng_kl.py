"""Pins for the oracle's RNG (C0) and per-row KL / log-ratio (C1 steps 1-3).

Each pin is independent of the oracle's own formula: published KAT vectors,
closed forms, a library routine (scipy), or a mathematical invariant.
"""
import os

import numpy as np
import pytest
import scipy.special as sps

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kat_rows():
    rows = []
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            w = [int(x, 16) for x in line.split()]
            rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat_rows())
def test_philox_kat(ctr, key, out):
    """Random123 kat_vectors (tests/golden/philox4x32_10_kat.txt)."""
    assert list(oracle.philox4x32_10(ctr, key)) == out


def test_res53_range_and_resolution():
    # res53 maps onto the 2^-53 grid of [0,1): extremes and one mid value.
    assert oracle.res53(0, 0) == 0.0
    assert oracle.res53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0 ** -53
    assert oracle.res53(0x80000000, 0) == 0.5


def test_uniforms_golden():
    """seed -> (key = (lo32, hi32), ctr = 0): seed 0 is KAT row 1 (D6)."""
    ua, us = oracle.uniforms(0)
    assert ua == 0.39904647231489565
    ua1, _ = oracle.uniforms(1)
    assert ua1 == 0.89025917570803093
    # the 2nd uniform of seed 0 comes from KAT row 1 words 2-3
    w = _kat_rows()[0][2]
    assert us == oracle.res53(w[2], w[3])


def test_uniforms_distribution():
    u = np.array([oracle.uniforms(s)[0] for s in range(20000)])
    assert 0.0 <= u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.01
    # KS distance against U[0,1)
    us = np.sort(u)
    ks = np.max(np.abs(us - np.arange(1, us.size + 1) / us.size))
    assert ks < 0.015


def _rng(seed):
    return np.random.default_rng(seed)


def test_kl_identity_is_exactly_zero():
    """KL(p||p) = 0 exactly."""
    r = _rng(0)
    for V in (2, 7, 1000):
        t = r.normal(0, 5, V)
        assert oracle.row_kld(t, t) == 0.0


def test_kl_nonnegative_gibbs():
    """Gibbs' inequality: KL >= 0 on random rows."""
    r = _rng(1)
    for _ in range(200):
        V = int(r.integers(2, 300))
        t = r.normal(0, r.uniform(0.1, 8), V)
        d = r.normal(0, r.uniform(0.1, 8), V)
        assert oracle.row_kld(t, d) >= 0.0


def test_kl_two_point_closed_form():
    """Two-point closed form a ln(a/b) + (1-a) ln((1-a)/(1-b)), evaluated on
    the fp32-rounded logits; S:47 prints 0.143841 for ([.5,.5],[.25,.75])."""
    t = np.float32([0.0, 0.0]).astype(np.float64)
    d = np.float32([np.log(0.25), np.log(0.75)]).astype(np.float64)
    a = 0.5
    b = 1.0 / (1.0 + np.exp(d[1] - d[0]))  # q_0 from the rounded logits
    closed = a * np.log(a / b) + (1 - a) * np.log((1 - a) / (1 - b))
    kl = oracle.row_kld(t, d)
    assert abs(kl - closed) < 1e-15
    assert abs(kl - 0.143841) < 5e-7


def test_kl_uniform_target_closed_form():
    """p uniform: KL = -ln V - mean(d) + LSE(d), with LSE from scipy."""
    r = _rng(2)
    for V in (3, 64, 4096):
        d = r.normal(0, 3, V)
        t = np.full(V, 1.25)
        expect = -np.log(V) - d.mean() + sps.logsumexp(d)
        assert abs(oracle.row_kld(t, d) - expect) <= 1e-12 * max(1.0, abs(expect))


def test_kl_against_scipy_rel_entr():
    """Library routine: sum(rel_entr(softmax(t), softmax(d)))."""
    r = _rng(3)
    for _ in range(50):
        V = int(r.integers(2, 2000))
        t = r.normal(0, r.uniform(0.5, 7), V)
        d = t + r.normal(0, r.uniform(0.01, 2), V)
        ref = np.sum(sps.rel_entr(sps.softmax(t), sps.softmax(d)))
        assert abs(oracle.row_kld(t, d) - ref) <= 1e-10 * max(ref, 1e-6)


def test_kl_shift_invariance():
    """Adding an exactly representable constant to a whole row changes nothing
    (integer-valued logits + 8.0 are exact in fp64)."""
    r = _rng(4)
    t = r.integers(-20, 20, 500).astype(np.float64)
    d = r.integers(-20, 20, 500).astype(np.float64)
    base = oracle.row_kld(t, d)
    assert abs(oracle.row_kld(t + 8.0, d) - base) <= 1e-14 * base
    assert abs(oracle.row_kld(t, d - 8.0) - base) <= 1e-14 * base


def test_log_ratio_against_scipy():
    r = _rng(5)
    for _ in range(50):
        V = int(r.integers(2, 500))
        t = r.normal(0, 4, V)
        d = r.normal(0, 4, V)
        x = int(r.integers(0, V))
        ref = sps.log_softmax(t)[x] - sps.log_softmax(d)[x]
        assert abs(oracle.row_log_ratio(t, d, x) - ref) < 1e-12 * max(1, abs(ref))
