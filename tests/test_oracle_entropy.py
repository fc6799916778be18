"""Pins of the oracle's draft entropy H(q) = -sum q log q, q = softmax(d)
(the paper's optional entropy signal), against
what fixes it independently of its code: closed forms, a library routine and
invariants."""
import math

import numpy as np
import pytest
import scipy.special
import scipy.stats

import oracle


@pytest.mark.parametrize("V", [1, 2, 7, 1000, 128256])
def test_uniform_is_log_v(V):
    # fp64 summation of V equal terms: relative error <= V u (u = 2^-53)
    assert oracle.row_entropy(np.full(V, 3.25)) == pytest.approx(math.log(V), rel=V * 1.2e-16 + 1e-14, abs=1e-15)


@pytest.mark.parametrize("a,b", [(0.0, 0.0), (1.0, -2.5), (7.0, 0.0), (-30.0, 5.0), (0.001, 0.0)])
def test_two_point_closed_form(a, b):
    p = 1.0 / (1.0 + math.exp(b - a))
    h = -sum(x * math.log(x) for x in (p, 1.0 - p) if x > 0.0)
    assert oracle.row_entropy(np.array([a, b])) == pytest.approx(h, rel=1e-12, abs=1e-15)


def test_matches_scipy_entropy_of_softmax():
    r = np.random.default_rng(3)
    for V, sigma in [(50, 1.0), (32000, 6.0), (32000, 0.3), (4096, 20.0)]:
        d = r.standard_normal(V) * sigma
        ref = scipy.stats.entropy(scipy.special.softmax(d))
        assert oracle.row_entropy(d) == pytest.approx(ref, rel=1e-10, abs=1e-13)


def test_one_hot_limit_and_bounds():
    d = np.full(1000, -2000.0)
    d[17] = 0.0
    assert oracle.row_entropy(d) == 0.0
    r = np.random.default_rng(4)
    for _ in range(20):
        V = int(r.integers(2, 3000))
        h = oracle.row_entropy(r.standard_normal(V) * r.uniform(0.1, 10))
        assert 0.0 <= h <= math.log(V) + 1e-12


def test_shift_invariance():
    r = np.random.default_rng(5)
    d = r.standard_normal(5000) * 4
    assert oracle.row_entropy(d + 1234.5) == pytest.approx(oracle.row_entropy(d), rel=1e-11)


def test_batch_rows_bf16_and_fp32():
    r = np.random.default_rng(6)
    d32 = (r.standard_normal((5, 777)) * 5).astype(np.float32)
    got = oracle.draft_entropy(d32, oracle.F32)
    for i in range(5):
        assert got[i] == oracle.row_entropy(d32[i].astype(np.float64))
    bf = (d32.view(np.uint32) >> 16).astype(np.uint16)
    dec = (bf.astype(np.uint32) << 16).view(np.float32)
    got = oracle.draft_entropy(bf, oracle.BF16)
    for i in range(5):
        assert got[i] == oracle.row_entropy(dec[i].astype(np.float64))
