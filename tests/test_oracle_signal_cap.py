"""Pins for the oracle's adapter (C2: Eq.1-8) and cap (C3: Eq.9-11).

Pins: the worked examples printed in SPEC.md (tests/golden/spec_examples.txt),
numpy's population variance (delta = 1), translation invariance, a weighted
Welford (West 1979) recurrence written independently of the two-pass form,
closed-form windows, Eq.8 branch boundaries, and an exhaustive MSE grid
search for the cap."""
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _examples():
    out = []
    with open(os.path.join(GOLD, "spec_examples.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, inp, exp, tol, cite = [x.strip() for x in line.split("|")]
            out.append((name, inp, float(exp), float(tol), cite))
    return out


def _kv(inp):
    d = {}
    for tok in inp.split():
        k, v = tok.split("=")
        d[k] = v
    return d


@pytest.mark.parametrize("name,inp,exp,tol,cite", _examples())
def test_spec_examples(name, inp, exp, tol, cite):
    a = _kv(inp) if "=" in inp else {}
    if name == "kld_two_point":
        got = oracle.row_kld(np.float64([0.0, 0.0]), np.log([0.25, 0.75]))
    elif name == "kld_identity":
        t = np.random.default_rng(0).normal(0, 3, 100)
        got = oracle.row_kld(t, t)
    elif name == "sf":
        got = oracle.scale_factor(float(a["mu"]))
    elif name == "wvar":
        got = oracle.weighted_variance(eval(a["v"]), float(a["delta"]))
    elif name == "calibrate":
        got = oracle.calibrate(int(a["sl_a_max"]), float(a["mu"]), float(a["max"]))[0]
    elif name == "calibrate_raw":
        got = oracle.calibrate(int(a["sl_a_max"]), float(a["mu"]), float(a["max"]))[1]
    elif name == "cap":
        sl = eval(a["sl"])
        cfg = oracle.Config(sl_min=1)
        got = oracle.next_sl(cfg, sl, [0] * len(sl))[1]
    elif name == "predict":
        got = oracle.predict_sl(float(a["penalty"]), int(a["sl_max"]))[0]
    elif name.startswith("uniform_seed"):
        got = oracle.uniforms(int(a["seed"]))[0]
    else:
        raise AssertionError(name)
    assert abs(got - exp) <= tol, (name, got, exp, cite)


def test_weighted_variance_delta1_is_population_variance():
    r = np.random.default_rng(1)
    for n in (1, 2, 5, 30):
        v = r.normal(0, 2, n)
        assert abs(oracle.weighted_variance(v, 1.0) - np.var(v)) <= 1e-12 * max(1, np.var(v))


def test_weighted_variance_translation_invariance():
    r = np.random.default_rng(2)
    v = r.uniform(0, 1, 30)
    a = oracle.weighted_variance(v, 0.85)
    b = oracle.weighted_variance(v + 3.0, 0.85)
    assert abs(a - b) <= 1e-12


def _west(values_recent_first, delta):
    """Weighted incremental mean/variance (D.H.D. West, CACM 22(9), 1979):
    an independent recurrence, not the two-pass Eq.7."""
    wsum = 0.0
    mean = 0.0
    s = 0.0
    for i, x in enumerate(values_recent_first):
        w = delta ** i
        wsum_new = wsum + w
        q = x - mean
        r = q * w / wsum_new
        mean += r
        s += wsum * q * r
        wsum = wsum_new
    return s / wsum


def test_weighted_variance_matches_west_recurrence():
    r = np.random.default_rng(3)
    for _ in range(300):
        n = int(r.integers(1, 31))
        v = r.exponential(0.3, n)
        dl = float(r.uniform(0.05, 1.0))
        a = oracle.weighted_variance(v, dl)
        b = _west(v, dl)
        assert abs(a - b) <= 1e-12 * max(abs(a), 1e-300) + 1e-300


def test_weighted_variance_closed_windows():
    """30 alternating {0.1, 0.9}: short = long = 0.158948137 -> WVIR 1;
    20 alternating then 10 x 0.5: short 0, long 0.0304735594."""
    alt = [0.1 if i % 2 == 0 else 0.9 for i in range(30)]
    recent = alt[::-1]
    s = oracle.weighted_variance(recent[:10], 0.85)
    l = oracle.weighted_variance(recent[:30], 0.85)
    assert abs(s - 0.158948137) < 1e-9 and abs(l - 0.158948137) < 1e-9
    hist = [0.1 if i % 2 == 0 else 0.9 for i in range(20)] + [0.5] * 10
    recent = hist[::-1]
    assert oracle.weighted_variance(recent[:10], 0.85) == 0.0
    assert abs(oracle.weighted_variance(recent, 0.85) - 0.0304735594) < 1e-9


def test_scale_factor_identities():
    """SF = 1 <=> mu = ln2/2 (Eq.3); SF monotone increasing."""
    assert abs(oracle.scale_factor(math.log(2) / 2) - 1.0) < 1e-15
    xs = np.linspace(0, 3, 200)
    sf = [oracle.scale_factor(x) for x in xs]
    assert all(b > a for a, b in zip(sf, sf[1:]))


def test_predict_values_and_branches():
    """WVIR = 1, SL_max = 8, SL_min = 2: mu 0.05 -> 7.368974 -> 7; 0.1 ->
    6.671583 -> 7; 0.2 -> 5.049052 -> 5; Eq.8 branches."""
    for mu, x_exp, sl_exp in [(0.05, 7.368974, 7), (0.1, 6.671583, 7), (0.2, 5.049052, 5)]:
        sl, x = oracle.predict_sl(oracle.scale_factor(mu), 8)
        assert sl == sl_exp and abs(x - x_exp) < 1e-6
    assert oracle.predict_sl(1.0, 8)[0] == 2
    assert oracle.predict_sl(1.0 + 1e-12, 8)[0] == 2
    assert oracle.predict_sl(0.0, 8)[0] == 8
    # rint is half-to-even: x = 2.5 -> 2, 3.5 -> 4
    assert oracle.predict_sl(1 - 0.5 / 6, 8)[0] == 2
    assert oracle.predict_sl(1 - 1.5 / 6, 8)[0] == 4
    # monotone non-increasing in mu_last
    prev = 99
    for mu in np.linspace(0, 2, 400):
        sl = oracle.predict_sl(oracle.scale_factor(mu), 8)[0]
        assert 2 <= sl <= 8 and sl <= prev
        prev = sl


def test_calibrate_edges():
    """mu = max -> ~2 SL_A,max; SL_A,max = 0 -> sl_min + 1; clamp."""
    assert oracle.calibrate(3, 0.4, 0.4)[0] == 6
    assert oracle.calibrate(0, 0.4, 0.9)[0] == 3
    assert oracle.calibrate(6, 0.4, 0.4, sl_ceiling=8)[0] == 8
    assert oracle.calibrate(1, 0.0, 0.4)[0] == 3  # clamp up to sl_min + 1


def _mse(c, x):
    return np.mean((c - np.asarray(x, dtype=np.float64)) ** 2)


def test_cap_is_mse_argmin_grid_search():
    """for 10^4 random vectors (B = 2..64) the cap attains the minimum
    Eq.9 MSE over all integer candidates in [sl_min, max]."""
    r = np.random.default_rng(5)
    cfg = oracle.Config()
    for _ in range(10_000):
        B = int(r.integers(2, 65))
        sl = r.integers(2, 9, B)
        _, cap = oracle.next_sl(cfg, sl, np.zeros(B, np.int32))
        best = min(_mse(c, sl) for c in range(2, int(sl.max()) + 1))
        assert abs(_mse(cap, sl) - best) <= 1e-12
        assert abs(cap - sl.mean()) <= 0.5


def test_cap_half_even_and_application():
    cfg = oracle.Config()
    assert oracle.next_sl(cfg, [2, 3], [0, 0])[1] == 2
    assert oracle.next_sl(cfg, [3, 4], [0, 0])[1] == 4
    nxt, cap = oracle.next_sl(cfg, [8, 2, 6, 4], [0, 0, 0, 1], budget=[9, 9, 1, 9])
    # calibrating sequence (last) is excluded from the mean and keeps calib_sl
    assert cap == 5 and list(nxt) == [5, 2, 1, 4]
    cfg0 = oracle.Config(cap_mode=0)
    nxt, cap = oracle.next_sl(cfg0, [8, 2], [0, 0])
    assert cap == 8 and list(nxt) == [8, 2]


def test_cap_partition_invariance():
    """Exact integer partials: any split into ranks gives the same cap."""
    r = np.random.default_rng(6)
    cfg = oracle.Config()
    for _ in range(200):
        B = int(r.integers(8, 200))
        sl = r.integers(2, 9, B).astype(np.int32)
        cal = (r.random(B) < 0.1).astype(np.int32)
        _, cap = oracle.next_sl(cfg, sl, cal)
        for n in (2, 4, 8):
            parts = [oracle.cap_partial(sl[j::n], cal[j::n]) for j in range(n)]
            s = sum(p[0] for p in parts)
            m = sum(p[1] for p in parts)
            if m == 0:
                continue
            q, rem = divmod(s, m)
            if 2 * rem > m or (2 * rem == m and q % 2 == 1):
                q += 1
            assert q == cap


def test_signal_closed_loop_examples():
    """observe/predict through the state: calibration (Eq.1) then Eq.8;
    ring capacity; warm-up WVIR = 1 (D9); flat history (D10)."""
    cfg = oracle.Config(calib_steps=2, calib_sl=4)
    st = oracle.OracleState(cfg, 4)
    slots = np.arange(2, dtype=np.int32)
    cu = np.int32([0, 3, 6])
    # step 1: calibrating
    kld = np.array([0.1, 0.2, 0.3, 0.05, 0.05, 0.05])
    sl, cal, dg = st.update_signal(slots, cu, kld, np.int32([2, 3]))
    assert list(sl) == [4, 4] and list(cal) == [1, 1]
    # step 2: calibration ends -> SL_max (Eq.1) and a real prediction
    kld2 = np.array([0.1, 0.1, 0.1, 0.05, 0.05, 0.05])
    sl, cal, dg = st.update_signal(slots, cu, kld2, np.int32([3, 3]))
    assert list(cal) == [0, 0]
    mu0 = (0.1 + 0.2 + 0.3 + 0.3) / 6
    expect0, _ = oracle.calibrate(3, mu0, 0.3, sl_ceiling=8)
    assert dg[0, 7] == expect0
    # seq 1: constant history 0.05 -> SL_max = rint(3 * (1 + .05/.050001)) = 6,
    # 6 observations < n_short -> WVIR = 1, penalty = SF(0.05)
    assert dg[1, 7] == 6 and dg[1, 4] == 1.0
    x = (1 - oracle.scale_factor(0.05)) * (6 - 2) + 2
    assert abs(dg[1, 6] - x) < 1e-12 and sl[1] == round(x)
    # many constant steps -> flat history guard keeps WVIR = 1
    for _ in range(10):
        sl, cal, dg = st.update_signal(slots, cu, kld2, np.int32([3, 3]))
    assert dg[1, 4] == 1.0 and dg[1, 3] < 1e-12


def test_signal_window_unit_step_means():
    cfg = oracle.Config(calib_steps=1, window_unit=1, n_short=2, n_long=4)
    st = oracle.OracleState(cfg, 1)
    means = []
    r = np.random.default_rng(8)
    for s in range(6):
        k = int(r.integers(1, 6))
        kl = r.exponential(0.2, k)
        means.append(kl.mean())
        sl, cal, dg = st.update_signal(np.int32([0]), np.int32([0, k]), kl, np.int32([k]))
    recent = means[::-1]
    vs = oracle.weighted_variance(recent[:2], 0.85)
    vl = oracle.weighted_variance(recent[:4], 0.85)
    assert abs(dg[0, 2] - vs) < 1e-15 and abs(dg[0, 3] - vl) < 1e-15
    assert abs(dg[0, 4] - vs / vl) < 1e-12
