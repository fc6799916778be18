"""Pins for the oracle's temperature (D20), masked-vocabulary (D21) and
draft-entropy predictor (D22) extensions — SURVEY §8(f) f1 and f2.

* temperature: sampling at temperature T means p = softmax(t / T), q =
  softmax(d / T) (P:312 evaluates T = 0 and T = 1; per-sequence temperature,
  P:490). Pinned by exact rescaling (T = 2^k on fp32 inputs is an exact
  division, so verify(t, d, T) must equal verify(t / T, d / T, T = 1) bit for
  bit), the T -> 0 limit (the greedy mode, D18), the two-point closed form at
  temperature T, and by brute force: verify-then-resample at temperature T
  reproduces target autoregressive sampling at temperature T.
* masks: a -inf logit (top-k / top-p filtering) has probability 0. Pinned by
  the compacted row (identical masks in t and d: the masked columns are not
  there at all), KL = +inf when the draft masks a token the target keeps, a
  target-masked token is never emitted, and by brute force with independently
  masked target and draft tables.
* entropy predictor: closed forms of SL_H and its effect on SL^ (no pin
  retypes the formula: the values below are worked by hand from D22)."""
import numpy as np
import pytest
import scipy.special as sps

import oracle
import synth
from tests import spec_sim


def _batch(V, k, seed, sigma=3.0):
    r = np.random.default_rng(seed)
    B = len(k)
    cu = synth.cu_from_k(k)
    nk = int(cu[-1])
    t = r.normal(0, sigma, (nk + B, V)).astype(np.float32)
    d = (t[np.concatenate([[cu[i] + i + j for j in range(k[i])] for i in range(B)])]
         + r.normal(0, 0.7, (nk, V))).astype(np.float32)
    tok = r.integers(0, V, nk).astype(np.int32)
    seeds = synth.slot_seeds(seed, 0, cu)
    return cu, tok, t, d, seeds


def _same(a, b):
    for f in ("accepted_len", "emitted", "kld", "log_ratio", "u_acc", "u_smp", "flags"):
        x, y = getattr(a, f), getattr(b, f)
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8)), f


# ---------------------------------------------------------------- temperature


def test_temperature_one_is_the_default():
    k = synth.random_k(40, 6, 3)
    cu, tok, t, d, seeds = _batch(50, k, 1)
    a = oracle.verify(cu, tok, t, d, seeds, oracle.F32)
    b = oracle.verify(cu, tok, t, d, seeds, oracle.F32, temperature=np.ones(len(k)))
    _same(a, b)


@pytest.mark.parametrize("T", [0.5, 2.0, 4.0, 0.25])
def test_temperature_is_exact_rescaling(T):
    """T a power of two: t / T is exact in fp32, so the tempered verification
    equals the plain one on pre-divided logits, bit for bit."""
    k = synth.random_k(60, 6, 4)
    cu, tok, t, d, seeds = _batch(40, k, 2)
    a = oracle.verify(cu, tok, t, d, seeds, oracle.F32, temperature=np.full(len(k), T))
    b = oracle.verify(cu, tok, (t / np.float32(T)).astype(np.float32), (d / np.float32(T)).astype(np.float32),
                      seeds, oracle.F32)
    _same(a, b)


def test_temperature_to_zero_is_greedy():
    """Integer logits with distinct maxima (gaps >= 1): at T = 1e-3 every p and
    q is one-hot in fp64 (e^-1000 = 0), so the sampling verification must be
    the greedy one (D18): the same accepted lengths and tokens for any seed."""
    r = np.random.default_rng(5)
    V, B = 12, 200
    k = synth.random_k(B, 5, 6)
    cu = synth.cu_from_k(k)
    nk = int(cu[-1])

    def rows(n):
        x = np.stack([r.permutation(V) for _ in range(n)]).astype(np.float32)  # distinct integers
        return x
    t = rows(nk + B)
    d = rows(nk)
    # draft tokens: mostly the draft argmax (x ~ q at T -> 0 is the argmax),
    # and sometimes the target argmax, so accepts and rejects both occur
    tok = d.argmax(1).astype(np.int32)
    tgt = np.concatenate([[cu[i] + i + j for j in range(k[i])] for i in range(B)])
    flip = r.random(nk) < 0.5
    tok[flip] = t[tgt[flip]].argmax(1)
    d[np.arange(nk), tok] = V + 1.0  # x is the draft argmax (q(x) = 1 at T -> 0)
    seeds = synth.slot_seeds(3, 0, cu)
    g = oracle.verify(cu, tok, t, d, seeds, oracle.F32, greedy=True)
    s = oracle.verify(cu, tok, t, d, seeds, oracle.F32, temperature=np.full(B, 1e-3))
    assert np.array_equal(g.accepted_len, s.accepted_len)
    assert np.array_equal(g.emitted, s.emitted)
    assert 0 < np.mean(g.accepted_len == np.asarray(k)) < 1


def test_temperature_zero_marks_greedy_sequences():
    """T_i = 0 makes sequence i greedy, the others sample at their T."""
    k = synth.random_k(50, 5, 7)
    cu, tok, t, d, seeds = _batch(30, k, 8)
    T = np.where(np.arange(len(k)) % 3 == 0, 0.0, 0.7)
    m = oracle.verify(cu, tok, t, d, seeds, oracle.F32, temperature=T)
    g = oracle.verify(cu, tok, t, d, seeds, oracle.F32, greedy=True)
    s = oracle.verify(cu, tok, t, d, seeds, oracle.F32, temperature=np.full(len(k), 0.7))
    for i in range(len(k)):
        ref = g if T[i] == 0 else s
        s0, s1 = cu[i] + i, cu[i + 1] + i + 1
        assert m.accepted_len[i] == ref.accepted_len[i]
        assert np.array_equal(m.emitted[s0:s1], ref.emitted[s0:s1])
    # greedy sequences keep T = 1 KLDs (D18)
    plain = oracle.verify(cu, tok, t, d, seeds, oracle.F32)
    for i in np.nonzero(T == 0)[0]:
        assert np.array_equal(m.kld[cu[i]:cu[i + 1]], plain.kld[cu[i]:cu[i + 1]])


def test_two_point_kl_closed_form_at_temperature():
    """p = softmax((a, b) / T), q = softmax((c, e) / T): KL = P ln(P/Q) +
    (1-P) ln((1-P)/(1-Q)) with P = 1/(1 + exp((b - a)/T))."""
    vals = np.float32([[0.0, 1.5], [0.0, -2.0], [3.0, 0.0]])
    dv = np.float32([[0.5, 0.0], [1.0, 1.0], [0.0, 0.25]])
    for T in (0.3, 0.8, 1.7):
        for a, c in zip(vals, dv):
            t = np.stack([a, a]).astype(np.float32)
            d = c[None, :].astype(np.float32)
            r = oracle.verify(np.int32([0, 1]), np.int32([0]), t, d, np.uint64([1, 2]), oracle.F32,
                              temperature=np.float64([T]))
            P = 1.0 / (1.0 + np.exp((float(a[1]) - float(a[0])) / T))
            Q = 1.0 / (1.0 + np.exp((float(c[1]) - float(c[0])) / T))
            kl = P * np.log(P / Q) + (1 - P) * np.log((1 - P) / (1 - Q))
            assert abs(r.kld[0] - kl) <= 1e-14 + 1e-12 * kl


@pytest.mark.parametrize("T,seed", [(0.6, 31), (1.8, 32)])
def test_distribution_exact_bruteforce_at_temperature(T, seed):
    """Verify-then-resample at temperature T reproduces target autoregressive
    sampling at temperature T (V = 5, depth 3, 10^6 runs; S:584 at T)."""
    tab = spec_sim.Tables(5, 3, seed, temp=T)

    def fn(cu, tokens, target, draft, seeds):
        r = oracle.verify(cu, tokens, target, draft, seeds, oracle.F32, temperature=np.full(len(cu) - 1, T))
        return r.accepted_len, r.emitted
    codes = spec_sim.run_generation(tab, 10 ** 6, fn, seed)
    spec_sim.check_distribution(tab, codes)


# ---------------------------------------------------------------- masks


def test_masked_columns_equal_the_compacted_row():
    """The same -inf mask in t and d: the result equals verification over the
    kept columns only (tokens remapped), because masked tokens have p = q = 0."""
    r = np.random.default_rng(11)
    V, keepn = 40, 17
    k = synth.random_k(80, 5, 12)
    cu, tok, t, d, seeds = _batch(V, k, 13)
    B = len(k)
    tgt = np.concatenate([[cu[i] + i + j for j in range(k[i])] for i in range(B)])
    cols = np.sort(r.choice(V, keepn, replace=False))
    mask = np.ones(V, bool)
    mask[cols] = False
    tm, dm = t.copy(), d.copy()
    tm[:, mask] = -np.inf
    dm[:, mask] = -np.inf
    tok = cols[r.integers(0, keepn, tok.size)].astype(np.int32)  # drafted from q: a kept token
    full = oracle.verify(cu, tok, tm, dm, seeds, oracle.F32, temperature=np.full(B, 0.9))
    remap = -np.ones(V, np.int64)
    remap[cols] = np.arange(keepn)
    comp = oracle.verify(cu, remap[tok].astype(np.int32), np.ascontiguousarray(t[:, cols]),
                         np.ascontiguousarray(d[:, cols]), seeds, oracle.F32, temperature=np.full(B, 0.9))
    assert np.array_equal(full.accepted_len, comp.accepted_len)
    em = np.where(full.emitted >= 0, remap[np.maximum(full.emitted, 0)], -1)
    assert np.array_equal(em, comp.emitted)
    assert np.allclose(full.kld, comp.kld, rtol=1e-13, atol=1e-15)
    assert np.allclose(full.log_ratio, comp.log_ratio, rtol=1e-12, atol=1e-14)
    assert tgt.size == int(cu[-1])


def test_draft_masking_a_target_token_gives_infinite_kl():
    """q_v = 0 < p_v for some v: KL(p || q) = +inf (D1, D21); the other
    outputs stay finite and valid."""
    k = [3, 2, 4]
    cu, tok, t, d, seeds = _batch(20, k, 21)
    d2 = d.copy()
    d2[1, 7] = -np.inf   # draft row 1 (sequence 0, position 1) masks token 7
    tok = np.where(tok == 7, 8, tok).astype(np.int32)
    r = oracle.verify(cu, tok, t, d2, seeds, oracle.F32)
    assert np.isinf(r.kld[1]) and r.kld[1] > 0
    assert np.isfinite(np.delete(r.kld, 1)).all()
    assert np.isfinite(r.log_ratio).all()


def test_target_masked_tokens_are_never_emitted():
    """A token the target masks (p = 0) is rejected whenever drafted and never
    drawn (recovery from max(0, p - q), bonus from p)."""
    r = np.random.default_rng(22)
    V = 10
    k = synth.random_k(400, 4, 23)
    cu, tok, t, d, seeds = _batch(V, k, 24)
    masked = r.random(t.shape) < 0.4
    masked[:, 0] = False
    tm = t.copy()
    tm[masked] = -np.inf
    res = oracle.verify(cu, tok, tm, d, seeds, oracle.F32)
    B = len(k)
    for i in range(B):
        a = res.accepted_len[i]
        s0 = cu[i] + i
        for j in range(a):
            assert not masked[s0 + j, tok[cu[i] + j]]
        if a < k[i]:
            assert not masked[s0 + a, res.emitted[s0 + a]]
        else:
            assert not masked[s0 + k[i], res.emitted[s0 + k[i]]]
    drafted_masked = np.array([masked[cu[i] + i + j, tok[cu[i] + j]] for i in range(B) for j in range(k[i])])
    assert np.all(res.log_ratio[drafted_masked] == -np.inf)


@pytest.mark.parametrize("mt,md,T,seed", [(0.3, 0.0, 1.0, 41), (0.0, 0.3, 1.0, 42), (0.3, 0.3, 0.8, 43)])
def test_distribution_exact_bruteforce_with_masks(mt, md, T, seed):
    """Independently masked target and draft tables (and a temperature):
    verify-then-resample still reproduces target sampling exactly."""
    tab = spec_sim.Tables(6, 3, seed, mask_t=mt, mask_d=md, temp=T)

    def fn(cu, tokens, target, draft, seeds):
        r = oracle.verify(cu, tokens, target, draft, seeds, oracle.F32,
                          temperature=None if T == 1.0 else np.full(len(cu) - 1, T))
        return r.accepted_len, r.emitted
    codes = spec_sim.run_generation(tab, 10 ** 6, fn, seed)
    spec_sim.check_distribution(tab, codes)


def test_masked_draft_token_and_empty_rows_are_invalid():
    k = [2, 2]
    cu, tok, t, d, seeds = _batch(8, k, 51)
    d2 = d.copy()
    d2[0, tok[0]] = -np.inf   # q(x) = 0: x cannot have been drafted
    with pytest.raises(ValueError):
        oracle.verify(cu, tok, t, d2, seeds, oracle.F32)
    t2 = t.copy()
    t2[1, :] = -np.inf        # everything masked: not a distribution
    with pytest.raises(ValueError):
        oracle.verify(cu, tok, t2, d, seeds, oracle.F32)


# ---------------------------------------------------------------- f2: D22


def test_entropy_sl_closed_forms():
    # H = 0: alpha = 1 -> SL_max
    assert oracle.entropy_sl(0.0, 0.5, 8, 2) == (8, 8.0)
    # gamma H >= 1: alpha = 0 -> SL_min
    assert oracle.entropy_sl(2.0, 0.5, 8, 2)[0] == 2
    assert oracle.entropy_sl(10.0, 0.5, 8, 2)[0] == 2
    # gamma H = 1/4: alpha = 1/2 -> x = 0.5 * 6 + 2 = 5
    sl, x = oracle.entropy_sl(0.25, 1.0, 8, 2)
    assert sl == 5 and abs(x - 5.0) < 1e-15
    # gamma H = 0.09: alpha = 0.7 -> x = 6.2 -> 6 ; half-even at x = 6.5: alpha = 0.75
    assert oracle.entropy_sl(0.09, 1.0, 8, 2)[0] == 6
    assert oracle.entropy_sl(0.0625, 1.0, 8, 2) == (6, 6.5)  # rint(6.5) = 6 (half to even, D11)
    # monotone non-increasing in H
    hs = np.linspace(0, 3, 200)
    v = [oracle.entropy_sl(h, 0.7, 8, 2)[0] for h in hs]
    assert all(a >= b for a, b in zip(v, v[1:]))


def _signal_run(entropy_mode, ent_fn, steps=12, B=6, seed=3):
    r = np.random.default_rng(seed)
    cfg = oracle.Config(calib_steps=2, calib_sl=4, entropy_mode=entropy_mode, entropy_gamma=0.5)
    st = oracle.OracleState(cfg, B)
    out = []
    for s in range(steps):
        k = r.integers(1, 8, B)
        cu = synth.cu_from_k(k)
        kld = r.gamma(2.0, 0.05, int(cu[-1]))
        acc = np.minimum(k, r.integers(0, 8, B))
        sl, cal, _ = st.update_signal(np.arange(B), cu, kld, acc, entropy=ent_fn(int(cu[-1])))
        out.append((sl.copy(), cal.copy()))
    return out


def test_entropy_mode_min_with_the_kld_prediction():
    base = _signal_run(0, lambda n: None)
    zero = _signal_run(1, lambda n: np.zeros(n))           # H = 0: SL_H = SL_max >= SL^
    huge = _signal_run(1, lambda n: np.full(n, 100.0))     # SL_H = SL_min
    for (b, cb), (z, cz), (h, ch) in zip(base, zero, huge):
        assert np.array_equal(b, z) and np.array_equal(cb, cz)
        assert np.array_equal(np.where(ch == 1, b, 2), h)  # calibrating sequences keep calib_sl
    mid = _signal_run(1, lambda n: np.full(n, 0.18))       # alpha = 0.7, SL_H = rint(0.7 SL_span + 2)
    for (b, cb), (m, cm) in zip(base, mid):
        assert np.all(m <= b)
