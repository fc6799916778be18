"""Pins for the oracle's verify (C1): accept test, first rejection, residual /
bonus inverse-CDF sample and the emitted-token layout.

The decisive pin is distributional: verify-then-resample must reproduce exact
target autoregressive sampling (brute force over all strings).
The rest are special cases the texts spell out and invariants
(S:145-147)."""
import numpy as np
import pytest
import scipy.special as sps

import oracle
import synth
from tests import spec_sim


def oracle_verify_fn(cu, tokens, target, draft, seeds, resample=oracle.RESAMPLE_FULL):
    r = oracle.verify(cu, tokens, target, draft, seeds, oracle.F32, resample=resample)
    return r.accepted_len, r.emitted


@pytest.mark.parametrize("V,L,seed,resample", [(4, 3, 11, 0), (8, 3, 12, 0), (2, 3, 13, 0),
                                               (8, 3, 14, 1), (4, 3, 15, 1)])
def test_distribution_exact_bruteforce(V, L, seed, resample):
    """S:584 acceptance #1: V <= 8, depth 3, 10^6 runs, TV <= 0.01 and chi^2,
    for both readings of the recovery draw (D23 proposals, D7 inverse CDF)."""
    tab = spec_sim.Tables(V, L, seed)
    codes = spec_sim.run_generation(
        tab, 10 ** 6, lambda *a: oracle_verify_fn(*a, resample=resample), seed)
    spec_sim.check_distribution(tab, codes)


def test_proposal_uniforms_are_philox_counter_j():
    """D23's uniforms: Philox4x32-10 at counter (j, 0, 0, 0) (KAT-pinned), res53 of
    words 0-1 and 2-3; counter 0 is D6's (u_acc, u_smp)."""
    for seed in (0, 1, 0xDEADBEEFCAFEF00D):
        key = [seed & 0xFFFFFFFF, seed >> 32]
        assert oracle.proposal_uniforms(seed, 0) == oracle.uniforms(seed)
        for j in (1, 2, 31, 32):
            w = [int(x) for x in oracle.philox4x32_10([j, 0, 0, 0], key)]
            r53 = lambda a, b: ((a >> 5) * 67108864.0 + (b >> 6)) / 9007199254740992.0
            assert oracle.proposal_uniforms(seed, j) == (r53(w[0], w[1]), r53(w[2], w[3]))


@pytest.mark.parametrize("seed", [41, 42])
def test_proposal_draw_reimplemented(seed):
    """D23 pinned by an independent re-implementation of every recovery draw:
    scipy softmax for p and q, numpy cumsum + searchsorted for each proposal
    v_j (smallest v with C_v > u_prop P), keep iff u_keep < max(0, p - q)_v / p_v,
    the first kept proposal is the token; none kept in 256 -> the D7 draw
    (flagged)."""
    V = 29
    k = np.array([1, 2, 3, 4, 2, 1, 3, 4] * 6)
    cu, tok, t, d, seeds = _batch(V, k, seed)
    d = (t[np.concatenate([np.arange(cu[i], cu[i + 1]) + i for i in range(len(k))])] +
         np.random.default_rng(seed).normal(0, 1.0, (int(cu[-1]), V))).astype(np.float32)
    r = np.random.default_rng(seed + 1)
    tok = np.array([r.choice(V, p=qq) for qq in sps.softmax(d.astype(np.float64), axis=1)], dtype=np.int32)
    res = oracle.verify(cu, tok, t, d, seeds, oracle.F32, resample=oracle.RESAMPLE_PROPOSAL)
    n_res = 0
    for i in range(len(k)):
        a, s0 = int(res.accepted_len[i]), int(cu[i]) + i
        if a == k[i]:
            continue
        n_res += 1
        p = sps.softmax(t[s0 + a].astype(np.float64))
        q = sps.softmax(d[cu[i] + a].astype(np.float64))
        c = np.cumsum(p)
        want = None
        for j in range(1, oracle.PROPOSALS + 1):
            up, uk = oracle.proposal_uniforms(int(seeds[s0 + a]), j)
            v = int(np.searchsorted(c, up * c[-1], side="right"))
            if uk < max(0.0, p[v] - q[v]) / p[v]:
                want = v
                break
        if want is None:
            assert res.flags[s0 + a] & oracle.FLAG_PROPOSAL_FALLBACK
            w = np.maximum(0.0, p - q)
            cw = np.cumsum(w)
            want = int(np.searchsorted(cw, res.u_smp[s0 + a] * cw[-1], side="right"))
        else:
            assert not (res.flags[s0 + a] & oracle.FLAG_PROPOSAL_FALLBACK)
        assert res.emitted[s0 + a] == want, (i, a)
    assert n_res > 20


def test_proposal_fallback_rate_is_one_minus_tv_to_the_k():
    """A proposal v ~ p is kept with probability sum_v p_v max(0, p_v - q_v) / p_v
    = TV(p, q), so all 256 proposals fail with probability (1 - TV)^256 (closed
    form; TV = 0.0033 here); the D7 draw then takes over (flag)."""
    t = np.float32([[0.0, 0.2, -0.3, 0.1, 0.4]])
    d = np.float32([[0.01, 0.19, -0.29, 0.1, 0.395]])
    p = sps.softmax(t[0].astype(np.float64))
    q = sps.softmax(d[0].astype(np.float64))
    tv = 0.5 * np.abs(p - q).sum()
    x = int(np.argmax(q / p))  # a token with p < q: rejected unless u < p/q
    B = 60000
    cu = np.arange(B + 1, dtype=np.int32)
    res = oracle.verify(cu, np.full(B, x, np.int32), np.repeat(t, 2 * B, axis=0), np.repeat(d, B, axis=0),
                        synth.slot_seeds(7, 0, cu), oracle.F32, nthreads=8, resample=oracle.RESAMPLE_PROPOSAL)
    rej_i = np.nonzero(res.accepted_len == 0)[0]
    rej = rej_i.size
    fb = int(np.sum((res.flags[2 * rej_i] & oracle.FLAG_PROPOSAL_FALLBACK) != 0))
    assert np.all(p[res.emitted[2 * rej_i]] > q[res.emitted[2 * rej_i]])   # only residual-support tokens
    want = (1 - tv) ** oracle.PROPOSALS
    sd = np.sqrt(want * (1 - want) / rej)
    assert 0.05 < want < 0.95 and rej > 300
    assert abs(fb / rej - want) < 5 * sd


def test_first_position_rejection_rate_is_tv():
    """P(reject at position 0) = 1 - sum_v min(p_v, q_v) = TV(p, q) when
    x ~ q (rejection sampling)."""
    tab = spec_sim.Tables(6, 2, 21, sigma_n=1.2)
    n = 400_000
    rec = {}

    def keep(cu, tokens, acc, emitted):
        rec["acc"] = acc.copy()

    spec_sim.run_generation(tab, n, oracle_verify_fn, 21, k_max=1, record_first=keep)
    tv = 0.5 * np.abs(tab.P[0] - tab.Q[0]).sum()
    rate = np.mean(rec["acc"] == 0)
    sd = np.sqrt(tv * (1 - tv) / n)
    assert abs(rate - tv) < 5 * sd


def _batch(V, k, seed, dtype=np.float32, same=False):
    r = np.random.default_rng(seed)
    B = len(k)
    cu = synth.cu_from_k(k)
    nk = int(cu[-1])
    t = r.normal(0, 3, (nk + B, V)).astype(dtype)
    if same:
        d = np.stack([t[cu[i] + i + j] for i in range(B) for j in range(k[i])]) if nk else t[:0]
    else:
        d = (r.normal(0, 3, (nk, V))).astype(dtype)
    tok = r.integers(0, V, nk).astype(np.int32)
    seeds = synth.slot_seeds(seed, 0, cu)
    return cu, tok, t, d, seeds


def test_draft_equals_target_accepts_all_and_bonus_follows_p():
    """draft == target -> accepted_count == k always; the bonus token is
    then distributed as p of target row k."""
    k = [3, 1, 4, 2] * 50
    cu, tok, t, d, seeds = _batch(16, k, 3, same=True)
    r = oracle.verify(cu, tok, t, d, seeds, oracle.F32)
    assert (r.accepted_len == np.asarray(k)).all()
    assert np.all(r.log_ratio == 0.0)
    assert np.all(r.kld == 0.0)
    # bonus row draws: same target row repeated, many seeds -> frequencies ~ p
    V, n = 5, 200_000
    row = np.float32([0.0, 1.0, -0.5, 2.0, 0.3])
    t = np.tile(row, (2 * n, 1))
    d = np.tile(row, (n, 1))
    cu1 = synth.cu_from_k(np.ones(n, np.int64))
    s = synth.slot_seeds(99, 0, cu1)
    r = oracle.verify(cu1, np.zeros(n, np.int32), t, d, s, oracle.F32)
    assert (r.accepted_len == 1).all()
    bonus = r.emitted[1::2]
    freq = np.bincount(bonus, minlength=V) / n
    p = sps.softmax(row.astype(np.float64))
    assert np.max(np.abs(freq - p)) < 5 * np.sqrt(p * (1 - p) / n).max()


def test_disjoint_one_hot_rejects_and_recovers_target_token():
    """draft one-hot at x, target one-hot at x' -> a = 0, token x'."""
    V = 8
    n = 64
    t = np.full((2 * n, V), -1e4, np.float32)
    d = np.full((n, V), -1e4, np.float32)
    t[0::2, 5] = 0.0
    t[1::2, :] = 0.0
    d[:, 2] = 0.0
    cu = synth.cu_from_k(np.ones(n, np.int64))
    r = oracle.verify(cu, np.full(n, 2, np.int32), t, d, synth.slot_seeds(7, 0, cu), oracle.F32)
    assert (r.accepted_len == 0).all()
    assert (r.emitted[0::2] == 5).all()
    assert (r.emitted[1::2] == -1).all()


def test_worked_example_v2():
    """t=(0,0), d=(0, ln 3) [fp32], x=1: r = 2/3 (up to fp32 rounding of ln 3);
    residual (0.25, 0) -> recovery is token 0. seed 0: u_acc=0.399 < 2/3 ->
    accept; seed 1: u_acc=0.890 -> reject -> token 0."""
    t = np.float32([[0.0, 0.0], [0.0, 0.0]])
    d = np.float32([[0.0, np.log(3.0)]])
    cu = np.int32([0, 1])
    tok = np.int32([1])
    r0 = oracle.verify(cu, tok, t, d, np.uint64([0, 5]), oracle.F32)
    assert abs(np.exp(r0.log_ratio[0]) - 2 / 3) < 1e-7
    assert r0.accepted_len[0] == 1 and r0.emitted[0] == 1
    for mode in (oracle.RESAMPLE_PROPOSAL, oracle.RESAMPLE_FULL):
        # token 0 is the only token with p > q: both readings must recover it
        r1 = oracle.verify(cu, tok, t, d, np.uint64([1, 5]), oracle.F32, resample=mode)
        assert r1.accepted_len[0] == 0 and r1.emitted[0] == 0 and r1.emitted[1] == -1
        if mode == oracle.RESAMPLE_FULL:
            assert abs(r1.samp_diag[0, 0] - 0.25) < 1e-7   # residual mass R = TV = 1/4
        else:
            assert abs(r1.samp_diag[0, 0] - 1.0) < 1e-7    # D23: the proposals' mass, sum p = 1
            assert not (r1.flags[0] & oracle.FLAG_PROPOSAL_FALLBACK)


def test_prefix_shape_and_layout():
    """emitted = accepted prefix + exactly one token + pads;
    KLD at every position."""
    k = synth.random_k(300, 8, 5)
    cu, tok, t, d, seeds = _batch(50, k, 6)
    r = oracle.verify(cu, tok, t, d, seeds, oracle.F32)
    for i in range(len(k)):
        a = r.accepted_len[i]
        s0 = cu[i] + i
        assert 0 <= a <= k[i]
        assert (r.emitted[s0:s0 + a] == tok[cu[i]:cu[i] + a]).all()
        assert 0 <= r.emitted[s0 + a] < 50
        assert (r.emitted[s0 + a + 1:s0 + k[i] + 1] == -1).all()
        acc = r.u_acc[s0:s0 + k[i]] < np.minimum(1, np.exp(r.log_ratio[cu[i]:cu[i] + k[i]]))
        first = np.argmin(acc) if not acc.all() else k[i]
        assert first == a
    assert np.all(r.kld > 0)


def test_accepted_len_invariant_to_tokens_after_rejection():
    """changing draft tokens after the first rejection changes nothing."""
    k = synth.random_k(200, 6, 8, k_min=2)
    cu, tok, t, d, seeds = _batch(30, k, 9)
    r = oracle.verify(cu, tok, t, d, seeds, oracle.F32)
    tok2 = tok.copy()
    for i in range(len(k)):
        a = r.accepted_len[i]
        for j in range(a + 1, k[i]):
            tok2[cu[i] + j] = (tok2[cu[i] + j] + 7) % 30
    r2 = oracle.verify(cu, tok2, t, d, seeds, oracle.F32)
    assert (r.accepted_len == r2.accepted_len).all()
    for i in range(len(k)):
        s0 = cu[i] + i
        a = r.accepted_len[i]
        assert (r.emitted[s0:s0 + a + 1] == r2.emitted[s0:s0 + a + 1]).all()


def test_bf16_matches_fp32_on_exact_values():
    """bf16 patterns convert exactly: integer-valued logits give identical results."""
    k = [2, 3, 1]
    r = np.random.default_rng(10)
    cu = synth.cu_from_k(k)
    nk = int(cu[-1])
    t = r.integers(-8, 8, (nk + 3, 40)).astype(np.float32)
    d = r.integers(-8, 8, (nk, 40)).astype(np.float32)
    tok = r.integers(0, 40, nk).astype(np.int32)
    s = synth.slot_seeds(1, 1, cu)

    def bf(x):
        return (x.view(np.uint32) >> 16).astype(np.uint16)

    a = oracle.verify(cu, tok, t, d, s, oracle.F32)
    b = oracle.verify(cu, tok, bf(t), bf(d), s, oracle.BF16)
    assert (a.emitted == b.emitted).all() and np.array_equal(a.kld, b.kld)


def test_multithreaded_identical():
    k = synth.random_k(64, 8, 3)
    cu, tok, t, d, seeds = _batch(100, k, 4)
    a = oracle.verify(cu, tok, t, d, seeds, oracle.F32, nthreads=1)
    b = oracle.verify(cu, tok, t, d, seeds, oracle.F32, nthreads=7)
    assert (a.emitted == b.emitted).all() and np.array_equal(a.kld, b.kld)


def test_invalid_inputs_raise():
    cu = np.int32([0, 1])
    t = np.zeros((2, 4), np.float32)
    d = np.zeros((1, 4), np.float32)
    with pytest.raises(ValueError):
        oracle.verify(cu, np.int32([9]), t, d, np.uint64([0, 1]), oracle.F32)


# ---------------------------------------------------------------- f1: T = 0 ---
def test_greedy_worked_example_and_tie_break():
    """T = 0 verification: accept iff x_j is the target
    argmax; the first mismatch (or the bonus row) emits the target argmax; equal
    maxima resolve to the smallest token id (D18)."""
    V = 5
    cu = np.int32([0, 2])
    t = np.float32([[0, 3, 1, 3, 2], [5, 1, 1, 1, 1], [0, 0, 0, 9, 0]])
    d = np.float32([[1, 1, 1, 1, 1], [0, 0, 0, 0, 0]])
    seeds = np.uint64([1, 2, 3])
    r = oracle.verify(cu, np.int32([1, 0]), t, d, seeds, oracle.F32, greedy=True)
    assert r.accepted_len.tolist() == [2] and r.emitted.tolist() == [1, 0, 3]
    r = oracle.verify(cu, np.int32([3, 0]), t, d, seeds, oracle.F32, greedy=True)  # 3 ties with 1: rejected
    assert r.accepted_len.tolist() == [0] and r.emitted.tolist() == [1, -1, -1]


def test_greedy_emits_the_target_argmax_sequence():
    """The defining property of greedy speculative decoding, by brute force on
    random batches: emitted[0..a] = argmax of target rows 0..a, every accepted
    draft token equals its row's argmax and the first rejected one does not;
    independent of the seeds; KLDs identical to the sampling mode."""
    r = np.random.default_rng(18)
    for trial in range(40):
        B, V = int(r.integers(1, 6)), int(r.integers(2, 40))
        k = r.integers(1, 6, B)
        cu = np.concatenate([[0], np.cumsum(k)]).astype(np.int32)
        nk = int(cu[-1])
        # small integer logits make ties frequent
        t = r.integers(-3, 4, (nk + B, V)).astype(np.float32)
        d = r.integers(-3, 4, (nk, V)).astype(np.float32)
        am = lambda row: int(np.flatnonzero(row == row.max())[0])
        toks = np.empty(nk, np.int32)
        for i in range(B):
            for j in range(k[i]):
                row = t[cu[i] + i + j]
                toks[cu[i] + j] = am(row) if r.random() < 0.7 else int(r.integers(0, V))
        s1 = r.integers(0, 2**63, nk + B, dtype=np.uint64)
        s2 = r.integers(0, 2**63, nk + B, dtype=np.uint64)
        g1 = oracle.verify(cu, toks, t, d, s1, oracle.F32, greedy=True)
        g2 = oracle.verify(cu, toks, t, d, s2, oracle.F32, greedy=True)
        smp = oracle.verify(cu, toks, t, d, s1, oracle.F32)
        assert np.array_equal(g1.accepted_len, g2.accepted_len) and np.array_equal(g1.emitted, g2.emitted)
        assert np.array_equal(g1.kld, smp.kld)
        for i in range(B):
            a, s0 = int(g1.accepted_len[i]), cu[i] + i
            for j in range(a):
                assert toks[cu[i] + j] == am(t[s0 + j]) == g1.emitted[s0 + j]
            if a < k[i]:
                assert toks[cu[i] + a] != am(t[s0 + a])
            assert g1.emitted[s0 + a] == am(t[s0 + a])
            assert (g1.emitted[s0 + a + 1:s0 + k[i] + 1] == -1).all()


@pytest.mark.parametrize("seed", [31, 32, 33])
def test_sample_diag_edges_pinned_full(seed):
    """The oracle's samp_diag (R, lo, hi) — the CDF edges the sample tie band of
    D16 is measured against — pinned by an independent inverse CDF: weights from
    scipy softmax (max(0, p - q) for a recovery draw, p for a bonus draw),
    numpy's sequential cumsum, and np.searchsorted for the smallest v with
    C_v > u R (D7)."""
    k = np.array([1, 2, 3, 4, 2, 1, 3, 4] * 4)
    cu, tok, t, d, seeds = _batch(37, k, seed)
    d = (t[np.concatenate([np.arange(cu[i], cu[i + 1]) + i for i in range(len(k))])] +
         np.random.default_rng(seed).normal(0, 0.7, (int(cu[-1]), 37))).astype(np.float32)
    # draft tokens ~ q so that both recovery and bonus draws occur
    r = np.random.default_rng(seed + 1)
    q_all = sps.softmax(d.astype(np.float64), axis=1)
    tok = np.array([r.choice(37, p=qq) for qq in q_all], dtype=np.int32)
    res = oracle.verify(cu, tok, t, d, seeds, oracle.F32)
    n_res = n_bonus = 0
    for i in range(len(k)):
        a, ki, s0 = int(res.accepted_len[i]), int(k[i]), int(cu[i]) + i
        p = sps.softmax(t[s0 + a].astype(np.float64))
        if a < ki:
            w = np.maximum(0.0, p - sps.softmax(d[cu[i] + a].astype(np.float64)))
            n_res += 1
        else:
            w = p
            n_bonus += 1
        c = np.cumsum(w)
        R, lo, hi = res.samp_diag[i]
        u = res.u_smp[s0 + a]
        v = int(np.searchsorted(c, u * c[-1], side="right"))
        assert res.emitted[s0 + a] == v
        assert abs(R - c[-1]) <= 1e-12 * c[-1]
        assert abs(lo - (c[v - 1] / c[-1] if v else 0.0)) <= 1e-12
        assert abs(hi - c[v] / c[-1]) <= 1e-12
        assert lo <= u < hi
    assert n_res > 0 and n_bonus > 0
