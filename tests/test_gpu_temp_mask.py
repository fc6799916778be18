"""Per-sequence temperature (D20), masked vocabularies (D21) and the
draft-entropy SL predictor (D22) through the CUDA path — SURVEY §8(f) f1/f2 —
against the fp64 oracle on the same inputs (bands of tests/parity.py; an
infinite KLD must be infinite on both sides)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity, spec_sim
from tests.gpu_util import dsde, gpu_verify, make_host_batch, to_device_inputs

pytestmark = pytest.mark.gpu

NEG_INF_BF16 = np.uint16(0xFF80)


@pytest.fixture(scope="module")
def m():
    return dsde()


def _vals(x):
    return (x.astype(np.uint32) << 16).view(np.float32) if x.dtype == np.uint16 else x


def _set_inf(x, mask):
    x = x.copy()
    if x.dtype == np.uint16:
        x[mask] = NEG_INF_BF16
    else:
        x[mask] = -np.inf
    return x


def _topk_mask(vals, keep, rng, frac=1.0):
    """True where a top-k filter removes the token (rows chosen with prob frac)."""
    n, V = vals.shape
    thr = -np.sort(-vals, axis=1)[:, keep - 1:keep]
    m = vals < thr
    m[rng.random(n) >= frac] = False
    return m


def _redraw_tokens(host, temps, rng):
    """x ~ q at the sequence's temperature over the draft's unmasked tokens
    (the harness stand-in for the draft model; Gumbel-max)."""
    cu = host["cu_sl"]
    d = _vals(host["draft"]).astype(np.float64)
    toks = host["draft_tokens"].copy()
    for i in range(cu.size - 1):
        T = 1.0 if temps is None or temps[i] == 0 else float(temps[i])
        for j in range(cu[i + 1] - cu[i]):
            row = d[cu[i] + j] / T
            g = row - np.log(-np.log(rng.random(row.size)))
            toks[cu[i] + j] = int(np.argmax(g))
    h = dict(host)
    h["draft_tokens"] = toks.astype(np.int32)
    return h


def _masked_host(V, k, seed, mode, keep, dtype=torch.bfloat16, profiles=("code", "low"), temps=None):
    host = make_host_batch(V, k, seed, dtype=dtype, profiles=profiles)
    rng = np.random.default_rng(seed + 1)
    cu = host["cu_sl"]
    B = cu.size - 1
    t, d = host["target"], host["draft"]
    tv, dv = _vals(t), _vals(d)
    draft_of_target = np.full(t.shape[0], -1)
    for i in range(B):
        for j in range(cu[i + 1] - cu[i]):
            draft_of_target[cu[i] + i + j] = cu[i] + j
    if mode in ("same", "target", "both"):
        mt = _topk_mask(tv, keep, rng, 0.8)
        t = _set_inf(t, mt)
        if mode == "same":
            md = np.zeros(d.shape, bool)
            has = draft_of_target >= 0
            md[draft_of_target[has]] = mt[has]
            d = _set_inf(d, md)
    if mode in ("draft", "both"):
        d = _set_inf(d, _topk_mask(dv, keep, rng, 0.8))
    h = dict(host)
    h["target"], h["draft"] = t, d
    return _redraw_tokens(h, temps, rng)


def _oracle(host, temps=None, greedy=False, resample=oracle.RESAMPLE_FULL):
    dt = oracle.BF16 if host["target"].dtype == np.uint16 else oracle.F32
    return oracle.verify(host["cu_sl"], host["draft_tokens"], host["target"], host["draft"], host["seeds"],
                         dt, nthreads=8, greedy=greedy,
                         temperature=None if temps is None else np.asarray(temps, np.float64), resample=resample)


def _check(m, st, host, dtype, temps=None):
    dev = to_device_inputs(host, dtype)
    tt = None if temps is None else torch.from_numpy(np.asarray(temps, np.float32)).cuda()
    st.set_temperature(tt)
    acc, em, kl, _ = gpu_verify(m, st, dev)
    st.set_temperature(None)
    o = _oracle(host, temps, resample=st.cfg.resample)
    rep = parity.compare_verify(host["cu_sl"], acc, em, kl, o)
    assert rep.ok(), str(rep)
    assert st.device_error() == (0, -1)
    return rep, kl, o


TEMPS = np.float32([0.0, 0.4, 0.7, 1.0, 1.3, 2.0])


@pytest.mark.parametrize("V,dtype,kmax,B", [
    (32000, torch.bfloat16, 8, 64), (8193, torch.float32, 6, 40), (128256, torch.bfloat16, 8, 12),
    (1003, torch.bfloat16, 3, 30),
])
@pytest.mark.parametrize("resample", [1, 0])
def test_temperature_parity(m, V, dtype, kmax, B, resample):
    st = m.State(m.Config.default(resample=resample), 4096)
    k = synth.random_k(B, kmax, V % 97)
    temps = np.random.default_rng(V).choice(TEMPS, B)
    host = _redraw_tokens(make_host_batch(V, k, 5 + V % 13, dtype=dtype, profiles=("code", "dialogue")), temps,
                          np.random.default_rng(1))
    rep, _, _ = _check(m, st, host, dtype, temps)
    print(rep)


def test_temperature_one_is_bit_identical(m):
    st = m.State(m.Config.default(), 512)
    k = synth.random_k(48, 8, 3)
    host = make_host_batch(32000, k, 9)
    dev = to_device_inputs(host, torch.bfloat16)
    a = gpu_verify(m, st, dev)
    st.set_temperature(torch.ones(48, dtype=torch.float32, device="cuda"))
    b = gpu_verify(m, st, dev)
    st.set_temperature(None)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


@pytest.mark.parametrize("mode", ["same", "target", "draft", "both"])
@pytest.mark.parametrize("V,dtype,keep", [(32000, torch.bfloat16, 40), (8193, torch.float32, 500),
                                          (128256, torch.bfloat16, 2000)])
@pytest.mark.parametrize("with_temp,resample", [(False, 1), (True, 1), (True, 0)])
def test_masked_parity(m, mode, V, dtype, keep, with_temp, resample):
    st = m.State(m.Config.default(masked=1, resample=resample), 4096)
    B = 24 if V > 100000 else 48
    k = synth.random_k(B, 6, len(mode) + V % 7)
    temps = np.random.default_rng(B + len(mode)).choice(TEMPS, B) if with_temp else None
    host = _masked_host(V, k, 30 + len(mode), mode, keep, dtype=dtype, temps=temps)
    rep, kl, o = _check(m, st, host, dtype, temps)
    if mode in ("draft", "both"):
        assert np.isinf(o.kld).any() and np.array_equal(np.isinf(kl), np.isinf(o.kld))
    print(mode, rep)


def test_masked_config_matches_plain_path_without_masks(m):
    """masked = 1 on finite logits gives the same decisions (KLD within the band)."""
    k = synth.random_k(64, 8, 4)
    host = make_host_batch(32000, k, 12)
    a = gpu_verify(m, m.State(m.Config.default(), 64), to_device_inputs(host, torch.bfloat16))
    b = gpu_verify(m, m.State(m.Config.default(masked=1), 64), to_device_inputs(host, torch.bfloat16))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.all(np.abs(a[2] - b[2]) <= 2e-5 * np.abs(a[2]) + 1e-9)


@pytest.mark.parametrize("mt,md,T,resample", [(0.3, 0.3, 0.8, 1), (0.4, 0.0, 1.0, 1), (0.3, 0.3, 0.8, 0)])
def test_masked_bruteforce_gpu(m, mt, md, T, resample):
    """Verify-then-resample through the CUDA path with masked tables (and a
    temperature) reproduces target sampling: chi^2 and TV; both
    recovery-draw readings."""
    st = m.State(m.Config.default(masked=1, resample=resample), 1)
    tab = spec_sim.Tables(6, 3, 77, mask_t=mt, mask_d=md, temp=T)

    def fn(cu, tokens, target, draft, seeds):
        host = dict(cu_sl=cu, draft_tokens=tokens, target=target, draft=draft, seeds=seeds)
        dev = to_device_inputs(host, torch.float32)
        B = cu.size - 1
        st.set_temperature(None if T == 1.0 else torch.full((B,), T, dtype=torch.float32, device="cuda"))
        acc, em, _, _ = gpu_verify(m, st, dev, with_flags=False)
        st.set_temperature(None)
        return acc, em
    codes = spec_sim.run_generation(tab, 10 ** 6, fn, 77)
    spec_sim.check_distribution(tab, codes)
    assert st.device_error() == (0, -1)


def test_bad_temperature_and_masked_draft_token_are_device_errors(m):
    st = m.State(m.Config.default(masked=1), 64)
    k = np.array([2, 3, 2])
    host = _masked_host(1024, k, 3, "draft", 100)
    d = host["draft"].copy()
    x = host["draft_tokens"][2]  # sequence 1, position 0: mask the drafted token in the draft
    d[2, x] = NEG_INF_BF16
    h = dict(host)
    h["draft"] = d
    st.set_temperature(torch.tensor([1.0, 1.0, -1.0], device="cuda"))
    acc, em, kl, _ = gpu_verify(m, st, to_device_inputs(h, torch.bfloat16))
    st.set_temperature(None)
    assert acc[0] >= 0 and acc[1] == -1 and acc[2] == -1
    code, _ = st.device_error()
    assert code in (2, 3)


# ---------------------------------------------------------------- whole step


def test_step_with_temperature_and_entropy_mode(m):
    """dsde_step with per-sequence temperatures and the D22
    entropy predictor: identical to the three separate calls (bit for bit), and
    SL^ equal to the oracle's signal fed with the GPU's own fp32 KLDs and
    draft entropies (outside 1e-9 rint ties)."""
    B, V = 64, 32000
    kw = dict(calib_steps=2, calib_sl=4, entropy_mode=1, entropy_gamma=0.5)
    ga, gb = m.Config.default(masked=0, **kw), m.Config.default(masked=0, **kw)
    sa, sb = m.State(ga, B), m.State(gb, B)
    pa, pb = m.Step(sa, B, V, torch.bfloat16, with_diag=True), m.Step(sb, B, V, torch.bfloat16, with_diag=True)
    ea = torch.empty(B * 16, dtype=torch.float32, device="cuda")
    eb = torch.empty(B * 16, dtype=torch.float32, device="cuda")
    sa.set_draft_entropy(ea)
    sb.set_draft_entropy(eb)
    temps = torch.from_numpy(np.random.default_rng(1).choice(TEMPS[1:], B).astype(np.float32)).cuda()
    sa.set_temperature(temps)
    sb.set_temperature(temps)
    ost = oracle.OracleState(oracle.Config(**kw), B)
    w = synth.Workload(B=B, V=V, dtype=torch.bfloat16, profiles=("code", "dialogue"), seed=91)
    k = np.full(B, 4, dtype=np.int64)
    ties = 0
    for s in range(12):
        inp = synth.generate_step(w, s, k, device="cuda")
        n = int(k.sum())
        oa = pa(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n)
        ob = pb(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n, fused=False)
        torch.cuda.synchronize()
        for x, y in ((oa.accepted_len, ob.accepted_len), (oa.emitted, ob.emitted), (oa.sl_hat, ob.sl_hat),
                     (oa.next_sl, ob.next_sl), (oa.cap, ob.cap), (ea[:n], eb[:n])):
            assert torch.equal(x, y)
        assert torch.equal(oa.kld.view(torch.int32), ob.kld.view(torch.int32))
        cu = inp.cu_sl.cpu().numpy()
        sl_o, cal_o, dg_o = ost.update_signal(np.arange(B), cu, oa.kld.cpu().numpy().astype(np.float64),
                                              oa.accepted_len.cpu().numpy(),
                                              entropy=ea[:n].cpu().numpy().astype(np.float64))
        sl_g = oa.sl_hat.cpu().numpy()
        for i in np.nonzero(sl_g != sl_o)[0]:
            assert abs((dg_o[i, 6] % 1.0) - 0.5) < 1e-9, (s, i)
            ties += 1
        k = oa.next_sl.cpu().numpy().astype(np.int64)
    assert ties <= 2
    assert sa.device_error() == (0, -1)


def test_entropy_mode_requires_the_draft_entropy(m):
    st = m.State(m.Config.default(entropy_mode=1), 8)
    step = m.Step(st, 8, 1024, torch.bfloat16)
    w = synth.Workload(B=8, V=1024, dtype=torch.bfloat16, seed=2)
    inp = synth.generate_step(w, 0, np.full(8, 2), device="cuda")
    with pytest.raises(m.DsdeError):
        step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, 16)
