"""T = 0 (greedy) verification through the CUDA path (dsde_config.greedy = 1;
SURVEY §8(f) f1, D18) against the fp64 oracle's greedy mode: accepted lengths
and emitted tokens bit-exact (argmax decisions have no tie band: equal maxima
resolve to the smallest token id on both sides), KLDs within the D16 band.
Integer-valued logits make equal maxima frequent; bonus rows exercise the
argmax draw pass."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity
from tests.gpu_util import dsde, gpu_verify, make_host_batch, to_device_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    return dsde()


@pytest.fixture(scope="module")
def gstate(m):
    return m.State(m.Config.default(greedy=1), 4096)


def _oracle_greedy(host, nthreads=8):
    dt = oracle.BF16 if host["target"].dtype == np.uint16 else oracle.F32
    return oracle.verify(host["cu_sl"], host["draft_tokens"], host["target"], host["draft"], host["seeds"],
                         dt, nthreads=nthreads, greedy=True)


def _check(m, st, host, dtype):
    acc, em, kl, _ = gpu_verify(m, st, to_device_inputs(host, dtype))
    o = _oracle_greedy(host)
    assert np.array_equal(acc, o.accepted_len), (acc, o.accepted_len)
    assert np.array_equal(em, o.emitted)
    err = np.abs(kl.astype(np.float64) - o.kld)
    assert np.all(err <= parity.KL_REL * np.abs(o.kld) + parity.KL_ABS)
    assert st.device_error() == (0, -1)
    return acc, o


def _argmax_drafts(host, frac, seed):
    """Replace a fraction of draft tokens by their row's target argmax (the
    smallest index of the maximum) so that long accepted runs occur."""
    r = np.random.default_rng(seed)
    cu = host["cu_sl"]
    toks = host["draft_tokens"].copy()
    t = host["target"]
    tv = (t.astype(np.uint32) << 16).view(np.float32) if t.dtype == np.uint16 else t
    for i in range(cu.size - 1):
        for j in range(cu[i + 1] - cu[i]):
            if r.random() < frac:
                row = tv[cu[i] + i + j]
                toks[cu[i] + j] = int(np.flatnonzero(row == row.max())[0])
    h = dict(host)
    h["draft_tokens"] = toks
    return h


@pytest.mark.parametrize("V,dtype,kmax,B", [
    (32000, torch.float32, 4, 8), (32000, torch.bfloat16, 8, 64), (128256, torch.bfloat16, 8, 12),
    (50000, torch.bfloat16, 8, 9), (1003, torch.bfloat16, 3, 7), (8193, torch.float32, 16, 5),
    (300007, torch.bfloat16, 3, 6),
    (2, torch.float32, 2, 16), (3, torch.bfloat16, 1, 16),
])
def test_greedy_parity(m, gstate, V, dtype, kmax, B):
    k = synth.random_k(B, kmax, V + 3 * B)
    host = make_host_batch(V, k, seed=V + B, dtype=dtype, profiles=("code", "low"))
    acc, o = _check(m, gstate, _argmax_drafts(host, 0.85, V), dtype)
    if B >= 32:  # both the bonus-argmax draw and the recovery path ran
        assert (acc == k).any() and (acc < k).any()


def test_greedy_ties_smallest_id(m, gstate):
    """Integer-valued logits: most rows have several equal maxima."""
    r = np.random.default_rng(5)
    B, V = 24, 3000
    k = synth.random_k(B, 6, 9)
    cu = synth.cu_from_k(k)
    nk = int(cu[-1])
    t = r.integers(-4, 5, (nk + B, V)).astype(np.float32)
    d = r.integers(-4, 5, (nk, V)).astype(np.float32)
    host = dict(cu_sl=cu, target=t, draft=d, draft_tokens=r.integers(0, V, nk).astype(np.int32),
                seeds=synth.slot_seeds(3, 0, cu))
    _check(m, gstate, _argmax_drafts(host, 0.9, 6), torch.float32)
    tb = dict(host, target=(t.view(np.uint32) >> 16).astype(np.uint16),
              draft=(d.view(np.uint32) >> 16).astype(np.uint16))
    _check(m, gstate, _argmax_drafts(tb, 0.9, 7), torch.bfloat16)


def test_greedy_full_size_step(m):
    """Config-3 shape through dsde_step with greedy = 1: the whole batch against
    the oracle's greedy mode, then the signal / cap run on the greedy KLDs."""
    B, V = 96, 128256
    cfg = m.Config.default(greedy=1)
    st = m.State(cfg, B)
    step = m.Step(st, B, V, torch.bfloat16)
    k = synth.random_k(B, 8, 21)
    host = make_host_batch(V, k, seed=21, profiles=("code",))
    host = _argmax_drafts(host, 0.9, 21)
    dev = to_device_inputs(host, torch.bfloat16)
    out = step(dev["cu_sl"], dev["draft_tokens"], dev["target"], dev["draft"], dev["seeds"], int(k.sum()))
    torch.cuda.synchronize()
    o = _oracle_greedy(host)
    assert np.array_equal(out.accepted_len.cpu().numpy(), o.accepted_len)
    assert np.array_equal(out.emitted.cpu().numpy(), o.emitted)
    assert st.device_error() == (0, -1)
