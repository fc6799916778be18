"""Draft entropy through the CUDA path: with
dsde_set_draft_entropy the stream kernel's opt-in variant also sums the draft's
own softmax per slice (Sd, E about the slice max of d), the finalize merges
them in fp64 and writes H(q) = log Sd - E / Sd per draft row. Compared element
by element with the oracle's definition -sum q log q (oracle.draft_entropy);
band |dH| <= 1e-5 H + 3e-7: relative to H, with an absolute floor (as the
KLD's 1e-9): the fp32 slice sums leave ~1e-7..3e-7 absolute in log Sd, and
near a one-hot draft the row max's slice rounds Sd = 1 + delta to 1, losing
log1p(delta) <= H / (1 + mean -ln q of the other tokens). The verify outputs must be bit-identical with and
without it."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity
from tests.gpu_util import dsde, gpu_verify, make_host_batch, oracle_verify, to_device_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    return dsde()


def _check_entropy(m, host, dtype, sharpen=None):
    dev = to_device_inputs(host, dtype)
    n = dev["draft_tokens"].numel()
    st0 = m.State(m.Config.default(), len(host["cu_sl"]) - 1)
    base = gpu_verify(m, st0, dev)
    st = m.State(m.Config.default(), len(host["cu_sl"]) - 1)
    ent = torch.full((n,), float("nan"), dtype=torch.float32, device="cuda")
    st.set_draft_entropy(ent)
    got = gpu_verify(m, st, dev)
    for a, b in zip(base[:3], got[:3]):
        assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    h_g = ent.cpu().numpy().astype(np.float64)
    h_o = oracle.draft_entropy(host["draft"], oracle.BF16 if dtype == torch.bfloat16 else oracle.F32)
    err = np.abs(h_g - h_o)
    assert np.all(np.isfinite(h_g))
    assert np.all(err <= 1e-5 * h_o + 3e-7), (np.max(err / (h_o + 1e-300)), h_o[np.argmax(err)], np.max(err))
    rep = parity.compare_verify(host["cu_sl"], got[0], got[1], got[2], oracle_verify(host))
    assert rep.ok(), str(rep)
    return h_o


@pytest.mark.parametrize("V,dtype,kmax,B", [
    (128256, torch.bfloat16, 8, 10), (32000, torch.bfloat16, 8, 24), (32000, torch.float32, 4, 8),
    (50000, torch.bfloat16, 8, 6), (8193, torch.float32, 16, 4), (1003, torch.bfloat16, 3, 7),
    (3, torch.bfloat16, 1, 16),
])
def test_draft_entropy_parity(m, V, dtype, kmax, B):
    k = synth.random_k(B, kmax, V + 5 * B)
    for prof in (("code",), ("dialogue", "low")):
        host = make_host_batch(V, k, seed=V * 3 + B, dtype=dtype, profiles=prof)
        _check_entropy(m, host, dtype)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_draft_entropy_flat_and_peaked_rows(m, dtype):
    """H near log V (flat draft) and near 0 (one dominant draft logit)."""
    r = np.random.default_rng(11)
    V, B, k = 32000, 4, 3
    cu = synth.cu_from_k(np.full(B, k))
    t = (r.standard_normal((B * k + B, V)) * 4).astype(np.float32)
    d = (r.standard_normal((B * k, V)) * 0.01).astype(np.float32)      # nearly uniform
    d[::2] = (r.standard_normal((d[::2].shape[0], V)) * 1.0).astype(np.float32)
    d[::2, 5] += 40.0                                                      # one-hot-like
    if dtype == torch.bfloat16:
        t = (t.view(np.uint32) >> 16).astype(np.uint16)
        d = (d.view(np.uint32) >> 16).astype(np.uint16)
    host = dict(cu_sl=cu, target=t, draft=d, draft_tokens=r.integers(0, V, B * k).astype(np.int32),
                seeds=synth.slot_seeds(9, 0, cu))
    h = _check_entropy(m, host, dtype)
    assert h[1] > np.log(V) - 0.01 and h[0] < 1e-10


def test_draft_entropy_in_dsde_step(m):
    """The whole-step launch (dsde_step) writes the same entropies."""
    B, V = 16, 32000
    k = synth.random_k(B, 8, 99)
    host = make_host_batch(V, k, seed=77)
    dev = to_device_inputs(host, torch.bfloat16)
    n = int(np.sum(k))
    st = m.State(m.Config.default(), B)
    step = m.Step(st, B, V, torch.bfloat16)
    ent = torch.zeros(n, dtype=torch.float32, device="cuda")
    st.set_draft_entropy(ent)
    step(dev["cu_sl"], dev["draft_tokens"], dev["target"], dev["draft"], dev["seeds"], n)
    torch.cuda.synchronize()
    h_o = oracle.draft_entropy(host["draft"], oracle.BF16)
    assert np.all(np.abs(ent.cpu().numpy() - h_o) <= 1e-5 * h_o + 3e-7)
    st.set_draft_entropy(None)
    ent.zero_()
    step(dev["cu_sl"], dev["draft_tokens"], dev["target"], dev["draft"], dev["seeds"], n)
    torch.cuda.synchronize()
    assert float(ent.abs().sum()) == 0.0  # off: nothing written
