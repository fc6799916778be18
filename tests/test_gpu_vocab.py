"""Vocabulary-parallel verification (include/dsde.h dsde_vp_*)
through the CUDA path: the logit columns split over n shards, the stages run
in one process with the exchanges as device reductions (VocabParallel.run_local)
and through dsde_vp_verify (NCCL, one rank). The vp stages implement the D7
recovery draw (dsde_config.resample = DSDE_RESAMPLE_FULL). The outputs must be bit-identical
to the unsharded dsde_verify — accepted lengths, emitted tokens, KLD bits,
flags — and within the D16 bands of the oracle."""
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


def _shard(x: torch.Tensor, v0: int, v1: int) -> torch.Tensor:
    """Columns [v0, v1) of every row as their own tensor, rows 16-byte aligned."""
    esz = x.element_size()
    w = v1 - v0
    ld = w + (-(w * esz) % 16) // esz
    out = torch.zeros((x.shape[0], ld), dtype=x.dtype, device=x.device)
    out[:, :w] = x[:, v0:v1]
    return out


def _run_vp(m, st, host, dtype, n):
    dev = to_device_inputs(host, dtype)
    V = dev["V"]
    vp = m.VocabParallel(st, V, n, dtype)
    sl = vp.shard_slices()
    ts = [_shard(dev["target"][:, :V], a, b) for a, b in sl]
    ds = [_shard(dev["draft"][:, :V], a, b) for a, b in sl]
    B = dev["cu_sl"].numel() - 1
    nk = dev["draft_tokens"].numel()
    acc = torch.full((B,), -7, dtype=torch.int32, device="cuda")
    em = torch.full((nk + B,), -7, dtype=torch.int32, device="cuda")
    kl = torch.full((nk,), float("nan"), dtype=torch.float32, device="cuda")
    fl = torch.zeros(nk + B, dtype=torch.uint8, device="cuda")
    vp.run_local(dev["cu_sl"], dev["draft_tokens"], ts, ds, dev["seeds"], acc, em, kl, fl)
    torch.cuda.synchronize()
    return acc.cpu().numpy(), em.cpu().numpy(), kl.cpu().numpy(), fl.cpu().numpy()


@pytest.mark.parametrize("V,dtype,kmax,B", [
    (128256, torch.bfloat16, 8, 24), (32000, torch.bfloat16, 8, 64), (50000, torch.bfloat16, 6, 40),
    (8193, torch.float32, 6, 32), (20000, torch.float32, 4, 24),
])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_vocab_parallel_bit_identical(m, V, dtype, kmax, B, n):
    st = m.State(m.Config.default(resample=m.RESAMPLE_FULL), 4096)  # the vp stages implement D7
    try:
        m.VocabParallel(st, V, n, dtype)
    except m.DsdeError:
        pytest.skip("too many shards for this vocabulary")
    k = synth.random_k(B, kmax, V % 101 + n)
    host = make_host_batch(V, k, 40 + n, dtype=dtype, profiles=("code", "low"))
    ref = gpu_verify(m, st, to_device_inputs(host, dtype))
    got = _run_vp(m, st, host, dtype, n)
    for a, b in zip(ref, got):
        assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    rep = parity.compare_verify(host["cu_sl"], got[0], got[1], got[2],
                                oracle_verify(host, resample=oracle.RESAMPLE_FULL))
    assert rep.ok(), str(rep)
    assert st.device_error() == (0, -1)


def test_vp_verify_single_shard_and_one_rank_nccl(m):
    V, B = 32000, 48
    st = m.State(m.Config.default(resample=m.RESAMPLE_FULL), 64)
    k = synth.random_k(B, 8, 5)
    host = make_host_batch(V, k, 6)
    dev = to_device_inputs(host, torch.bfloat16)
    ref = gpu_verify(m, st, dev)
    vp = m.VocabParallel(st, V, 1, torch.bfloat16)
    nk = int(k.sum())
    ws = vp.workspace(B, nk)
    comm = m.Comm(m.Comm.unique_id(), 1, 0)
    for c in (None, comm):
        acc = torch.full((B,), -7, dtype=torch.int32, device="cuda")
        em = torch.full((nk + B,), -7, dtype=torch.int32, device="cuda")
        kl = torch.full((nk,), float("nan"), dtype=torch.float32, device="cuda")
        fl = torch.zeros(nk + B, dtype=torch.uint8, device="cuda")
        vp.verify(dev["cu_sl"], dev["draft_tokens"], dev["target"], dev["draft"], dev["seeds"], acc, em, kl, fl,
                  ws, comm=c)
        torch.cuda.synchronize()
        for a, b in zip(ref, (acc.cpu().numpy(), em.cpu().numpy(), kl.cpu().numpy(), fl.cpu().numpy())):
            assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    comm.close()


def test_vp_rejects_unsupported_modes(m):
    for kw in ({"greedy": 1, "resample": 1}, {"masked": 1, "resample": 1}, {"resample": 0}):
        st = m.State(m.Config.default(**kw), 8)
        with pytest.raises(m.DsdeError):
            vp = m.VocabParallel(st, 4096, 2, torch.bfloat16)
            host = make_host_batch(4096, np.full(4, 2), 1)
            _run_vp(m, st, host, torch.bfloat16, 2)
