"""with dsde_config.device_rows = 1 the kernels read the row
count sum_i k_i = cu_sl[B] on the device and size their grids for a capacity,
so the launch configuration of dsde_step no longer depends on the speculation
lengths (device data) and one CUDA graph, captured once, replays steps
with any SL pattern. Every replay is checked against the fp64 oracle (verify
outputs) and against eager dsde_step with device_rows = 0 on a second state
(outputs, SL^, next SL and cap bit-identical)."""
import numpy as np
import pytest
import torch

from tests import parity
from tests.gpu_util import dsde, make_host_batch, oracle_verify, to_device_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    return dsde()


@pytest.mark.parametrize("V,dtype,resample", [(32000, torch.bfloat16, 1), (8193, torch.float32, 1),
                                              (32000, torch.bfloat16, 0)])
def test_graph_captured_step_replays_any_sl_pattern(m, V, dtype, resample):
    B, kmax = 32, 8
    cap_rows = B * kmax
    st_g = m.State(m.Config.default(device_rows=1, resample=resample), B)
    st_e = m.State(m.Config.default(resample=resample), B)
    sg = m.Step(st_g, B, V, dtype, max_draft_rows=cap_rows)
    se = m.Step(st_e, B, V, dtype, max_draft_rows=cap_rows)
    esz = 2 if dtype == torch.bfloat16 else 4
    ld = V + (-(V * esz) % 16) // esz
    dev = "cuda"
    cu = torch.zeros(B + 1, dtype=torch.int32, device=dev)
    tok = torch.zeros(cap_rows, dtype=torch.int32, device=dev)
    tgt = torch.zeros((cap_rows + B, ld), dtype=dtype, device=dev)
    dft = torch.zeros((cap_rows, ld), dtype=dtype, device=dev)
    seeds = torch.zeros(cap_rows + B, dtype=torch.int64, device=dev)

    def load(t, k):
        host = make_host_batch(V, k, seed=1234 + V, dtype=dtype, profiles=("code", "low"), step=t)
        d = to_device_inputs(host, dtype)
        n = int(k.sum())
        cu.copy_(d["cu_sl"])
        tok[:n].copy_(d["draft_tokens"])
        tgt[: n + B].copy_(d["target"])
        dft[:n].copy_(d["draft"])
        seeds[: n + B].copy_(d["seeds"])
        return host, d, n

    rng = np.random.default_rng(V)
    # warm-up outside the capture (first-call kernel attributes) on a throwaway state
    warm = m.Step(m.State(m.Config.default(device_rows=1, resample=resample), B), B, V, dtype,
                  max_draft_rows=cap_rows)
    load(0, np.full(B, 4))
    warm(cu, tok, tgt, dft, seeds, cap_rows)
    torch.cuda.synchronize()

    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        sg(cu, tok, tgt, dft, seeds, cap_rows)
    for t in range(8):
        if t == 0:
            k = np.full(B, 4)
        elif t == 3:
            k = np.ones(B, dtype=np.int64)              # a tenth of the capacity
        elif t == 5:
            k = np.full(B, kmax)                        # exactly the capacity
        else:
            k = rng.integers(1, kmax + 1, B)
        host, d, n = load(t, k)
        g.replay()
        se(d["cu_sl"], d["draft_tokens"], d["target"], d["draft"], d["seeds"], n)
        torch.cuda.synchronize()
        acc_g, em_g = sg.accepted_len.cpu().numpy(), sg.emitted[: n + B].cpu().numpy()
        kl_g = sg.kld[:n].cpu().numpy()
        assert np.array_equal(acc_g, se.accepted_len.cpu().numpy()), t
        assert np.array_equal(em_g, se.emitted[: n + B].cpu().numpy()), t
        assert np.array_equal(kl_g.view(np.uint32), se.kld[:n].cpu().numpy().view(np.uint32)), t
        for name in ("sl_hat", "next_sl", "cap"):
            assert torch.equal(getattr(sg, name), getattr(se, name)), (t, name)
        rep = parity.compare_verify(host["cu_sl"], acc_g, em_g, kl_g, oracle_verify(host, resample=resample))
        assert rep.ok(), (t, str(rep))
    assert st_g.device_error()[0] == 0 and st_e.device_error()[0] == 0


def test_device_rows_beyond_capacity_is_a_device_error(m):
    """cu_sl[B] larger than the capacity: the sequences whose rows end beyond it
    are rejected on the device (DSDE_DERR_BAD_SL, accepted_len = -1), the rest
    are verified; nothing is read past the capacity."""
    B, V = 6, 4096
    k = np.array([3, 3, 3, 3, 3, 3])
    host = make_host_batch(V, k, seed=3)
    d = to_device_inputs(host, torch.bfloat16)
    st = m.State(m.Config.default(device_rows=1), B)
    cap_rows = 12  # sequences 4 and 5 end at rows 15 and 18
    ws = torch.empty(m.workspace_size(B, cap_rows, V, torch.bfloat16) + 256, dtype=torch.uint8, device="cuda")
    ws = ws[(-ws.data_ptr()) % 256:]
    acc = torch.full((B,), -7, dtype=torch.int32, device="cuda")
    em = torch.full((cap_rows + B,), -7, dtype=torch.int32, device="cuda")
    kld = torch.zeros(cap_rows, dtype=torch.float32, device="cuda")
    m.dsde_verify(st, V, cap_rows, d["cu_sl"], d["draft_tokens"][:cap_rows], d["target"][: cap_rows + B],
                  d["draft"][:cap_rows], d["seeds"][: cap_rows + B], acc, em, kld, None, ws)
    torch.cuda.synchronize()
    a = acc.cpu().numpy()
    assert list(a[4:]) == [-1, -1]
    assert np.all((a[:4] >= 0) & (a[:4] <= 3))
    code, seq = st.device_error()
    assert code == 1 and seq in (4, 5)  # DSDE_DERR_BAD_SL
    # the first four sequences match the oracle on their own
    sub = parity.subset_batch(host, [0, 1, 2, 3])
    o = oracle_verify(sub)
    n4 = 12
    # (their emitted slots are the first n4 + 4: slot of (i, j) = cu_sl[i] + i + j)
    rep = parity.compare_verify(sub["cu_sl"], a[:4], em.cpu().numpy()[: n4 + 4], kld.cpu().numpy()[:n4], o)
    assert rep.ok(), str(rep)
