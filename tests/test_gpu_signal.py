"""GPU parity of dsde_update_signal / dsde_next_sl against the oracle, and the
closed-loop DSDE step (verify -> signal -> cap) on configs 1 and 2 with the
oracle's speculation lengths teacher-forced into both sides."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity
from tests.gpu_util import dsde, oracle_verify, to_device_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def m():
    return dsde()


def _cfg_pair(m, **kw):
    return m.Config.default(**kw), oracle.Config(**kw)


def _sl_tie(x, band):
    return np.isfinite(x) and abs((x - np.floor(x)) - 0.5) < band


@pytest.mark.parametrize("kw", [
    {}, {"window_unit": 1}, {"calib_steps": 0}, {"calib_steps": 2, "delta": 1.0},
    {"n_short": 3, "n_long": 7, "sl_ceiling": 4, "calib_sl": 4}, {"cap_mode": 0},
])
def test_signal_and_cap_on_identical_klds(m, kw):
    """Predictor fed identical fp32 KLDs: SL^ bit-exact except pre-round values
    within 1e-9 of n + 1/2; variances within 1e-5 relative (D16)."""
    gc, oc = _cfg_pair(m, **kw)
    B = 97
    st = m.State(gc, B)
    ost = oracle.OracleState(oc, B)
    rng = np.random.default_rng(len(str(kw)))
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    ties = 0
    for step in range(70):
        k = rng.integers(1, gc.sl_ceiling + 1, B)
        cu = synth.cu_from_k(k)
        scale = rng.choice([0.001, 0.05, 0.5], B)
        kl = (rng.exponential(1.0, int(cu[-1])) * np.repeat(scale, k)).astype(np.float32)
        if step % 9 == 0:
            kl[: k[0]] = 0.25  # some flat stretches
        acc = rng.integers(0, k + 1).astype(np.int32)
        sl_o, cal_o, dg_o = ost.update_signal(np.arange(B), cu, kl.astype(np.float64), acc)
        sl_g = torch.empty(B, dtype=torch.int32, device="cuda")
        dg_g = torch.empty((B, 8), dtype=torch.float64, device="cuda")
        cu_d = torch.from_numpy(cu).cuda()
        m.dsde_update_signal(st, slots, cu_d, torch.from_numpy(kl).cuda(), torch.from_numpy(acc).cuda(),
                             sl_g, dg_g)
        sl_g, dg_g = sl_g.cpu().numpy(), dg_g.cpu().numpy()
        for i in range(B):
            if sl_g[i] != sl_o[i]:
                assert _sl_tie(dg_o[i, 6], 1e-9), (step, i, sl_g[i], sl_o[i], dg_o[i])
                ties += 1
        for col in (0, 1, 2, 3, 4, 5, 7):
            a, b = dg_g[:, col], dg_o[:, col]
            both_nan = np.isnan(a) & np.isnan(b)
            ok = both_nan | (np.abs(a - b) <= 1e-5 * np.abs(b) + 1e-12)
            assert ok.all(), (step, col, a[~ok][:4], b[~ok][:4])
        # cap + next SL on identical SL^ (use the oracle's to isolate a7)
        budget = rng.integers(1, 10, B).astype(np.int32) if step % 3 == 0 else None
        nx_o, cap_o = oracle.next_sl(oc, sl_o, cal_o, budget)
        nx_g = torch.empty(B, dtype=torch.int32, device="cuda")
        cap_g = torch.empty(1, dtype=torch.int32, device="cuda")
        sl_in = torch.from_numpy(sl_o).cuda()
        m.dsde_next_sl(st, slots, sl_in, None if budget is None else torch.from_numpy(budget).cuda(),
                       nx_g, cap_g)
        assert cap_g.item() == cap_o
        assert np.array_equal(nx_g.cpu().numpy(), nx_o)
    assert ties <= 2


def test_state_export_import_replay(m):
    gc = m.Config.default()
    B = 16
    st = m.State(gc, B)
    slots = torch.arange(B, dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(3)
    def step(seed):
        r = np.random.default_rng(seed)
        k = r.integers(1, 9, B)
        cu = torch.from_numpy(synth.cu_from_k(k)).cuda()
        kl = torch.from_numpy(r.exponential(0.1, int(k.sum())).astype(np.float32)).cuda()
        acc = torch.from_numpy(r.integers(0, k + 1).astype(np.int32)).cuda()
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        m.dsde_update_signal(st, slots, cu, kl, acc, out)
        return out.cpu().numpy()
    for s in range(8):
        step(s)
    snap = st.export()
    a = [step(100 + s) for s in range(12)]
    st.load(snap)
    b = [step(100 + s) for s in range(12)]
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    # reset clears a slot back to calibration
    st.reset(torch.tensor([0], dtype=torch.int32, device="cuda"))
    out = step(999)
    assert out[0] == gc.calib_sl


@pytest.mark.parametrize("fused", [True, False], ids=["dsde_step", "three_calls"])
@pytest.mark.parametrize("cfg_id", [1, 2])
def test_closed_loop_parity(m, cfg_id, fused):
    """Configs 1-2: the full DSDE step for 64 steps; each side computes its own
    KLDs; the oracle's next SL is teacher-forced into both (D16). Run through
    the fused dsde_step call and through dsde_verify / dsde_update_signal /
    dsde_next_sl."""
    if cfg_id == 1:
        B, V, dtype, profiles, ceiling, steps = 4, 32000, torch.float32, ("code",), 4, 64
    else:
        B, V, dtype, profiles, ceiling, steps = 64, 32000, torch.bfloat16, ("code", "dialogue"), 8, 64
    gc, oc = _cfg_pair(m, sl_ceiling=ceiling, calib_sl=min(4, ceiling))
    st = m.State(gc, B)
    ost = oracle.OracleState(oc, B)
    stepper = m.Step(st, B, V, dtype, with_diag=True)
    w = synth.Workload(B=B, V=V, dtype=dtype, profiles=profiles, seed=100 + cfg_id)
    k = np.full(B, gc.calib_sl)
    total = parity.Report()
    tainted = np.zeros(B, bool)
    sl_ties = 0
    for s in range(steps):
        inp = synth.generate_step(w, s, k, device="cuda")
        host = inp.host_arrays()
        out = stepper(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, int(k.sum()), fused=fused)
        torch.cuda.synchronize()
        o = oracle_verify(host)
        rep = parity.compare_verify(host["cu_sl"], out.accepted_len.cpu().numpy(), out.emitted.cpu().numpy(),
                                    out.kld.cpu().numpy(), o)
        assert rep.ok(), (s, str(rep))
        total.merge(rep)
        if rep.accept_ties:
            acc_g = out.accepted_len.cpu().numpy()
            tainted |= acc_g != o.accepted_len
        sl_o, cal_o, dg_o = ost.update_signal(np.arange(B), host["cu_sl"], o.kld, o.accepted_len)
        nx_o, cap_o = oracle.next_sl(oc, sl_o, cal_o)
        sl_g = out.sl_hat.cpu().numpy()
        for i in range(B):
            if tainted[i]:
                continue
            if sl_g[i] != sl_o[i]:
                assert _sl_tie(dg_o[i, 6], 1e-4), (s, i, sl_g[i], sl_o[i], dg_o[i])
                sl_ties += 1
        if not tainted.any() and np.array_equal(sl_g, sl_o):
            assert out.cap.item() == cap_o
            assert np.array_equal(out.next_sl.cpu().numpy(), nx_o)
        k = nx_o.astype(np.int64)
    print(f"cfg{cfg_id}: {total} sl_ties={sl_ties}")


@pytest.mark.parametrize("B,V,resample", [(64, 32000, 1), (256, 4096, 1), (512, 4096, 1), (2048, 4096, 1),
                                          (64, 32000, 0), (256, 4096, 0), (2048, 4096, 0)])
def test_step_matches_three_calls(m, B, V, resample):
    """dsde_step (one fused launch: verify + signal + cap) and the three separate
    calls give bit-identical results and state, step after step, with and
    without a per-sequence budget; B spans the batch sizes of configs 2-5
    (the launch shapes bench.py times; a small V keeps it cheap)."""
    dtype = torch.bfloat16
    gc, _ = _cfg_pair(m, sl_ceiling=8, calib_sl=4)
    gc.resample = resample  # D23: the proposal rounds differ (the signal warp is busy in dsde_step), not the result
    sa, sb = m.State(gc, B), m.State(gc, B)
    pa, pb = m.Step(sa, B, V, dtype, with_diag=True), m.Step(sb, B, V, dtype, with_diag=True)
    w = synth.Workload(B=B, V=V, dtype=dtype, profiles=("code", "low"), seed=77)
    k = np.full(B, 4)
    for s in range(12):
        inp = synth.generate_step(w, s, k, device="cuda")
        n = int(k.sum())
        # every third step a per-sequence token budget clamps the next SL
        bud = (torch.arange(B, dtype=torch.int32, device="cuda") % 7 + 1) if s % 3 == 1 else None
        oa = pa(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n, budget=bud, fused=True)
        ob = pb(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n, budget=bud, fused=False)
        if bud is not None:
            assert torch.all(oa.next_sl <= bud), s
        torch.cuda.synchronize()
        for f in ("accepted_len", "emitted", "kld", "sl_hat", "next_sl", "cap"):
            x, y = getattr(oa, f).cpu(), getattr(ob, f).cpu()
            assert torch.equal(x, y), (s, f)
        da, db = oa.diag.cpu().nan_to_num(-7.0), ob.diag.cpu().nan_to_num(-7.0)
        bad = (da != db).nonzero().tolist()
        assert not bad, (s, bad[:4], [(da[i, j].item(), db[i, j].item()) for i, j in bad[:4]])
        k = oa.next_sl.cpu().numpy().astype(np.int64)
    assert sa.device_error() == (0, -1) and sb.device_error() == (0, -1)


def test_step_with_single_rank_nccl_comm(m):
    """The multi-GPU cap path of dsde_step (the pass kernel without the fused cap, the
    exact int64 partial, ncclAllReduce, k_cap_apply) on a one-rank NCCL
    communicator: bit-identical to the single-GPU path, step after step, for
    cap_mode 1 (sum) and 0 (sum + max all-reduces)."""
    B, V, dtype = 48, 32000, torch.bfloat16
    comm = m.Comm(m.Comm.unique_id(), 1, 0)
    try:
        for cap_mode in (1, 0):
            gc, _ = _cfg_pair(m, sl_ceiling=8, calib_sl=4)
            gc.cap_mode = cap_mode
            gc.calib_steps = 2
            sa, sb = m.State(gc, B), m.State(gc, B)
            pa = m.Step(sa, B, V, dtype, with_diag=True, comm=comm)
            pb = m.Step(sb, B, V, dtype, with_diag=True)
            w = synth.Workload(B=B, V=V, dtype=dtype, profiles=("code", "dialogue"), seed=91 + cap_mode)
            k = np.full(B, 4)
            for s in range(8):
                inp = synth.generate_step(w, s, k, device="cuda")
                n = int(k.sum())
                oa = pa(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n)
                ob = pb(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n)
                torch.cuda.synchronize()
                for f in ("accepted_len", "emitted", "kld", "sl_hat", "next_sl", "cap"):
                    assert torch.equal(getattr(oa, f).cpu(), getattr(ob, f).cpu()), (cap_mode, s, f)
                k = oa.next_sl.cpu().numpy().astype(np.int64)
            assert sa.device_error() == (0, -1)
    finally:
        comm.close()
