"""Parity of the exact launch configuration bench.py times (VERDICT r1 "next" #1).

dsde_step at V = 128256 bf16 with B = 256 (config 3), 512 (config 4, low
acceptance: residual-heavy) and 2048 (config 5's whole batch on one GPU),
closed loop for a few steps. EVERY sequence of every step is compared with
the fp64 oracle (tests/parity.py bands: accepted lengths / tokens bit-exact
outside counted |u - p/q| < 1e-6 ties, KLD within 1e-5 relative). The GPU's
own fp32 KLDs and accepted lengths are then fed to the oracle's signal and cap
(identical inputs): SL^ must be bit-exact except pre-round
values within 1e-9 of n + 1/2, and the cap and next SLs exact. The oracle's
next SLs drive the following step (teacher forcing), so the layouts stay
identical on both sides.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests import parity
from tests.gpu_util import dsde, oracle_verify

pytestmark = pytest.mark.gpu

V = 128256


@pytest.fixture(scope="module")
def m():
    return dsde()


def device_subset(s, ids):
    """Oracle-format host copy of sequences `ids` of a device batch (gathered on
    the device: a full batch is several GB)."""
    cu = s.cu_sl.cpu().numpy().astype(np.int64)
    trow, drow, k = [], [], []
    for i in ids:
        ki = int(cu[i + 1] - cu[i])
        k.append(ki)
        trow.extend(range(cu[i] + i, cu[i] + i + ki + 1))
        drow.extend(range(cu[i], cu[i] + ki))
    t = s.target.index_select(0, torch.tensor(trow, device=s.target.device))[:, :s.V].cpu()
    d = s.draft.index_select(0, torch.tensor(drow, device=s.draft.device))[:, :s.V].cpu()
    t = t.view(torch.int16).numpy().view(np.uint16)
    d = d.view(torch.int16).numpy().view(np.uint16)
    seeds = s.seeds.cpu().numpy().view(np.uint64)
    toks = s.draft_tokens.cpu().numpy()
    return dict(cu_sl=np.concatenate([[0], np.cumsum(k)]).astype(np.int32), target=t, draft=d,
                draft_tokens=np.concatenate([toks[cu[i]:cu[i] + ki] for i, ki in zip(ids, k)]),
                seeds=np.concatenate([seeds[cu[i] + i:cu[i] + i + ki + 1] for i, ki in zip(ids, k)]))


def compare_all(s, out, chunk=256, resample=oracle.RESAMPLE_FULL):
    """Every sequence of the step against the oracle, in chunks of sequences.
    Returns the merged report and the oracle's accepted lengths / KLDs."""
    B = s.cu_sl.numel() - 1
    cu = s.cu_sl.cpu().numpy()
    acc, em, kl = out.accepted_len.cpu().numpy(), out.emitted.cpu().numpy(), out.kld.cpu().numpy()
    rep = parity.Report()
    for c0 in range(0, B, chunk):
        ids = np.arange(c0, min(B, c0 + chunk))
        sub = device_subset(s, ids)
        o = oracle_verify(sub, nthreads=16, resample=resample)
        a2, e2, k2 = parity.gather_subset_outputs(cu, ids, acc, em, kl)
        r = parity.compare_verify(sub["cu_sl"], a2, e2, k2, o, seq_ids=ids)
        rep.merge(r)
    return rep


@pytest.mark.parametrize("B,profiles,steps,V,resample", [
    (256, ("code",), 3, V, 1),                     # config 3 (and config 5's per-GPU shard at 8 GPUs)
    (512, ("low",), 3, V, 1),                      # config 4: low acceptance, residual-heavy
    (2048, ("code", "dialogue", "low"), 2, V, 1),  # config 5's whole batch on one GPU
    (64, ("low",), 2, 256000, 1),                  # Gemma-like vocabulary
    (256, ("code",), 2, V, 0),                     # the D23 recovery draw (speculative first proposal)
    (512, ("low",), 2, V, 0),
    (2048, ("code", "dialogue", "low"), 1, V, 0),  # 8-warp tail CTAs, several rounds per CTA
    (64, ("low",), 2, 256000, 0),                  # > kSpecSub slices: proposals built at draw time
], ids=["cfg3_B256", "cfg4_B512", "cfg5_B2048", "gemma_V256000_B64",
        "cfg3_B256_d23", "cfg4_B512_d23", "cfg5_B2048_d23", "gemma_V256000_B64_d23"])
def test_dsde_step_full_size_every_sequence(m, B, profiles, steps, V, resample):
    cfg_g = m.Config.default(calib_steps=1, calib_sl=4, resample=resample)
    cfg_o = oracle.Config(calib_steps=1, calib_sl=4)
    st = m.State(cfg_g, B)
    ost = oracle.OracleState(cfg_o, B)
    stepper = m.Step(st, B, V, torch.bfloat16, with_diag=True)
    w = synth.Workload(B=B, V=V, dtype=torch.bfloat16, profiles=profiles, seed=B + 17)
    k = np.full(B, 4, dtype=np.int64)
    total = parity.Report()
    sl_ties = 0
    for step in range(steps):
        s = synth.generate_step(w, step + 40, k, device="cuda")
        out = stepper(s.cu_sl, s.draft_tokens, s.target, s.draft, s.seeds, int(k.sum()))
        torch.cuda.synchronize()
        rep = compare_all(s, out, resample=resample)
        assert rep.ok(), (step, str(rep))
        total.merge(rep)
        # the GPU's own KLDs / accepted lengths into the oracle signal + cap (identical inputs)
        cu = s.cu_sl.cpu().numpy()
        kl_g = out.kld.cpu().numpy().astype(np.float64)
        acc_g = out.accepted_len.cpu().numpy()
        sl_o, cal_o, dg_o = ost.update_signal(np.arange(B), cu, kl_g, acc_g)
        sl_g = out.sl_hat.cpu().numpy()
        diff = np.nonzero(sl_g != sl_o)[0]
        for i in diff:
            x = dg_o[i, 6]
            assert np.isfinite(x) and abs((x - np.floor(x)) - 0.5) < 1e-9, (step, i, sl_g[i], sl_o[i])
        sl_ties += diff.size
        nx_o, cap_o = oracle.next_sl(cfg_o, sl_o, cal_o)
        if diff.size == 0:
            assert out.cap.item() == cap_o, (step, out.cap.item(), cap_o)
            assert np.array_equal(out.next_sl.cpu().numpy(), nx_o), step
        k = nx_o.astype(np.int64)
    assert st.device_error() == (0, -1)
    print(f"B={B}: {total} sl_ties={sl_ties}")
