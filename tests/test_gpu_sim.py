"""The closed-loop decode simulator driving the library (sim/, SURVEY §8(f)
f4) with SPEC's batch-engine cost model: budgets are met exactly,
runs are bit-reproducible, a homogeneous batch scales perfectly and
the adaptive cap never lengthens a step (the straggler bound)."""
import numpy as np
import pytest
import torch

import sim

pytestmark = pytest.mark.gpu


def test_budget_met_and_reproducible():
    a = sim.run_until_done(16, 24, dict(), V=8192, seed=3, keep_reports=True)
    b = sim.run_until_done(16, 24, dict(), V=8192, seed=3, keep_reports=True)
    assert a.total_emitted == 16 * 24
    assert a.simulated_time == b.simulated_time and a.total_steps == b.total_steps
    assert [r.accepted for r in a.reports] == [r.accepted for r in b.reports]
    # progress: every active sequence emits >= 1 token per step
    assert all(min(r.emitted) >= 1 for r in a.reports)


@pytest.mark.parametrize("cap_mode", [0, 1])
def test_homogeneous_batch_scales_perfectly(cap_mode):
    """Identical sequences: every step's max k equals every k, so throughput
    is exactly proportional to the batch size."""
    one = sim.run_until_done(1, 32, dict(cap_mode=cap_mode), V=8192, seed=5, homogeneous=True)
    for B in (4, 16):
        r = sim.run_until_done(B, 32, dict(cap_mode=cap_mode), V=8192, seed=5, homogeneous=True)
        assert r.simulated_time == one.simulated_time
        assert r.throughput == pytest.approx(B * one.throughput, rel=1e-12)


def test_cap_bounds_every_step():
    """With the cap every step's proposed max k is at most the cap the
    library applied (Eq.11, D14), which never exceeds the uncapped max."""
    r = sim.run_until_done(32, 48, dict(cap_mode=1, calib_steps=2), V=8192, seed=9, keep_reports=True)
    caps = [rep.cap for rep in r.reports]
    ks = [max(rep.k) for rep in r.reports]
    assert all(k <= c for k, c in zip(ks[1:], caps[:-1]))


def test_cap_improves_throughput_scaling():
    """Fig. SL_cap_test direction: on a heterogeneous
    straggler workload the capped throughput ratio at batch 32 exceeds the
    uncapped one (profiles/r2_cap_scaling.json: 30.0x vs 25.0x at 64)."""
    res = sim.throughput_scaling(batch_sizes=(1, 32), budget=48, V=8192, seed=11)
    cap = res["cap"][-1]["scaling"]
    nocap = res["no_cap"][-1]["scaling"]
    assert cap > nocap, (cap, nocap)
