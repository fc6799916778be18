"""Closed-loop decode simulator driving the CUDA library.

A batch of sequences, each with a token budget, is decoded step by step:
every step the library verifies the batch's ragged drafts (dsde_step: verify
-> signal -> SL prediction -> adaptive cap, on the GPU), the accepted tokens
plus the recovery / bonus token are emitted, finished sequences retire at the
step boundary, and the next step drafts the SLs the library returned (already
capped and clamped to each sequence's remaining budget). The draft and target
logits are synthetic (synth/, seeded; the stand-in for the two models).

Time is SPEC's batch-engine cost model (the paper measures wall
clock on GPUs, "invented — artifact plumbing"): per step
    draft_phase_time  = c_draft * max_i k_i            (drafting is sequential per token)
    verify_phase_time = c_verify_base + c_verify_per_token * max_i k_i
so a straggler's long SL stalls the whole batch (Fig.3) and the cap
(Eq.11) bounds it. The GPU time of each dsde_step is recorded as
well (CUDA events). `throughput_scaling` is the Fig. SL_cap_test experiment
(S:479-487): simulated tokens per second for batch sizes 1..64
with and without the cap, and the ratio to batch size 1.

This is a harness around the library (test / experiment infrastructure):
nothing here computes a step of the method.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

import synth


@dataclass
class CostModel:
    """SPEC CostModel, simulated seconds; all components > 0."""
    c_draft: float = 1.0
    c_verify_base: float = 4.0
    c_verify_per_token: float = 0.5

    def step_time(self, kmax: int) -> tuple[float, float]:
        return self.c_draft * kmax, self.c_verify_base + self.c_verify_per_token * kmax


@dataclass
class StepReport:
    step: int
    k: list           # proposed k of each active sequence (after cap and budget)
    accepted: list
    emitted: list     # tokens emitted this step (accepted + 1, budget-clamped)
    cap: int
    draft_time: float
    verify_time: float
    gpu_ms: float


@dataclass
class RunMetrics:
    total_emitted: int = 0
    total_steps: int = 0
    simulated_time: float = 0.0
    gpu_ms: float = 0.0
    accepted: int = 0
    proposed: int = 0
    per_step_sl: list = field(default_factory=list)
    reports: list = field(default_factory=list)

    @property
    def throughput(self) -> float:
        """emitted tokens per simulated second"""
        return self.total_emitted / self.simulated_time

    @property
    def block_efficiency(self) -> float:
        return self.total_emitted / max(1, sum(len(r.k) for r in self.reports))

    @property
    def acceptance_rate(self) -> float:
        return self.accepted / max(1, self.proposed)


def run_until_done(B: int, budget: int, cfg_kw: dict, cost: CostModel | None = None, V: int = 32000,
                   dtype=torch.bfloat16, profiles=("code", "dialogue", "low"), seed: int = 7,
                   homogeneous: bool = False, keep_reports: bool = False, device="cuda") -> RunMetrics:
    """Decode B sequences of `budget` tokens each through the library.
    cfg_kw: dsde_config fields (e.g. cap_mode=0 for no cap). homogeneous: every
    sequence sees the same logits and seeds (sequence 0's), so predictions
    never diverge."""
    import paper_2509_01083_b200 as m

    cost = cost or CostModel()
    cfg = m.Config.default(**cfg_kw)
    st = m.State(cfg, B)
    w = synth.Workload(B=B, V=V, dtype=dtype, profiles=profiles, seed=seed)
    ws = torch.empty(m.workspace_size(B, B * m.DSDE_MAX_SL, V, dtype) + 256, dtype=torch.uint8, device=device)
    ws = ws[(-ws.data_ptr()) % 256:]
    remaining = np.full(B, budget, dtype=np.int64)
    k_next = np.full(B, cfg.calib_sl, dtype=np.int64)
    met = RunMetrics()
    i32 = dict(dtype=torch.int32, device=device)
    step = 0
    while True:
        act = np.nonzero(remaining > 0)[0]
        if act.size == 0:
            break
        n = act.size
        k = np.minimum(k_next[act], remaining[act])
        # the step's inputs: the whole batch generated (retired sequences with
        # k = 1, dropped below), so a sequence's logits do not depend on which
        # others are still running
        kf = np.ones(B, dtype=np.int64)
        kf[act] = k
        if homogeneous:
            kf[:] = k[0]
        full = synth.generate_step(w, step, kf, device=device)
        cu_f = synth.cu_from_k(kf)
        if homogeneous:
            # every sequence gets sequence 0's rows and seeds
            src = np.zeros(B, dtype=np.int64)
        else:
            src = np.arange(B)
        trows = np.concatenate([cu_f[src[i]] + src[i] + np.arange(kf[src[i]] + 1) for i in act])
        drows = np.concatenate([cu_f[src[i]] + np.arange(kf[src[i]]) for i in act])
        ti = torch.from_numpy(trows).to(device)
        di = torch.from_numpy(drows).to(device)
        cu = torch.from_numpy(synth.cu_from_k(k)).to(device)
        nk = int(k.sum())
        target = full.target.index_select(0, ti)
        draft = full.draft.index_select(0, di)
        toks = full.draft_tokens.index_select(0, di)
        seeds = full.seeds.index_select(0, ti)
        slots = torch.from_numpy(act.astype(np.int32)).to(device)
        # budget for the NEXT step: what is left after this one emits at least one token each
        acc = torch.empty(n, **i32)
        em = torch.empty(nk + n, **i32)
        kld = torch.empty(nk, dtype=torch.float32, device=device)
        sl_hat = torch.empty(n, **i32)
        nxt = torch.empty(n, **i32)
        cap = torch.empty(1, **i32)
        bud = torch.from_numpy(np.maximum(remaining[act] - 1, 1).astype(np.int32)).to(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.dsde_step(st, V, nk, slots, cu, toks, target, draft, seeds, bud, acc, em, kld, None, sl_hat, None,
                    nxt, cap, ws)
        e1.record()
        torch.cuda.synchronize()
        a = acc.cpu().numpy().astype(np.int64)
        if (a < 0).any():
            raise RuntimeError(f"device error {st.device_error()}")
        emitted = np.minimum(a + 1, remaining[act])
        remaining[act] -= emitted
        k_next[act] = nxt.cpu().numpy()
        dt, vt = cost.step_time(int(k.max()))
        met.total_emitted += int(emitted.sum())
        met.total_steps += 1
        met.simulated_time += dt + vt
        met.gpu_ms += e0.elapsed_time(e1)
        met.accepted += int(a.sum())
        met.proposed += nk
        met.per_step_sl.append(int(k.max()))
        if keep_reports:
            met.reports.append(StepReport(step, k.tolist(), a.tolist(), emitted.tolist(), int(cap.item()), dt, vt,
                                          e0.elapsed_time(e1)))
        else:
            met.reports.append(StepReport(step, k.tolist(), [], [], 0, dt, vt, 0.0))
        step += 1
        if step > 100 * budget:
            raise RuntimeError("no progress")
    return met


def throughput_scaling(batch_sizes=(1, 2, 4, 8, 16, 32, 64), budget: int = 64, cost: CostModel | None = None,
                       **kw) -> dict:
    """Fig. SL_cap_test / S:479-487: tokens per simulated second for each batch
    size, with the Eq.11 cap (cap_mode 1) and without it (cap_mode 0), and the
    scaling ratio relative to batch size 1."""
    out = {}
    for mode, name in ((1, "cap"), (0, "no_cap")):
        rows = []
        for B in batch_sizes:
            r = run_until_done(B, budget, dict(cap_mode=mode), cost=cost, **kw)
            rows.append(dict(B=B, throughput=r.throughput, steps=r.total_steps, emitted=r.total_emitted,
                             simulated_time=r.simulated_time, gpu_ms=r.gpu_ms, acceptance=r.acceptance_rate,
                             mean_step_sl=float(np.mean(r.per_step_sl))))
        base = rows[0]["throughput"]
        for row in rows:
            row["scaling"] = row["throughput"] / base
        out[name] = rows
    return out
