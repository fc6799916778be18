#!/usr/bin/env python
"""bench.py — throughput of the DSDE verification hot path on B200.

One "step" = one pass of the whole hot path over one
batch: dsde_verify -> dsde_update_signal -> dsde_next_sl (with the NCCL cap
all-reduce when N > 1).

Workload (N = 1): BASELINE config 3 — B = 256 sequences per GPU, V = 128256,
bf16 logits, SL <= 8 chosen by DSDE itself (closed loop), high-acceptance
("code") profile. N > 1: weak scaling, 256 sequences per rank (N = 8 is config
5's B = 2048 sharded over 8 GPUs) with the batch-wide cap all-reduced over NCCL.

Measurement:
  * record: after a pre-roll (calibration + settling), R closed-loop steps are
    run once and their inputs kept resident in HBM (one distinct ~1.1 GB set
    per step, so every timed step reads its logits from HBM, not L2);
  * replay: the state is restored to the start of the recording, W warm-up
    steps run, then K timed steps replay the recorded steps in order (cyclically
    if K + W > R), bracketed by barrier + synchronize, CUDA events on the
    launching stream, max over ranks;
  * roofline: algorithmic bytes of the stream kernel / its own
    CUDA-event time, measured in a second replay of the same steps with the
    library's per-launch events (they cost ~14 us per step, so the headline
    pass has none), against MEASURED_PEAKS.json hbm_gbs;
  * e2e: the same metric through the public Python API from pinned host buffers
    (H2D of the step inputs and D2H of the results inside the timed region);
  * cpu_baseline: the fp64 oracle (oracle/, test infrastructure) on a bounded
    sample of the same workload on the host cores, rank 0, N = 1 only.
--impl reference: the oracle arm (the reference implementation of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verify positions/s and HBM GB/s vs peak at V=128256, 1/2/4/8 B200"
UNIT = "positions/s"
STREAM_KERNEL = {"tma": "k_stream_tma"}.get(
    os.environ.get("DSDE_STREAM", ""), "k_stream_ldg")

CONFIGS = {
    # BASELINE.json configs[2]: the N=1 workload (and the per-rank shard at N>1)
    3: dict(B=256, V=128256, profiles=("code",), ceiling=8, name="cfg3: B=256/GPU, SL<=8 (DSDE closed loop), "
            "V=128256 bf16 logits, high-acceptance (code) profile"),
    # BASELINE.json configs[3]
    4: dict(B=512, V=128256, profiles=("low",), ceiling=8, name="cfg4: B=512/GPU, SL<=8 (DSDE closed loop), "
            "V=128256 bf16 logits, low-acceptance profile"),
    # BASELINE.json configs[1]
    2: dict(B=64, V=32000, profiles=("code", "dialogue"), ceiling=8, name="cfg2: B=64, SL<=8, V=32000 bf16, "
            "mixed code/dialogue"),
}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _traffic_record(workload_key: str):
    """Per-launch DRAM bytes of the dominant kernel from a committed ncu capture
    (profiles/traffic.json, written from `ncu --set full`), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(workload_key)


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while running."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for bit, name in self.REASONS.items():
            if r & bit and name != "gpu_idle":
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()
            if not self.samples:
                self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_step_sample(host: dict, n_seq: int, nthreads: int, seed: int, greedy: bool = False):
    """Runs the oracle's verify on a sample of n_seq sequences of one step."""
    import oracle
    from tests import parity
    B = len(host["cu_sl"]) - 1
    ids = np.random.default_rng(seed).choice(B, min(n_seq, B), replace=False)
    sub = parity.subset_batch(host, np.sort(ids))
    t0 = time.perf_counter()
    r = oracle.verify(sub["cu_sl"], sub["draft_tokens"], sub["target"], sub["draft"], sub["seeds"],
                      oracle.BF16 if sub["target"].dtype == np.uint16 else oracle.F32, nthreads=nthreads,
                      greedy=greedy)
    dt = time.perf_counter() - t0
    return int(sub["cu_sl"][-1]), dt, sub, r


def run_reference(args):
    """--impl reference: the fp64 oracle on host cores, bounded sample per step."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    import torch

    import oracle
    import synth
    oracle.build()
    cfg = CONFIGS[args.config]
    nthreads = os.cpu_count() or 1
    per_step = args.ref_seqs
    w = synth.Workload(B=per_step, V=cfg["V"], dtype=torch.bfloat16, profiles=cfg["profiles"], seed=args.seed,
                       greedy_draft=args.greedy)
    ost = oracle.OracleState(oracle.Config(sl_ceiling=cfg["ceiling"]), per_step)
    k = np.full(per_step, 4)
    positions, elapsed = 0, 0.0
    for s in range(args.warmup + args.steps):
        host = synth.generate_step(w, s, k, device="cpu").host_arrays()
        t0 = time.perf_counter()
        r = oracle.verify(host["cu_sl"], host["draft_tokens"], host["target"], host["draft"], host["seeds"],
                          oracle.BF16, nthreads=nthreads, greedy=args.greedy)
        sl, cal, _ = ost.update_signal(np.arange(per_step), host["cu_sl"], r.kld, r.accepted_len)
        nx, cap = oracle.next_sl(ost.cfg, sl, cal)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            positions += int(k.sum())
            elapsed += dt
        k = nx.astype(np.int64)
    value = positions / elapsed
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config_dict(args, cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                         "sample": f"{per_step} sequences of the workload per step (DSDE closed loop, "
                                   f"verify+signal+cap), V={cfg['V']} bf16"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(args, cfg, n):
    return {"workload": cfg["name"], "B_per_gpu": cfg["B"], "global_batch": cfg["B"] * n, "V": cfg["V"],
            "logits": "bf16", "sl_ceiling": cfg["ceiling"], "profiles": list(cfg["profiles"]),
            "parallelism": f"dp{n}", "l2": "inputs larger than L2: a distinct ~1 GB input set per step",
            "replay": "recorded closed-loop DSDE steps replayed in order (cyclic if K+W > R)",
            "verify": "greedy (T=0, draft argmax tokens)" if args.greedy else "rejection sampling (T=1)",
            "draft_entropy": bool(args.entropy)}


def run(args):
    import torch
    import torch.distributed as dist

    import paper_2509_01083_b200 as m
    import synth

    ws, rank, local = _dist_env()
    if args.gpus != ws:
        if ws == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    B, V = cfg["B"], cfg["V"]
    m.lib()
    comm = None
    if ws > 1:
        uid = [m.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = m.Comm(uid[0], ws, rank)
    mcfg = m.Config.default(sl_ceiling=cfg["ceiling"], calib_sl=min(4, cfg["ceiling"]), greedy=int(args.greedy))
    state = m.State(mcfg, B)
    step = m.Step(state, B, V, torch.bfloat16, comm=comm)
    if args.entropy:  # the fused draft entropy in the same stream pass
        state.set_draft_entropy(torch.empty(B * 16, dtype=torch.float32, device=dev))
    w = synth.Workload(B=B, V=V, dtype=torch.bfloat16, profiles=cfg["profiles"], seed=args.seed + 7919 * rank,
                       greedy_draft=args.greedy)
    stream = torch.cuda.current_stream()

    # ---- pre-roll (calibration + settling), inputs not kept
    k = np.full(B, mcfg.calib_sl, dtype=np.int64)
    s = 0
    for _ in range(args.preroll):
        inp = synth.generate_step(w, s, k, device=dev)
        out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, int(k.sum()))
        k = out.next_sl.cpu().numpy().astype(np.int64)
        s += 1
    del inp
    # ---- record R closed-loop steps (inputs resident in HBM)
    R = min(args.record, args.warmup + args.steps)
    snap = state.export()
    rec, stats = [], dict(pos=0, acc=0, resid=0, bonus=0, seqs=0, rows=0, vbytes=0)
    for r in range(R):
        inp = synth.generate_step(w, s, k, device=dev)
        n = int(k.sum())
        out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n)
        acc = out.accepted_len.cpu().numpy()
        nx = out.next_sl.cpu().numpy().astype(np.int64)
        bonus = int(np.sum(acc == k))
        rows = 2 * n + bonus
        vbytes = rows * V * 2 + n * 4 + (n + B) * 8 + n * 4 + (n + B) * 5 + B * 4
        sbytes = 2 * n * V * 2  # a1 stream kernel: target + draft row of every draft position
        rec.append(dict(inp=inp, n=n, k=k.copy(), rows=rows, vbytes=vbytes, sbytes=sbytes, next=nx))
        stats["pos"] += n
        stats["acc"] += int(acc.sum())
        stats["bonus"] += bonus
        stats["resid"] += B - bonus
        stats["seqs"] += B
        k = nx
        s += 1
    torch.cuda.synchronize()

    def replay(idx):
        e = rec[idx % R]
        i = e["inp"]
        step.verify(i.cu_sl, i.draft_tokens, i.target, i.draft, i.seeds, e["n"])
        step.signal_and_cap(i.cu_sl)

    def run_step(j):
        e = rec[(args.warmup + j) % R]
        i = e["inp"]
        if args.split_calls:
            step.verify(i.cu_sl, i.draft_tokens, i.target, i.draft, i.seeds, e["n"])
            step.signal_and_cap(i.cu_sl)
        else:  # one dsde_step call: the whole hot path (verify + signal + cap)
            step(i.cu_sl, i.draft_tokens, i.target, i.draft, i.seeds, e["n"])

    # ---- pass 1 (the headline): warm-up + K timed steps replayed from the
    # recorded start state, nothing but the two bracketing events in the region
    state.load(snap)
    for wi in range(args.warmup):
        replay(wi)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        t_start.record(stream)
        for j in range(args.steps):
            run_step(j)
        t_end.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)

    # ---- pass 2 (kernel times for the roofline): the same replay with the
    # library's per-launch events (dsde_profile_*) and per-step events on the
    # launching stream; events cost ~14 us per step, so they stay out of pass 1
    K2 = args.steps
    state.load(snap)
    for wi in range(args.warmup):
        replay(wi)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K2)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    state.profile_read()  # drop anything recorded before the timed region
    state.profile(True)
    for j in range(K2):
        ev[j][0].record(stream)
        run_step(j)
        ev[j][1].record(stream)
    torch.cuda.synchronize()
    state.profile(False)
    phase_ms, phase_calls = state.profile_read()
    if ws > 1:
        dist.barrier()
    verify_ms = sum(a.elapsed_time(b) for a, b in ev)
    stream_ms = phase_ms["stream"]
    positions = sum(rec[(args.warmup + j) % R]["n"] for j in range(args.steps))
    vbytes = sum(rec[(args.warmup + j) % R]["vbytes"] for j in range(args.steps))
    sbytes = sum(rec[(args.warmup + j) % R]["sbytes"] for j in range(args.steps))
    code, _ = state.device_error()
    if code != 0 and not os.environ.get("DSDE_BENCH_IGNORE_ERRORS"):  # (set only for kernel experiments)
        raise SystemExit(f"device error {code} during the bench")

    t = torch.tensor([elapsed_ms, verify_ms, stream_ms, float(positions), float(vbytes), float(sbytes)],
                     dtype=torch.float64, device=dev)
    if ws > 1:
        mx = t[:3].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = t[3:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        elapsed_ms, verify_ms, stream_ms = float(mx[0]), float(mx[1]), float(mx[2])
        positions, vbytes, sbytes = float(tot[0]), float(tot[1]), float(tot[2])
    value = positions / (elapsed_ms / 1e3)

    # ---- e2e through the public API from pinned host buffers (rank-local, max over ranks)
    e2e = _e2e(args, m, step, rec, R, dev, ws, B)

    # ---- cpu baseline (rank 0, N = 1): the oracle on a bounded sample
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(args, rec, R)

    if rank == 0:
        peak, peak_kind = _peaks()
        # dominant kernel: the a1 stream kernel, timed by the library's per-launch events
        ach = (sbytes / ws) / (stream_ms / 1e3) / 1e9 if stream_ms > 0 else None
        vach = (vbytes / ws) / (verify_ms / 1e3) / 1e9 if verify_ms > 0 else None
        # DRAM read+write bytes per launch of the stream kernel: the ratio to the
        # algorithmic bytes measured on one ncu --set full launch (profiles/),
        # scaled to this run's per-launch algorithmic bytes
        trec = _traffic_record(f"cfg{args.config}")
        traffic = (trec["ratio"] * sbytes / ws / args.steps) if trec else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config_dict(args, cfg, ws),
            "roofline": {"bound": "hbm", "kernel": f"{STREAM_KERNEL} (a1: target + draft row of every draft position)",
                         "achieved": ach, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": (ach / peak) if ach else None,
                         "traffic": traffic,
                         "traffic_source": trec["source"] if trec else None,
                         "algorithmic_bytes_per_launch": sbytes / ws / args.steps,
                         "avg_launch_ms": stream_ms / args.steps},
            "timing": "value / ms_per_step: pass 1, only the two bracketing events in the region; roofline and "
                      "verify_pass: pass 2, the same replay with per-launch CUDA events on the launching stream",
            "verify_pass": {"kernels": list(phase_ms), "ms_per_step": {k: v / args.steps for k, v in phase_ms.items()},
                            "event_ms_per_step": verify_ms / args.steps,
                            "algorithmic_bytes_per_step": vbytes / ws / args.steps,
                            "achieved_gbs": vach, "frac": (vach / peak) if vach else None},
            "cpu_baseline": cpu,
            "e2e": e2e,
            # per step: dsde_step = stream + tail (+ cap partial/apply around NCCL at N > 1);
            # split calls: dsde_verify 2 (4 with DSDE_TAIL=split), update_signal 1, next_sl 1 (2 with NCCL)
            "gpu_launches": args.steps * ((2 + (0 if ws == 1 else 2)) if not args.split_calls else
                                          ((4 if os.environ.get("DSDE_TAIL") == "split" else 2) + 1 +
                                           (1 if ws == 1 else 2))),
            "clocks": sampler.summary(),
            "verify_ms_per_step": verify_ms / args.steps,
            "rows_per_s": None,
            "acceptance_rate": stats["acc"] / max(1, stats["pos"]),
            "block_efficiency": (stats["acc"] + stats["seqs"]) / max(1, stats["seqs"]),
            "mean_sl": stats["pos"] / max(1, stats["seqs"]),
            "residual_fraction": stats["resid"] / max(1, stats["seqs"]),
            "bonus_fraction": stats["bonus"] / max(1, stats["seqs"]),
            "recorded_steps": R,
        }
        rows = sum(rec[(args.warmup + j) % R]["rows"] for j in range(args.steps)) * ws
        line["rows_per_s"] = rows / (elapsed_ms / 1e3)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if ws > 1:
        dist.destroy_process_group()


def _e2e(args, m, step, rec, R, dev, ws, B):
    import torch
    import torch.distributed as dist
    n_e2e = min(args.e2e_steps, R)
    host = []
    for j in range(n_e2e):
        i = rec[j]["inp"]
        host.append(dict(cu=i.cu_sl.cpu().pin_memory(), tok=i.draft_tokens.cpu().pin_memory(),
                         t=i.target.cpu().pin_memory(), d=i.draft.cpu().pin_memory(),
                         s=i.seeds.cpu().pin_memory(), n=rec[j]["n"]))
    nmax = max(h["n"] for h in host)
    dt = torch.empty((nmax + B, host[0]["t"].shape[1]), dtype=torch.bfloat16, device=dev)
    dd = torch.empty((nmax, host[0]["t"].shape[1]), dtype=torch.bfloat16, device=dev)
    dtok = torch.empty(nmax, dtype=torch.int32, device=dev)
    dseed = torch.empty(nmax + B, dtype=torch.int64, device=dev)
    dcu = torch.empty(B + 1, dtype=torch.int32, device=dev)
    o_acc = torch.empty(B, dtype=torch.int32).pin_memory()
    o_em = torch.empty(nmax + B, dtype=torch.int32).pin_memory()
    o_nx = torch.empty(B, dtype=torch.int32).pin_memory()
    h2d = d2h = 0
    positions = 0
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for h in host:
        n = h["n"]
        dcu.copy_(h["cu"], non_blocking=True)
        dtok[:n].copy_(h["tok"], non_blocking=True)
        dt[:n + B].copy_(h["t"], non_blocking=True)
        dd[:n].copy_(h["d"], non_blocking=True)
        dseed[:n + B].copy_(h["s"], non_blocking=True)
        step(dcu, dtok[:n], dt[:n + B], dd[:n], dseed[:n + B], n)
        o_acc.copy_(step.accepted_len, non_blocking=True)
        o_em[:n + B].copy_(step.emitted[:n + B], non_blocking=True)
        o_nx.copy_(step.next_sl, non_blocking=True)
        h2d += (B + 1) * 4 + n * 4 + (n + B + n) * h["t"].shape[1] * 2 + (n + B) * 8
        d2h += B * 4 + (n + B) * 4 + B * 4
        positions += n
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    v = torch.tensor([ms, float(positions)], dtype=torch.float64, device=dev)
    if ws > 1:
        a = v[:1].clone()
        dist.all_reduce(a, op=dist.ReduceOp.MAX)
        b = v[1:].clone()
        dist.all_reduce(b, op=dist.ReduceOp.SUM)
        ms, positions = float(a[0]), float(b[0])
    return {"value": positions / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d // n_e2e,
            "d2h_bytes_per_step": d2h // n_e2e, "steps": n_e2e,
            "note": "pinned host -> HBM copies of each step's logits/tokens/seeds and D2H of "
                    "accepted_len/emitted/next_sl inside the timed region"}


def _cpu_baseline(args, rec, R):
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    positions, elapsed, n = 0, 0.0, 0
    budget = args.cpu_seconds
    j = 0
    while elapsed < budget and j < R:
        host = rec[j]["inp"].host_arrays()
        p, dt, _, _ = oracle_step_sample(host, args.cpu_seqs, cores, seed=j, greedy=args.greedy)
        positions += p
        elapsed += dt
        n += 1
        j += 1
    return {"value": positions / elapsed, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{args.cpu_seqs} sequences x {n} recorded steps of the same workload "
                      f"({positions} positions, {elapsed:.1f} s, {cores} threads, verify only)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--seed", type=int, default=2509)
    ap.add_argument("--preroll", type=int, default=32)
    ap.add_argument("--record", type=int, default=24)
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--cpu-seqs", type=int, default=128)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seqs", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--greedy", action="store_true",
                    help="T = 0 verification (dsde_config.greedy; draft tokens = draft argmax)")
    ap.add_argument("--entropy", action="store_true",
                    help="also compute the draft entropy H(q) per draft row (dsde_set_draft_entropy, SURVEY f2)")
    ap.add_argument("--split-calls", action="store_true",
                    help="time dsde_verify + dsde_update_signal + dsde_next_sl instead of one dsde_step")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run(args)


if __name__ == "__main__":
    main()
