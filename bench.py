#!/usr/bin/env python
"""bench.py — throughput of the DSDE verification hot path on B200.

One "step" = one pass of the whole hot path over one
batch: one dsde_step call = verify (a1-a4) + signal / SL^ (a5-a6) + cap (a7),
i.e. the row stream k_stream_ldg and the tail k_tail (with the NCCL cap
all-reduce between two small kernels when N > 1).

Workloads (BASELINE.json configs, --config): 1 = B 4, V 32000 fp32, SL <= 4;
2 = B 64, V 32000 bf16, code + dialogue; 3 (default) = B 256 per GPU,
V 128256 bf16, code profile (N = 8 is config 5's B = 2048 sharded, weak
scaling); 4 = B 512, V 128256, low acceptance; 5 = B 2048 in total, V 128256,
mixed profiles, sharded 2048/N per rank (strong scaling). SLs are chosen by
DSDE itself (closed loop).

Measurement:
  * record: after a pre-roll (calibration + settling), R closed-loop steps are
    run once and their inputs kept resident in HBM (a distinct input set per
    step, ~0.7-1.1 GB at config 3, so every timed step reads its logits from
    HBM, not L2); their outputs are kept for the parity check;
  * replay: the state is restored to the start of the recording, W warm-up
    steps run, then K timed steps replay the recorded steps in order (cyclically
    if K + W > R), bracketed by barrier + synchronize, CUDA events on the
    launching stream, max over ranks (pass 1: nothing else in the region);
  * roofline (pass 2, the same replay with the library's per-launch events):
    the dominant kernel k_stream_ldg's algorithmic bytes (the
    target + draft row of every draft position) over its own CUDA-event time,
    against MEASURED_PEAKS.json hbm_gbs; `whole_step` = the step's algorithmic
    bytes (plus the bonus row of every fully accepted sequence) over pass 1's
    ms_per_step;
  * parity: the fp64 oracle (oracle/, test infrastructure) recomputes a fixed
    sample of sequences of every recorded step it has time for and compares
    them with the GPU's outputs (tests/parity.py bands; ties counted);
  * e2e: the same metric through the public Python API from pinned host buffers
    (H2D of the step inputs and D2H of the results inside the timed region);
  * cpu_baseline: the oracle (verify + signal + cap) on that bounded sample, on
    the host cores, rank 0, N = 1 only; plus a 1-thread figure and the CPU model.
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
STREAM_KERNEL = "k_stream_ldg"

CONFIGS = {
    # BASELINE.json configs[0]: the small case (closed loop, correctness config)
    1: dict(B=4, V=32000, profiles=("code",), ceiling=4, dtype="f32", name="cfg1: B=4, SL<=4, V=32000 fp32 "
            "logits (DSDE closed loop)"),
    # BASELINE.json configs[1]
    2: dict(B=64, V=32000, profiles=("code", "dialogue"), ceiling=8, name="cfg2: B=64, SL<=8, V=32000 bf16, "
            "mixed code/dialogue (DSDE closed loop)"),
    # BASELINE.json configs[2]: the N=1 workload (and the per-rank shard at N>1)
    3: dict(B=256, V=128256, profiles=("code",), ceiling=8, name="cfg3: B=256/GPU, SL<=8 (DSDE closed loop), "
            "V=128256 bf16 logits, high-acceptance (code) profile"),
    # BASELINE.json configs[3]
    4: dict(B=512, V=128256, profiles=("low",), ceiling=8, name="cfg4: B=512/GPU, SL<=8 (DSDE closed loop), "
            "V=128256 bf16 logits, low-acceptance profile"),
    # BASELINE.json configs[4]: B=2048 in total, sharded over the ranks (2048/N each)
    5: dict(B=2048, V=128256, profiles=("code", "dialogue", "low"), ceiling=8, strong=True,
            name="cfg5: B=2048 total sharded over the GPUs, SL<=8 (DSDE closed loop), V=128256 bf16, "
                 "mixed code/dialogue/low profiles, cap via NCCL"),
    # the Gemma-27B/2B pair of the paper's low-acceptance study (eager-mode V)
    6: dict(B=256, V=256000, profiles=("low",), ceiling=8, name="cfg6 (SURVEY f4): B=256/GPU, SL<=8 (DSDE "
            "closed loop), V=256000 bf16 (Gemma-like), low-acceptance profile"),
}


def _resample(args) -> int:
    """dsde_config.resample / oracle reading of the recovery draw (D23 or D7)."""
    return 0 if getattr(args, "resample", "full") == "proposal" else 1


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


def _torch_dtype(cfg):
    import torch
    return torch.float32 if cfg.get("dtype") == "f32" else torch.bfloat16


def _per_rank_B(cfg, ws):
    if cfg.get("strong"):
        if cfg["B"] % ws:
            raise SystemExit(f"config B={cfg['B']} does not split over {ws} ranks")
        return cfg["B"] // ws
    return cfg["B"]


def run_reference(args):
    """--impl reference: the fp64 oracle on the host cores (verify + signal + cap),
    a bounded sample of the workload's sequences per step."""
    ws, rank, _ = _dist_env()
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    cfg = CONFIGS[args.config]
    tdt = _torch_dtype(cfg)
    nthreads = os.cpu_count() or 1
    per_step = min(args.ref_seqs, _per_rank_B(cfg, ws) * ws)
    w = synth.Workload(B=per_step, V=cfg["V"], dtype=tdt, profiles=cfg["profiles"], seed=args.seed,
                       greedy_draft=args.greedy)
    ost = oracle.OracleState(oracle.Config(sl_ceiling=cfg["ceiling"], calib_sl=min(4, cfg["ceiling"])), per_step)
    k = np.full(per_step, min(4, cfg["ceiling"]))
    positions, elapsed = 0, 0.0
    odt = oracle.F32 if cfg.get("dtype") == "f32" else oracle.BF16
    for s in range(args.warmup + args.steps):
        host = synth.generate_step(w, s, k, device="cpu").host_arrays()
        t0 = time.perf_counter()
        r = oracle.verify(host["cu_sl"], host["draft_tokens"], host["target"], host["draft"], host["seeds"],
                          odt, nthreads=nthreads, greedy=args.greedy, resample=_resample(args))
        sl, cal, _ = ost.update_signal(np.arange(per_step), host["cu_sl"], r.kld, r.accepted_len)
        nx, cap = oracle.next_sl(ost.cfg, sl, cal)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            positions += int(k.sum())
            elapsed += dt
        k = nx.astype(np.int64)
    value = positions / elapsed
    conf = _config_dict(args, cfg, args.gpus)
    conf.update({"B_per_gpu": per_step, "global_batch": per_step,
                 "sample": f"{per_step} sequences of the {cfg['name'].split(':')[0]} workload per step "
                           f"(the oracle cannot run the full batch in minutes)"})
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": conf,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                         "cpu_model": _cpu_model(),
                         "sample": f"{per_step} sequences per step, DSDE closed loop (verify + signal + cap), "
                                   f"V={cfg['V']} {cfg.get('dtype', 'bf16')}, {nthreads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(args, cfg, n):
    B = _per_rank_B(cfg, n)
    return {"workload": cfg["name"], "B_per_gpu": B, "global_batch": B * n, "V": cfg["V"],
            "logits": cfg.get("dtype", "bf16"), "sl_ceiling": cfg["ceiling"], "profiles": list(cfg["profiles"]),
            "parallelism": f"dp{n}", "l2": "inputs larger than L2: a distinct input set per replayed step "
                                         "(HBM-resident recording, cyclic)" if cfg["V"] > 100000 else
            "one distinct input set per replayed step (R of them, cyclic; a step's set is smaller than L2)",
            "replay": "recorded closed-loop DSDE steps replayed in order (cyclic if K+W > R)",
            "verify": "greedy (T=0, draft argmax tokens)" if args.greedy else "rejection sampling (T=1)",
            "recovery_draw": "D23 proposals from p (then D7)" if _resample(args) == 0 else "D7 full residual CDF",
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
    B, V = _per_rank_B(cfg, ws), cfg["V"]
    tdt = _torch_dtype(cfg)
    esz = 4 if tdt == torch.float32 else 2
    m.lib()
    comm = None
    if ws > 1:
        uid = [m.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = m.Comm(uid[0], ws, rank)
    mcfg = m.Config.default(sl_ceiling=cfg["ceiling"], calib_sl=min(4, cfg["ceiling"]), greedy=int(args.greedy),
                              resample=_resample(args))
    state = m.State(mcfg, B)
    step = m.Step(state, B, V, tdt, comm=comm)
    if args.entropy:  # the fused draft entropy in the same stream pass
        state.set_draft_entropy(torch.empty(B * 16, dtype=torch.float32, device=dev))
    w = synth.Workload(B=B, V=V, dtype=tdt, profiles=cfg["profiles"], seed=args.seed + 7919 * rank,
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
    # ---- record R closed-loop steps (inputs resident in HBM), bounded by memory
    per_step_bytes = (2 * B * cfg["ceiling"] + B) * V * esz
    free, _ = torch.cuda.mem_get_info(dev)
    R = max(1, min(args.record, args.warmup + args.steps, int(0.5 * free // max(1, per_step_bytes))))
    snap = state.export()
    rec, stats = [], dict(pos=0, acc=0, resid=0, bonus=0, seqs=0, rows=0, vbytes=0, sbytes=0)
    for r in range(R):
        inp = synth.generate_step(w, s, k, device=dev)
        n = int(k.sum())
        out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n)
        acc = out.accepted_len.cpu().numpy()
        nx = out.next_sl.cpu().numpy().astype(np.int64)
        bonus = int(np.sum(acc == k))
        rows = 2 * n + bonus
        # SURVEY §8(d) algorithmic bytes: logits of every draft position's row pair and of
        # every bonus row, tokens, seeds, outputs (kld, emitted, flags, accepted_len)
        vbytes = rows * V * esz + n * 4 + (n + B) * 8 + n * 4 + (n + B) * 5 + B * 4
        sbytes = 2 * n * V * esz  # the stream kernel's rows: target + draft row of every draft position
        rec.append(dict(inp=inp, n=n, k=k.copy(), rows=rows, vbytes=vbytes, sbytes=sbytes, next=nx, acc=acc.copy(),
                        emitted=out.emitted.cpu().numpy().copy(), kld=out.kld.cpu().numpy().copy()))
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
        step(i.cu_sl, i.draft_tokens, i.target, i.draft, i.seeds, e["n"], fused=not args.split_calls)

    def run_step(j):
        replay(args.warmup + j)

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
    # the replay reproduces the recording (verify outputs depend only on the inputs)
    last = rec[(args.warmup + args.steps - 1) % R]
    replay_identical = bool(np.array_equal(step.accepted_len.cpu().numpy(), last["acc"]) and
                            np.array_equal(step.kld[:last["n"]].cpu().numpy().view(np.uint32),
                                           last["kld"][:last["n"]].view(np.uint32)))

    # ---- pass 2 (kernel times for the roofline): the same replay with the
    # library's per-launch events (dsde_profile_*) and per-step events on the
    # launching stream; events cost a few us per step, so they stay out of pass 1
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
    step_ms2 = sum(a.elapsed_time(b) for a, b in ev)
    pass_ms = phase_ms["stream"]
    positions = sum(rec[(args.warmup + j) % R]["n"] for j in range(args.steps))
    vbytes = sum(rec[(args.warmup + j) % R]["vbytes"] for j in range(args.steps))
    sbytes = sum(rec[(args.warmup + j) % R]["sbytes"] for j in range(args.steps))
    code, _ = state.device_error()
    if code != 0 and not os.environ.get("DSDE_BENCH_IGNORE_ERRORS"):  # (set only for kernel experiments)
        raise SystemExit(f"device error {code} during the bench")

    # ---- multi-GPU: the cap all-reduce on its own (dsde_next_sl with and
    # without the communicator), and the per-rank row imbalance
    multi = None
    if ws > 1:
        multi = _allreduce_cost(m, state, step, comm, B, dist, stream)
    t = torch.tensor([elapsed_ms, step_ms2, pass_ms, float(positions), float(vbytes), float(sbytes)],
                     dtype=torch.float64, device=dev)
    if ws > 1:
        mx = t[:3].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = t[3:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        rows_r = torch.tensor([float(positions)], dtype=torch.float64, device=dev)
        allrows = [torch.zeros_like(rows_r) for _ in range(ws)]
        dist.all_gather(allrows, rows_r)
        allrows = [float(x.item()) for x in allrows]
        multi["positions_per_rank_max_over_mean"] = max(allrows) / (sum(allrows) / ws)
        multi["positions_per_rank"] = allrows
        elapsed_ms, step_ms2, pass_ms = float(mx[0]), float(mx[1]), float(mx[2])
        positions, vbytes, sbytes = float(tot[0]), float(tot[1]), float(tot[2])
    value = positions / (elapsed_ms / 1e3)

    # ---- e2e through the public API from pinned host buffers (rank-local, max over ranks)
    e2e = _e2e(args, m, step, rec, R, dev, ws, B)

    # ---- cpu baseline + parity sample (rank 0, N = 1): the oracle on a bounded sample
    cpu, par = None, None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu, par = _cpu_baseline(args, cfg, rec, R)

    if rank == 0:
        peak, peak_kind = _peaks()
        ach = (sbytes / ws) / (pass_ms / 1e3) / 1e9 if pass_ms > 0 else None
        trec = _traffic_record(f"cfg{args.config}")
        traffic = (trec["ratio"] * sbytes / ws / args.steps) if trec else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": _config_dict(args, cfg, ws),
            "roofline": {"bound": "hbm",
                         "kernel": f"{STREAM_KERNEL} (a1, the row stream: the dominant kernel)",
                         "achieved": ach, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": (ach / peak) if ach else None,
                         "traffic": traffic,
                         "traffic_source": trec["source"] if trec else None,
                         "algorithmic_bytes_per_launch": sbytes / ws / args.steps,
                         "avg_launch_ms": pass_ms / args.steps},
            "timing": "value / ms_per_step: pass 1, only the two bracketing events in the region; roofline: "
                      "pass 2, the same replay with per-launch CUDA events on the launching stream",
            "phases_ms_per_step": {k_: v / args.steps for k_, v in phase_ms.items()},
            "step_pass2_ms": step_ms2 / args.steps,
            "whole_step": {"algorithmic_bytes_per_step": vbytes / ws / args.steps,
                           "achieved_gbs": (vbytes / ws) / (elapsed_ms / 1e3) / 1e9,
                           "frac": (vbytes / ws) / (elapsed_ms / 1e3) / 1e9 / peak},
            "cpu_baseline": cpu,
            "parity": par,
            "replay_identical": replay_identical,
            "e2e": e2e,
            # our kernels per step: k_stream_ldg + k_tail; split calls: + k_update_signal +
            # k_cap_local; N > 1: + k_cap_partial / k_cap_apply
            "gpu_launches": args.steps * ((2 if ws == 1 else 4) if not args.split_calls else (4 if ws == 1 else 5)),
            "clocks": sampler.summary(),
            "multi_gpu": multi,
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


def _allreduce_cost(m, state, step, comm, B, dist, stream, iters=200):
    """Device time of dsde_next_sl with the communicator (k_cap_partial + the NCCL
    int64 all-reduce + k_cap_apply) minus the single-GPU dsde_next_sl (k_cap_local)."""
    import torch
    snap = state.export()

    def timed(c):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(iters):
            m.dsde_next_sl(state, step.slots, step.sl_hat, None, step.next_sl, step.cap, c)
        b.record(stream)
        torch.cuda.synchronize()
        v = torch.tensor([a.elapsed_time(b) / iters * 1e3], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    with_comm = timed(comm)
    local = timed(None)
    state.load(snap)
    return {"cap_with_allreduce_us": with_comm, "cap_local_us": local,
            "allreduce_us": with_comm - local, "collective": "ncclAllReduce int64[2] sum (cap_mode 1)"}


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
    ldt = host[0]["t"].dtype
    esz = host[0]["t"].element_size()
    dt = torch.empty((nmax + B, host[0]["t"].shape[1]), dtype=ldt, device=dev)
    dd = torch.empty((nmax, host[0]["t"].shape[1]), dtype=ldt, device=dev)
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
        h2d += (B + 1) * 4 + n * 4 + (n + B + n) * h["t"].shape[1] * esz + (n + B) * 8
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


def _cpu_baseline(args, cfg, rec, R):
    """The oracle (verify + signal + cap) on a fixed sample of sequences of the
    recorded steps, timed on the host cores, and the parity of those sequences'
    GPU outputs (accepted lengths, tokens, KLDs) against it."""
    import oracle
    from tests import parity
    oracle.build()
    cores = os.cpu_count() or 1
    B = len(rec[0]["acc"])
    ids = np.sort(np.random.default_rng(args.seed).choice(B, min(args.cpu_seqs, B), replace=False))
    ost = oracle.OracleState(oracle.Config(sl_ceiling=cfg["ceiling"], calib_sl=min(4, cfg["ceiling"])), len(ids))
    odt = oracle.F32 if cfg.get("dtype") == "f32" else oracle.BF16
    rep = parity.Report()
    positions, elapsed, n = 0, 0.0, 0
    while elapsed < args.cpu_seconds and n < R:
        e = rec[n]
        host = e["inp"].host_arrays()
        sub = parity.subset_batch(host, ids)
        t0 = time.perf_counter()
        o = oracle.verify(sub["cu_sl"], sub["draft_tokens"], sub["target"], sub["draft"], sub["seeds"], odt,
                          nthreads=cores, greedy=args.greedy, resample=_resample(args))
        sl, cal, _ = ost.update_signal(np.arange(len(ids)), sub["cu_sl"], o.kld, o.accepted_len)
        oracle.next_sl(ost.cfg, sl, cal)
        elapsed += time.perf_counter() - t0
        positions += int(sub["cu_sl"][-1])
        a2, e2, k2 = parity.gather_subset_outputs(host["cu_sl"], ids, e["acc"], e["emitted"], e["kld"])
        rep.merge(parity.compare_verify(sub["cu_sl"], a2, e2, k2, o, seq_ids=ids))
        n += 1
    # one thread, a smaller sample (a few seconds)
    host = rec[0]["inp"].host_arrays()
    sub1 = parity.subset_batch(host, ids[:max(1, min(len(ids), 8))])
    t0 = time.perf_counter()
    oracle.verify(sub1["cu_sl"], sub1["draft_tokens"], sub1["target"], sub1["draft"], sub1["seeds"], odt,
                  nthreads=1, greedy=args.greedy, resample=_resample(args))
    one = int(sub1["cu_sl"][-1]) / (time.perf_counter() - t0)
    cpu = {"value": positions / elapsed, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
           "one_thread_value": one,
           "sample": f"{len(ids)} fixed sequences x {n} recorded steps of the same workload "
                     f"({positions} positions, {elapsed:.1f} s, {cores} threads, verify + signal + cap); "
                     f"one_thread_value: verify of {len(sub1['cu_sl']) - 1} sequences on 1 thread"}
    par = {"ok": rep.ok(), "seqs_checked": rep.seqs, "positions_checked": rep.positions,
           "steps_checked": n, "accept_ties": rep.accept_ties, "sample_ties": rep.sample_ties,
           "kl_max_rel": rep.kl_max_rel, "kl_out_of_band": rep.kl_bad, "mismatches": len(rep.mismatches),
           "bands": "accepted lengths / tokens bit-exact outside counted |u - p/q| < 1e-6 ties; "
                    "KLD |err| <= 1e-5 |KL| + 1e-9 (tests/parity.py)"}
    return cpu, par


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
    ap.add_argument("--resample", default="full", choices=["proposal", "full"],
                    help="the recovery draw's reading: D7 full residual CDF (default) or D23 proposals from p")
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
