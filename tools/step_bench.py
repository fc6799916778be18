"""Quick kernel timing of dsde_verify / dsde_step on fixed synthetic inputs
(measurement only; no closed loop, so it also runs on experiment builds whose
outputs are not meaningful). Prints the median µs per call over --iters calls
and the achieved algorithmic GB/s of the logit rows (2 rows per draft position
+ the bonus rows reported by the call).

usage: python tools/step_bench.py [--config 3] [--iters 30] [--sets 3]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_01083_b200 as m  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--sets", type=int, default=3, help="distinct input sets, rotated (L2 flush)")
    ap.add_argument("--kmean", type=float, default=5.0)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    B, V = cfg["B"], cfg["V"]
    tdt = torch.float32 if cfg.get("dtype") == "f32" else torch.bfloat16
    esz = 4 if tdt == torch.float32 else 2
    st = m.State(m.Config.default(sl_ceiling=cfg["ceiling"], calib_steps=0), B)
    step = m.Step(st, B, V, tdt)
    w = synth.Workload(B=B, V=V, dtype=tdt, profiles=cfg["profiles"], seed=5)
    rng = np.random.default_rng(1)
    sets = []
    for s in range(args.sets):
        k = np.clip(rng.poisson(args.kmean, B), 1, cfg["ceiling"])
        sets.append((synth.generate_step(w, s + 50, k, device="cuda"), int(k.sum())))
    # outputs of one call per set (for the bonus-row count), then timed batches
    # of back-to-back calls (the GPU never idles waiting for the host)
    rows = []
    for inp, n in sets:
        out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n)
        torch.cuda.synchronize()
        acc = out.accepted_len.cpu().numpy()
        k = np.diff(inp.cu_sl.cpu().numpy())
        rows.append(2 * n + int(np.sum(acc == k)))
    times = []
    for rep in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for it in range(args.iters):
            inp, n = sets[it % len(sets)]
            step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, n)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e3 / args.iters)
    t = float(np.median(times))
    byt = float(np.mean(rows)) * V * esz
    print(f"cfg{args.config} B={B} V={V}: {t:.1f} us/call (p10 {np.percentile(times, 10):.1f}, "
          f"p90 {np.percentile(times, 90):.1f}), {byt / t / 1e3:.0f} GB/s algorithmic, "
          f"positions/call {np.mean([s[1] for s in sets]):.0f}, err={st.device_error()}")


if __name__ == "__main__":
    main()
