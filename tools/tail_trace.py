"""Phase trace of k_tail (measurement only). Rebuild the library with
DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 first; then this runs a few closed-loop
dsde_step calls of a bench config and prints the globaltimer phases of each
CTA's first sequence relative to the earliest post-wait stamp (µs): wait
(start -> after griddepcontrol.wait), finalize, layout, draw, select, split
by the draw mode.

usage: DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 python paper_2509_01083_b200/_build.py --force
       python tools/tail_trace.py [--config 3] [--steps 8]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (CONFIGS)
import paper_2509_01083_b200 as m  # noqa: E402
import synth  # noqa: E402

MODES = {0: "none", 1: "resid", 2: "bonus", 3: "error", 4: "argmax"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--resample", type=int, default=0, help="dsde_config.resample (0: D23, 1: D7)")
    ap.add_argument("--layout-end", action="store_true", help="trace build 4: slot 7 = seq_layout's own end")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    B, V = cfg["B"], cfg["V"]
    L = m.lib()
    fn = L.dsde_debug_tail_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    mcfg = m.Config.default(sl_ceiling=cfg["ceiling"], calib_sl=min(4, cfg["ceiling"]), resample=args.resample)
    state = m.State(mcfg, B)
    step = m.Step(state, B, V, torch.bfloat16)
    w = synth.Workload(B=B, V=V, dtype=torch.bfloat16, profiles=cfg["profiles"], seed=0)
    k = np.full(B, mcfg.calib_sl, dtype=np.int64)
    rows = []
    for s in range(args.steps):
        inp = synth.generate_step(w, s, k, device="cuda")
        out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, int(k.sum()))
        torch.cuda.synchronize()
        k = out.next_sl.cpu().numpy().astype(np.int64)
        if s < args.steps // 2:
            continue
        n = min(B, 8192)
        buf = (ctypes.c_ulonglong * (8 * n))()
        assert fn(buf, n) == 0
        a = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
        t0 = a[:, 1].min()
        slot7 = (a[:, 7] - a[:, 2]) if args.layout_end else a[:, 7]
        rows.append(np.stack([(a[:, 1] - a[:, 0]), a[:, 2] - a[:, 1], a[:, 3] - a[:, 2], a[:, 4] - a[:, 3],
                              a[:, 5] - a[:, 4], a[:, 5] - t0, a[:, 6] & 0xff, slot7], 1))
    r = np.concatenate(rows).astype(np.float64)
    r[:, :6] /= 1e3
    print(f"cfg{args.config} B={B}: per CTA (first sequence), µs: wait / finalize / layout / draw / select / end-from-first")
    for mode in np.unique(r[:, 6]).astype(int):
        x = r[r[:, 6] == mode]
        print(f"  {MODES.get(mode, mode):6s} n={len(x):5d} mean " + " / ".join(f"{v:6.2f}" for v in x[:, :6].mean(0))
              + "   max " + " / ".join(f"{v:6.2f}" for v in x[:, :6].max(0))
              + (f"   D23 first proposal of the last round: mean {x[:, 7].mean():.1f} max {x[:, 7].max():.0f}"
                 if mode == 1 and 0 < x[:, 7].max() < 1000 else "")
              + (f"   (trace 2/3) repeated select / draw: mean {x[:, 7][x[:, 7] > 0].mean() / 1e3:.2f} us"
                 if x[:, 7].max() >= 1000 else ""))


if __name__ == "__main__":
    main()
