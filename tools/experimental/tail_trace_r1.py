"""Phase trace of k_tail (measurement only). Rebuild the library with
DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 first; then this replays a few closed-loop
steps of a bench config and prints, per CTA, the globaltimer phases after the
PDL wait: finalize, draw masses, select (µs), split by draw mode.

usage: DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 python paper_2509_01083_b200/_build.py --force
       python tools/tail_trace.py [--config 3] [--steps 6]
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
    ap.add_argument("--steps", type=int, default=40)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    B, V = cfg["B"], cfg["V"]
    L = m.lib()
    fn = L.dsde_debug_tail_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    mcfg = m.Config.default(sl_ceiling=cfg["ceiling"], calib_sl=min(4, cfg["ceiling"]))
    state = m.State(mcfg, B)
    step = m.Step(state, B, V, torch.bfloat16)
    w = synth.Workload(B=B, V=V, dtype=torch.bfloat16, profiles=cfg["profiles"], seed=0)
    dev = torch.device("cuda", 0)
    k = np.full(B, mcfg.calib_sl, dtype=np.int64)
    buf = np.zeros(B * 6, dtype=np.uint64)
    agg = {}
    for s in range(args.steps):
        inp = synth.generate_step(w, s, k, device=dev)
        out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, int(k.sum()))
        k = out.next_sl.cpu().numpy().astype(np.int64)
        torch.cuda.synchronize()
        if s < args.steps - 4:
            continue
        assert fn(buf.ctypes.data, B) == 0
        t = buf.reshape(B, 6).astype(np.int64)
        t0 = t[:, 0].min()
        mode = (t[:, 5] & 0xFF).astype(int)
        sm = (t[:, 5] >> 8).astype(int)
        print(f"step {s}: Σk={int(k.sum())} span {(t[:, 3].max() - t0) / 1e3:.1f} µs; wait-release spread "
              f"{(t[:, 0].max() - t0) / 1e3:.1f} µs; SMs used {len(set(sm))}")
        for md in sorted(set(mode)):
            sel = mode == md
            fin = (t[sel, 1] - t[sel, 0]) / 1e3
            drw = (t[sel, 2] - t[sel, 1]) / 1e3
            slc = (t[sel, 3] - t[sel, 2]) / 1e3
            srch = (t[sel, 4] - t[sel, 2]) / 1e3 if md in (1, 2) else slc * 0
            end = (t[sel, 3] - t0) / 1e3
            print(f"  {MODES.get(md, md):7s} n={sel.sum():4d} finalize {fin.mean():5.1f} (max {fin.max():5.1f})  "
                  f"draw {drw.mean():5.1f} (max {drw.max():5.1f})  select {slc.mean():5.1f} (max {slc.max():5.1f})  "
                  f"(search {srch.mean():4.1f})  end max {end.max():5.1f}")
        last = int(np.argmax(t[:, 3]))
        print(f"  last CTA {last} ({MODES.get(int(mode[last]))}, SM {sm[last]}, "
              f"{int(np.sum(sm == sm[last]))} CTAs on it): start {(t[last, 0] - t0) / 1e3:.1f} "
              f"fin {(t[last, 1] - t[last, 0]) / 1e3:.1f} draw {(t[last, 2] - t[last, 1]) / 1e3:.1f} "
              f"sel {(t[last, 3] - t[last, 2]) / 1e3:.1f} (search {(t[last, 4] - t[last, 2]) / 1e3:.1f})")


if __name__ == "__main__":
    main()
