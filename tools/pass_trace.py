"""Timeline trace of the persistent pass kernel k_pass (measurement only).

Rebuild the library with DSDE_NVCC_FLAGS=-DDSDE_PASS_TRACE=1 first; then this
replays closed-loop steps of a bench config and prints, for the last step, the
distribution over warps of (stream-loop end, kernel end, blocking-wait time,
deferred draws, finalizes, draw units) and over sequences of (last row done,
published, token selected), all in µs from the kernel's first warp start.

usage: DSDE_NVCC_FLAGS=-DDSDE_PASS_TRACE=1 python paper_2509_01083_b200/_build.py --force
       python tools/pass_trace.py [--config 3] [--steps 8]
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


def pct(x, qs=(0, 10, 50, 90, 100)):
    x = np.asarray(x, dtype=np.float64)
    return " ".join(f"p{q}={np.percentile(x, q):8.1f}" for q in qs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=8)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    B, V = cfg["B"], cfg["V"]
    L = m.lib()
    fn = L.dsde_debug_pass_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    mcfg = m.Config.default(sl_ceiling=cfg["ceiling"], calib_sl=min(4, cfg["ceiling"]))
    state = m.State(mcfg, B)
    tdt = torch.float32 if cfg.get("dtype") == "f32" else torch.bfloat16
    step = m.Step(state, B, V, tdt)
    w = synth.Workload(B=B, V=V, dtype=tdt, profiles=cfg["profiles"], seed=0)
    k = np.full(B, mcfg.calib_sl, dtype=np.int64)
    for s in range(args.steps):
        inp = synth.generate_step(w, s, k, device="cuda")
        torch.cuda.synchronize()
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        out = step(inp.cu_sl, inp.draft_tokens, inp.target, inp.draft, inp.seeds, int(k.sum()))
        ev[1].record()
        torch.cuda.synchronize()
        k = out.next_sl.cpu().numpy().astype(np.int64)
    nw = 8192
    wt = np.zeros(nw * 8, dtype=np.uint64)
    st = np.zeros(4096 * 4, dtype=np.uint64)
    assert fn(wt.ctypes.data, nw, st.ctypes.data, 4096) == 0
    wt = wt.reshape(nw, 8).astype(np.int64)
    st = st.reshape(4096, 4).astype(np.int64)[:B]
    used = wt[:, 0] > 0
    wt = wt[used]
    t0 = wt[:, 0].min()
    us = lambda x: (x - t0) / 1e3  # noqa: E731
    print(f"cfg{args.config} B={B} positions={int(k.sum())} step event ms={ev[0].elapsed_time(ev[1]):.3f} "
          f"warps={used.sum()}")
    print("warp start   ", pct(us(wt[:, 0])))
    print("loop end     ", pct(us(wt[:, 1])))
    print("warp end     ", pct(us(wt[:, 2])))
    print("wait us      ", pct(wt[:, 3] / 1e3))
    print("defers       ", pct(wt[:, 4]), "total", wt[:, 4].sum())
    print("row finalizes", pct(wt[:, 5]), "total", wt[:, 5].sum())
    print("seq finalizes", pct(wt[:, 6]), "total", wt[:, 6].sum())
    print("draw units   ", pct(wt[:, 7]), "total", wt[:, 7].sum())
    print("seq last row ", pct(us(st[:, 0])))
    print("seq published", pct(us(st[:, 1])))
    print("seq selected ", pct(us(st[:, 2])))
    print("publish - lastrow us", pct((st[:, 1] - st[:, 0]) / 1e3))
    print("select - publish us ", pct((st[:, 2] - st[:, 1]) / 1e3))
    order = np.argsort(st[:, 0])
    print("last-row time by sequence index (every 16th):",
          " ".join(f"{i}:{us(st[i, 0]):.0f}" for i in range(0, B, max(1, B // 16))))


if __name__ == "__main__":
    main()
