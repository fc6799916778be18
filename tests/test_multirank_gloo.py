"""N > 1 path on CPU: world_size-2 torch.distributed (gloo) runs of the batch
partition of SURVEY §8(e).

Each rank owns a contiguous shard of the batch (as bench.py shards it), forms
the exact int64 cap partial (sum SL^, N active, max SL^) of its shard, and the
partials are all-reduced (sum, + max for cap_mode 0) exactly as dsde_next_sl
does over NCCL. The cap is then applied with the library's host-callable rule
(dsde_cap_value, the same code the device kernels use) and must equal the
single-process cap of the whole batch (oracle.next_sl) on every rank, for any
shard sizes (ragged included). No GPU is needed: the collective is gloo and the
cap rule is a host function of libdsde.so.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2509_01083_b200 as m
        res = []
        for cap_mode, sl, cal, cuts in cases:
            lo, hi = cuts[rank], cuts[rank + 1]
            mine, mine_cal = sl[lo:hi], cal[lo:hi]
            act = mine_cal == 0
            part = torch.tensor([int(mine[act].sum()), int(act.sum())], dtype=torch.int64)
            mx = torch.tensor([int(mine[act].max()) if act.any() else 0], dtype=torch.int64)
            dist.all_reduce(part, op=dist.ReduceOp.SUM)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            cfg = m.Config.default(cap_mode=cap_mode)
            cap = m.cap_value(cfg, int(part[0]), int(part[1]), int(mx[0]))
            # next SL of this rank's shard, as k_cap_apply forms it
            nxt = np.where(mine_cal != 0, cfg.calib_sl, np.minimum(mine, cap))
            res.append((cap, nxt.tolist()))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _cases():
    r = np.random.default_rng(7)
    cases = []
    for t in range(24):
        B = int(r.integers(2, 300))
        sl = r.integers(2, 9, B).astype(np.int64)
        cal = (r.random(B) < 0.15).astype(np.int64)
        if t == 0:
            cal[:] = 1  # every sequence calibrating: cap = ceiling
        cut = int(r.integers(0, B + 1)) if t % 3 else B // 2  # ragged shards, empty shards too
        cases.append((0 if t % 4 == 3 else 1, sl, cal, [0, cut, B]))
    return cases


@pytest.mark.timeout(180)
def test_cap_allreduce_world2_matches_single_process():
    cases = _cases()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, 2, port, cases, q)) for rk in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=150) for _ in procs)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for ci, (cap_mode, sl, cal, cuts) in enumerate(cases):
        cfg = oracle.Config(cap_mode=cap_mode)
        nxt_o, cap_o = oracle.next_sl(cfg, sl.astype(np.int32), cal.astype(np.int32))
        for rk in range(2):
            cap, nxt = got[rk][ci]
            assert cap == cap_o, (ci, rk, cap, cap_o)
            assert nxt == nxt_o[cuts[rk]:cuts[rk + 1]].tolist(), (ci, rk)
