"""The vocabulary-parallel exchange pattern (include/dsde.h
dsde_vp_*) on CPU with world_size-2 gloo.

Each rank holds a column shard [v0, v1) of every target and draft row (the
split at a multiple of the 2048-token stream slice, as dsde_vp_sizes places
it) and only ever touches its own columns. It forms exact fp64 per-shard row
statistics (max and scaled sums of t and d, the scaled sum of e^t (t - d)) and
the owner of each draft token contributes (t_x, d_x); these are all-gathered
/ all-reduced (sum), and every rank combines them into the same KLD, accept
test and first rejection. The drawn row's per-shard masses (residual
max(0, p - q) or bonus p) are all-gathered; every rank finds the crossing
shard, whose owner scans its columns for the token; an all-reduce (max) gives
it to all ranks. The result must equal the single-process oracle on the full
rows: accepted lengths and tokens exactly, KLD to 1e-12. (The GPU stages do
the same with slice partials and NCCL; tests/test_gpu_vocab.py checks them
bit for bit against the unsharded kernels.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch(V, k, seed):
    r = np.random.default_rng(seed)
    B = len(k)
    cu = synth.cu_from_k(k)
    nk = int(cu[-1])
    t = (r.normal(0, 3, (nk + B, V))).astype(np.float32)
    tgt = np.concatenate([[cu[i] + i + j for j in range(k[i])] for i in range(B)])
    d = (t[tgt] + r.normal(0, 0.8, (nk, V)) + r.uniform(-2, 2, (nk, 1))).astype(np.float32)
    tok = np.array([int(np.argmax(d[j] - np.log(-np.log(r.random(V))))) for j in range(nk)], np.int32)
    return cu, tok, t, d, synth.slot_seeds(seed, 0, cu)


def _gather(x: np.ndarray, world: int) -> np.ndarray:
    """all_gather of a float64 array -> [world, ...]"""
    t = torch.from_numpy(np.ascontiguousarray(x, np.float64))
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return np.stack([o.numpy() for o in out])


def _worker(rank, world, port, V, cut, cases, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v0, v1 = (0, cut) if rank == 0 else (cut, V)
        res = []
        for k, seed in cases:
            cu, tok, tf, df, seeds = _batch(V, k, seed)
            B = len(k)
            T = tf[:, v0:v1].astype(np.float64)  # this rank's columns only
            D = df[:, v0:v1].astype(np.float64)
            nk = int(cu[-1])
            tgt = np.concatenate([[cu[i] + i + j for j in range(k[i])] for i in range(B)])
            # 1. per-shard statistics of every draft row (and the bonus rows' t)
            mt, md = T.max(1), D.max(1)
            st = np.exp(T - mt[:, None]).sum(1)
            sd = np.exp(D - md[:, None]).sum(1)
            at = (np.exp(T[tgt] - mt[tgt, None]) * (T[tgt] - D)).sum(1)
            own = (tok >= v0) & (tok < v1)
            xl = np.zeros((nk, 2))
            xl[own, 0] = T[tgt[own], tok[own] - v0]
            xl[own, 1] = D[own, tok[own] - v0]
            G = _gather(np.concatenate([mt, st]), world)
            Gd = _gather(np.stack([md, sd, at], 1), world)
            xlt = torch.from_numpy(xl)
            dist.all_reduce(xlt, op=dist.ReduceOp.SUM)  # exactly one owner per token
            xl = xlt.numpy()
            n_t = T.shape[0]
            MT = G[:, :n_t].max(0)
            lse_t = MT + np.log((G[:, n_t:] * np.exp(G[:, :n_t] - MT)).sum(0))
            MD = Gd[:, :, 0].max(0)
            lse_d = MD + np.log((Gd[:, :, 1] * np.exp(Gd[:, :, 0] - MD)).sum(0))
            e_mt = np.exp(G[:, :n_t][:, tgt] - lse_t[tgt])
            kl = (Gd[:, :, 2] * e_mt).sum(0) - lse_t[tgt] + lse_d  # E_p[t - d] - lse_t + lse_d
            # 2. accept test and first rejection (the same on every rank)
            lr = (xl[:, 0] - lse_t[tgt]) - (xl[:, 1] - lse_d)
            acc_len, emitted = np.zeros(B, np.int64), np.full(nk + B, -1, np.int64)
            draw = []
            for i in range(B):
                a = k[i]
                for j in range(k[i]):
                    ua, _ = oracle.uniforms(int(seeds[cu[i] + i + j]))
                    if not ua < min(1.0, np.exp(lr[cu[i] + j])):
                        a = j
                        break
                acc_len[i] = a
                emitted[cu[i] + i: cu[i] + i + a] = tok[cu[i]: cu[i] + a]
                _, us = oracle.uniforms(int(seeds[cu[i] + i + a]))
                draw.append((i, a, us))
            # 3. per-shard masses of each drawn row, all-gathered
            W = np.zeros((B, v1 - v0))
            for i, a, _ in draw:
                p = np.exp(T[cu[i] + i + a] - lse_t[cu[i] + i + a])
                if a < k[i]:
                    q = np.exp(D[cu[i] + a] - lse_d[cu[i] + a])
                    W[i] = np.maximum(p - q, 0.0)
                else:
                    W[i] = p
            Gm = _gather(W.sum(1), world)  # [world, B]
            # 4. crossing shard; its owner scans its columns; all-reduce (max)
            tok_out = np.full(B, -1, np.int64)
            for i, a, us in draw:
                R = Gm[:, i].sum()
                target = us * R
                c = np.cumsum(Gm[:, i])
                s = int(np.argmax(c > target)) if (c > target).any() else world - 1
                if s == rank:
                    base = c[s] - Gm[s, i]
                    cum = base + np.cumsum(W[i])
                    hit = np.nonzero((cum > target) & (W[i] > 0))[0]
                    tok_out[i] = v0 + (hit[0] if hit.size else int(np.nonzero(W[i] > 0)[0][-1]))
            tt = torch.from_numpy(tok_out)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            for i, a, _ in draw:
                emitted[cu[i] + i + a] = int(tt[i])
            res.append((acc_len.tolist(), emitted.tolist(), kl.tolist()))
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_vocab_parallel_exchange_world2_matches_single_process():
    V, cut = 5000, 2048
    cases = [(synth.random_k(12, 5, s), 100 + s) for s in range(6)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, V, cut, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (k, seed) in enumerate(cases):
        cu, tok, t, d, seeds = _batch(V, k, seed)
        o = oracle.verify(cu, tok, t, d, seeds, oracle.F32, resample=oracle.RESAMPLE_FULL)  # the vp exchange is D7
        for r in range(2):
            acc, em, kl = got[r][ci]
            assert np.array_equal(np.asarray(acc), o.accepted_len), (ci, r)
            assert np.array_equal(np.asarray(em), o.emitted), (ci, r)
            assert np.allclose(kl, o.kld, rtol=1e-12, atol=1e-14)
