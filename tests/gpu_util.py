"""Helpers for the -m gpu tests: run the CUDA path through the C-ABI binding."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import synth


def require_gpu():
    if not torch.cuda.is_available():
        raise RuntimeError("GPU test on a box without CUDA")


def dsde():
    import paper_2509_01083_b200 as m
    m.lib()  # loud failure if the extension is missing
    return m


def to_device_inputs(host: dict, dtype: torch.dtype, device="cuda", ld_pad: int = 0):
    """numpy host batch (oracle format) -> device tensors for dsde_verify."""
    t, d = host["target"], host["draft"]
    V = t.shape[1]
    esz = 2 if dtype == torch.bfloat16 else 4
    ld_pad += (-(V + ld_pad) * esz) % 16 // esz   # rows must start 16-byte aligned
    def dev(x):
        if dtype == torch.bfloat16:
            a = torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16)
        else:
            a = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        if ld_pad:
            full = torch.zeros((a.shape[0], V + ld_pad), dtype=a.dtype)
            full[:, :V] = a
            a = full
        return a.to(device)
    return dict(cu_sl=torch.from_numpy(np.asarray(host["cu_sl"], np.int32)).to(device),
                draft_tokens=torch.from_numpy(np.asarray(host["draft_tokens"], np.int32)).to(device),
                target=dev(t), draft=dev(d),
                seeds=torch.from_numpy(np.asarray(host["seeds"], np.uint64).view(np.int64)).to(device),
                V=V)


def gpu_verify(m, state, dev: dict, with_flags=True):
    cu = dev["cu_sl"]
    B = cu.numel() - 1
    n = dev["draft_tokens"].numel()
    V = dev["V"]
    ws = torch.empty(m.workspace_size(B, n, V, dev["target"].dtype) + 256, dtype=torch.uint8, device="cuda")
    ws = ws[(-ws.data_ptr()) % 256:]
    acc = torch.full((B,), -7, dtype=torch.int32, device="cuda")
    emitted = torch.full((n + B,), -7, dtype=torch.int32, device="cuda")
    kld = torch.full((n,), float("nan"), dtype=torch.float32, device="cuda")
    flags = torch.zeros(n + B, dtype=torch.uint8, device="cuda") if with_flags else None
    m.dsde_verify(state, V, n, cu, dev["draft_tokens"], dev["target"], dev["draft"], dev["seeds"],
                  acc, emitted, kld, flags, ws)
    torch.cuda.synchronize()
    return (acc.cpu().numpy(), emitted.cpu().numpy(), kld.cpu().numpy(),
            flags.cpu().numpy() if flags is not None else None)


def oracle_verify(host: dict, nthreads: int = 8, resample: int = oracle.RESAMPLE_FULL):
    dt = oracle.BF16 if host["target"].dtype == np.uint16 else oracle.F32
    return oracle.verify(host["cu_sl"], host["draft_tokens"], host["target"], host["draft"],
                         host["seeds"], dt, nthreads=nthreads, resample=resample)


def make_host_batch(V, k, seed, dtype=torch.bfloat16, profiles=("code",), step=0):
    w = synth.Workload(B=len(k), V=V, dtype=dtype, profiles=profiles, seed=seed)
    s = synth.generate_step(w, step, k, device="cpu")
    return s.host_arrays()
