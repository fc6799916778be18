"""Chooses the draft-noise sigma_n of each synthetic acceptance profile.

Per-position acceptance of speculative sampling with x ~ q is
alpha = E[sum_v min(p_v, q_v)]. For a profile (sigma_t range, target
alpha from Table I block efficiencies / P:427) this bisects sigma_n so that the
mean over sampled rows of synth's own generator (bf16-rounded logits,
V = 128256, a per-sequence draft offset) hits alpha. Generator parameter only:
no test expectation is derived from it. Prints the table for synth.PROFILES.
"""
import sys

import numpy as np
import scipy.special as sps
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth  # noqa: E402


def mean_alpha(name, sigma_n, rows=48, V=128256, seed=7):
    p0 = synth.PROFILES[name]
    prof = synth.Profile(name, p0.alpha, p0.sigma_t_lo, p0.sigma_t_hi, sigma_n)
    synth.PROFILES["_cal"] = prof
    w = synth.Workload(B=rows, V=V, dtype=torch.bfloat16, profiles=("_cal",), seed=seed, phases=False)
    s = synth.generate_step(w, 0, np.ones(rows, np.int64))
    t = s.target.float().numpy()
    d = s.draft.float().numpy()
    rows_t = np.arange(rows) * 2  # target row of (i, 0) is cu[i] + i = 2i
    P = sps.softmax(t[rows_t].astype(np.float64), axis=1)
    Q = sps.softmax(d.astype(np.float64), axis=1)
    return float(np.mean(np.minimum(P, Q).sum(axis=1)))


def solve(name, alpha):
    lo, hi = 0.01, 5.0
    for _ in range(14):
        mid = (lo * hi) ** 0.5
        if mean_alpha(name, mid) > alpha:
            lo = mid
        else:
            hi = mid
    return (lo * hi) ** 0.5


if __name__ == "__main__":
    for name in ("code", "dialogue", "low"):
        a = synth.PROFILES[name].alpha
        sn = solve(name, a)
        print(f"{name}: alpha={a} sigma_n={sn:.4f} check={mean_alpha(name, sn, rows=96, seed=11):.4f}")
