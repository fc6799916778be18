"""Brute-force harness for the distributional exactness of verify-then-resample.

Test helper (not product code). A tiny autoregressive "model pair" is a pair
of logit tables indexed by context (all token strings of length <= L over a
vocabulary of V <= 8). Generation of L tokens runs speculative steps through
a ``verify_fn`` (the oracle or the CUDA path) until every run has L tokens;
the empirical distribution of the L-token strings must equal exact target
autoregressive sampling, P(s) = prod_m p(s_m | s_<m).

The draft proposals x_j ~ q(. | context) are drawn here with numpy's own
generator from an exact softmax of the draft table (this is the stand-in
draft model, not the method under test).
"""
from __future__ import annotations

import numpy as np
import scipy.special as sps
import scipy.stats as st

import synth


class Tables:
    """temp: sampling temperature of both models (p = softmax(T / temp));
    mask_t / mask_d: probability that an entry of the target / draft table is
    masked (-inf, as a top-k / top-p filter leaves it); every row keeps at
    least one token of the target's support unmasked in both tables."""

    def __init__(self, V: int, L: int, seed: int, sigma_t=1.5, sigma_n=0.9, dtype=np.float32,
                 temp: float = 1.0, mask_t: float = 0.0, mask_d: float = 0.0):
        self.V, self.L = V, L
        self.temp = temp
        self.off = [0]
        for m in range(L + 1):
            self.off.append(self.off[-1] + V ** m)
        n = self.off[-1]
        r = np.random.default_rng(seed)
        self.T = (r.normal(0, sigma_t, (n, V))).astype(dtype)
        self.D = (self.T.astype(np.float64) + r.normal(0, sigma_n, (n, V))
                  + r.uniform(-3, 3, (n, 1))).astype(dtype)
        if mask_t > 0 or mask_d > 0:
            keep = r.integers(0, V, n)  # one token per row that neither table masks
            mt = r.random((n, V)) < mask_t
            md = r.random((n, V)) < mask_d
            mt[np.arange(n), keep] = False
            md[np.arange(n), keep] = False
            self.T[mt] = -np.inf
            self.D[md] = -np.inf
        self.P = sps.softmax(self.T.astype(np.float64) / temp, axis=1)
        self.Q = sps.softmax(self.D.astype(np.float64) / temp, axis=1)

    def index(self, ctx_code: np.ndarray, length: np.ndarray) -> np.ndarray:
        """Row index of contexts given as base-V codes of the given lengths."""
        return np.asarray(self.off, dtype=np.int64)[length] + ctx_code

    def exact(self) -> np.ndarray:
        """Exact probability of every length-L string (base-V code order)."""
        V, L = self.V, self.L
        prob = np.ones(1)
        for m in range(L):
            rows = self.P[self.off[m]: self.off[m] + V ** m]          # [V^m, V]
            prob = (prob[:, None] * rows).reshape(-1)
        return prob


def run_generation(tab: Tables, n_runs: int, verify_fn, seed: int, k_max: int = 3,
                   record_first=None):
    """Generate L tokens per run through speculative steps; returns the base-V
    codes of the first L tokens of each run. ``verify_fn(cu_sl, tokens,
    target, draft, seeds) -> (accepted_len, emitted)`` (numpy in/out)."""
    V, L = tab.V, tab.L
    rng = np.random.default_rng(seed + 1)
    code = np.zeros(n_runs, np.int64)     # base-V code of the current context
    length = np.zeros(n_runs, np.int64)
    step = 0
    while True:
        act = np.nonzero(length < L)[0]
        if act.size == 0:
            break
        B = act.size
        rem = L - length[act]
        # ragged k in [1, min(k_max, remaining)]
        k = 1 + (synth.splitmix64(np.uint64(step * 1000003) + act.astype(np.uint64))
                 % np.minimum(k_max, rem).astype(np.uint64)).astype(np.int64)
        cu = synth.cu_from_k(k)
        nk = int(cu[-1])
        c_code = code[act].copy()
        c_len = length[act].copy()
        tokens = np.zeros(nk, np.int32)
        trow = np.zeros(nk + B, np.int64)
        drow = np.zeros(nk, np.int64)
        cc, cl = c_code.copy(), c_len.copy()
        for j in range(int(k.max()) + 1):
            live = np.nonzero(j <= k)[0]
            idx = tab.index(cc[live], cl[live])
            trow[cu[live] + live + j] = idx
            live_d = np.nonzero(j < k)[0]
            if live_d.size == 0:
                break
            idx_d = tab.index(cc[live_d], cl[live_d])
            drow[cu[live_d] + j] = idx_d
            # x_j ~ q(. | context): inverse transform with numpy's generator
            q = tab.Q[idx_d]
            u = rng.random(live_d.size)
            x = (np.cumsum(q, axis=1) > u[:, None]).argmax(axis=1)
            tokens[cu[live_d] + j] = x
            cc[live_d] = cc[live_d] * V + x
            cl[live_d] += 1
        target = tab.T[trow]
        draft = tab.D[drow]
        seeds = synth.slot_seeds(seed, step, cu)
        acc, emitted = verify_fn(cu, tokens, target, draft, seeds)
        if record_first is not None and step == 0:
            record_first(cu, tokens, acc, emitted)
        acc = np.asarray(acc, dtype=np.int64)
        assert ((acc >= 0) & (acc <= k)).all()
        for m in range(int(k.max()) + 1):
            take = np.nonzero((m <= acc) & (length[act] < L))[0]
            tkn = np.asarray(emitted)[cu[take] + take + m].astype(np.int64)
            assert ((tkn >= 0) & (tkn < V)).all()
            r = act[take]
            code[r] = code[r] * V + tkn
            length[r] += 1
        step += 1
    return code


def check_distribution(tab: Tables, codes: np.ndarray, tv_max=0.01, p_min=1e-3):
    exact = tab.exact()
    n = codes.size
    counts = np.bincount(codes, minlength=exact.size).astype(np.float64)
    emp = counts / n
    tv = 0.5 * np.abs(emp - exact).sum()
    expc = exact * n
    m = expc >= 5
    chi2 = np.sum((counts[m] - expc[m]) ** 2 / expc[m])
    # lump the sparse cells into one
    if (~m).any():
        lo_e, lo_c = expc[~m].sum(), counts[~m].sum()
        if lo_e > 0:
            chi2 += (lo_c - lo_e) ** 2 / lo_e
            dof = int(m.sum())
        else:
            dof = int(m.sum()) - 1
    else:
        dof = int(m.sum()) - 1
    p = st.chi2.sf(chi2, dof)
    assert tv <= tv_max, f"TV {tv}"
    assert p > p_min, f"chi2 {chi2} dof {dof} p {p}"
    return tv, p
