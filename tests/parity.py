"""GPU-vs-oracle comparison rules (test infrastructure).

Bands (from BASELINE.json north_star and SURVEY §8(c) D16):
* KLD:           |KL_gpu - KL_o| <= 1e-5 |KL_o| + 1e-9            (fp64 oracle)
* accept ties:   a_gpu != a_o only if |u_acc - min(1, r_o)| < 1e-6 at j = min(a_gpu, a_o)
* sample ties:   token_gpu != token_o only if |u_smp - C/R| < 1e-6 at an edge of
                 the oracle's token (C_{v-1}/R or C_v/R), or (D23 recovery draws)
                 a proposal's |u_prop - C/P| or |u_keep - max(0, p - q)/p| < 1e-6
* everything else (accepted lengths, emitted tokens, pads) bit-exact.
Ties are counted and returned, never silently ignored.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

KL_REL, KL_ABS, TIE = 1e-5, 1e-9, 1e-6


@dataclass
class Report:
    seqs: int = 0
    positions: int = 0
    accept_ties: int = 0
    sample_ties: int = 0
    mismatches: list = field(default_factory=list)
    kl_max_rel: float = 0.0
    kl_bad: int = 0

    def ok(self) -> bool:
        return not self.mismatches and self.kl_bad == 0

    def merge(self, o: "Report"):
        self.seqs += o.seqs
        self.positions += o.positions
        self.accept_ties += o.accept_ties
        self.sample_ties += o.sample_ties
        self.mismatches += o.mismatches
        self.kl_max_rel = max(self.kl_max_rel, o.kl_max_rel)
        self.kl_bad += o.kl_bad

    def __str__(self):
        return (f"seqs={self.seqs} positions={self.positions} accept_ties={self.accept_ties} "
                f"sample_ties={self.sample_ties} kl_max_rel={self.kl_max_rel:.3e} kl_bad={self.kl_bad} "
                f"mismatches={self.mismatches[:5]}")


def compare_verify(cu, acc_g, emit_g, kld_g, o, seq_ids=None) -> Report:
    """cu: int32 [B+1]; acc_g/emit_g/kld_g: GPU numpy outputs; o: oracle.VerifyResult."""
    cu = np.asarray(cu, dtype=np.int64)
    B = cu.size - 1
    rep = Report(seqs=B, positions=int(cu[-1]))
    # KLD at every position
    kg = np.asarray(kld_g, dtype=np.float64)
    ko = o.kld
    with np.errstate(invalid="ignore"):
        err = np.where(kg == ko, 0.0, np.abs(kg - ko))  # (+inf on both sides: masked support, D21)
    band = KL_REL * np.abs(ko) + KL_ABS
    rep.kl_bad = int(np.sum(~(err <= band)))
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(ko > 0, err / np.abs(ko), 0.0)
    rep.kl_max_rel = float(np.nanmax(rel)) if rel.size else 0.0
    for i in range(B):
        sid = i if seq_ids is None else int(seq_ids[i])
        k = int(cu[i + 1] - cu[i])
        s0 = int(cu[i]) + i
        ag, ao = int(acc_g[i]), int(o.accepted_len[i])
        if ag != ao:
            j = min(ag, ao)
            r = np.exp(o.log_ratio[cu[i] + j]) if j < k else 1.0
            if j < k and abs(o.u_acc[s0 + j] - min(1.0, r)) < TIE:
                rep.accept_ties += 1
                continue
            rep.mismatches.append(("accepted_len", sid, ag, ao))
            continue
        eg = np.asarray(emit_g[s0:s0 + k + 1])
        eo = o.emitted[s0:s0 + k + 1]
        if not np.array_equal(eg[:ag], eo[:ao]):
            rep.mismatches.append(("prefix", sid))
            continue
        if not np.all(eg[ag + 1:] == -1):
            rep.mismatches.append(("pad", sid))
            continue
        if eg[ag] != eo[ao]:
            R, lo, hi = o.samp_diag[i]
            u = o.u_smp[s0 + ao]
            # the oracle flags a sample tie for any uniform it drew within 1e-6 of
            # a decision edge: the D7 draw's u_smp at a CDF edge, or (D23) a
            # proposal's u_prop at a CDF edge of p / its u_keep at the keep
            # probability
            if (o.flags[s0 + ao] & 2) or abs(u - lo) < TIE or abs(u - hi) < TIE:
                rep.sample_ties += 1
                continue
            rep.mismatches.append(("token", sid, int(eg[ag]), int(eo[ao]), float(u), float(lo), float(hi)))
    return rep


def subset_batch(host: dict, seq_ids) -> dict:
    """Repack the inputs of a subset of sequences into a self-contained batch
    (sequences are independent in verify, so the oracle can check samples)."""
    cu = np.asarray(host["cu_sl"], dtype=np.int64)
    t_rows, d_rows, toks, seeds, k = [], [], [], [], []
    for i in seq_ids:
        ki = int(cu[i + 1] - cu[i])
        k.append(ki)
        t_rows.append(host["target"][cu[i] + i: cu[i] + i + ki + 1])
        d_rows.append(host["draft"][cu[i]: cu[i] + ki])
        toks.append(host["draft_tokens"][cu[i]: cu[i] + ki])
        seeds.append(host["seeds"][cu[i] + i: cu[i] + i + ki + 1])
    cu2 = np.concatenate([[0], np.cumsum(k)]).astype(np.int32)
    return dict(cu_sl=cu2, target=np.concatenate(t_rows), draft=np.concatenate(d_rows),
                draft_tokens=np.concatenate(toks), seeds=np.concatenate(seeds))


def gather_subset_outputs(cu, seq_ids, acc, emitted, kld):
    cu = np.asarray(cu, dtype=np.int64)
    a, e, kl = [], [], []
    for i in seq_ids:
        ki = int(cu[i + 1] - cu[i])
        a.append(acc[i])
        e.append(emitted[cu[i] + i: cu[i] + i + ki + 1])
        kl.append(kld[cu[i]: cu[i] + ki])
    return np.asarray(a), np.concatenate(e), np.concatenate(kl)
