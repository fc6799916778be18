"""CPU oracle for the DSDE verification hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path
(``paper_2509_01083_b200``) never imports it and shares no code with it.

This module is a thin ctypes/numpy wrapper over ``oracle/dsde_oracle.c`` (plain
C, fp64, sequential loops; see that file's header for the paper citations).
Functions whose pins live in ``tests/test_oracle_*.py``:

* ``philox4x32_10`` / ``uniforms``  — Random123 KAT vectors (D6).
* ``row_kld`` / ``row_log_ratio``   — KL(p||p)=0, Gibbs, two-point closed form,
  uniform-p closed form, scipy ``rel_entr``, shift invariance.
* ``verify``                        — brute-force distribution test (S:144,
  S:584), one-hot special cases, worked V=2 example, prefix shape.
* ``weighted_variance`` etc.        — S:217-219 examples, delta=1 population
  variance (numpy), translation invariance, Welford/West agreement (Eq.5-7).
* ``next_sl``                       — exhaustive MSE grid search (Eq.9-11).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dsde_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

F32, BF16 = 0, 1

FLAG_ACCEPT_TIE = 1
FLAG_SAMPLE_TIE = 2
FLAG_FALLBACK = 4
FLAG_PROPOSAL_FALLBACK = 8   # D23: no proposal kept, the D7 draw was used

# the recovery draw's reading (D23 proposals from p, or D7 inverse CDF over max(0, p - q))
RESAMPLE_PROPOSAL, RESAMPLE_FULL = 0, 1
PROPOSALS = 256


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no GPU code involved)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fvisibility=hidden",
               "-fno-fast-math", "-ffp-contract=off", "-o", _LIB_PATH, _SRC, "-lm", "-lpthread"]
        subprocess.check_call(cmd)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        L.oracle_philox4x32_10.argtypes = [P, P, P]
        L.oracle_res53.argtypes = [C.c_uint32, C.c_uint32]
        L.oracle_res53.restype = C.c_double
        L.oracle_uniforms.argtypes = [C.c_uint64, P, P]
        L.oracle_row_kld.argtypes = [C.c_int, P, P]
        L.oracle_row_kld.restype = C.c_double
        L.oracle_row_log_ratio.argtypes = [C.c_int, P, P, C.c_int]
        L.oracle_row_entropy.argtypes = [C.c_int, P]
        L.oracle_row_entropy.restype = C.c_double
        L.oracle_draft_entropy.argtypes = [C.c_int, C.c_int, C.c_int, P, C.c_int64, P]
        L.oracle_draft_entropy.restype = None
        L.oracle_row_log_ratio.restype = C.c_double
        L.oracle_verify.argtypes = [C.c_int, C.c_int, C.c_int, P, P, P, C.c_int64, P, C.c_int64,
                                    P, P, P, P, P, P, P, P, P, C.c_int]
        L.oracle_verify.restype = C.c_int
        L.oracle_verify_mode.argtypes = list(L.oracle_verify.argtypes) + [C.c_int]
        L.oracle_verify_mode.restype = C.c_int
        L.oracle_verify_temp.argtypes = list(L.oracle_verify.argtypes) + [C.c_int, C.c_void_p, C.c_int]
        L.oracle_proposal_uniforms.argtypes = [C.c_uint64, C.c_uint32, P, P]
        L.oracle_verify_temp.restype = C.c_int
        L.oracle_weighted_variance.argtypes = [P, C.c_int, C.c_double]
        L.oracle_weighted_variance.restype = C.c_double
        L.oracle_scale_factor.argtypes = [C.c_double]
        L.oracle_scale_factor.restype = C.c_double
        L.oracle_calibrate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                       C.c_double, P]
        L.oracle_calibrate.restype = C.c_int
        L.oracle_predict_sl.argtypes = [C.c_double, C.c_int, C.c_int, P]
        L.oracle_predict_sl.restype = C.c_int
        L.oracle_state_new.argtypes = [P, C.c_int]
        L.oracle_state_new.restype = C.c_void_p
        L.oracle_state_free.argtypes = [P]
        L.oracle_state_reset.argtypes = [P, P, C.c_int]
        L.oracle_update_signal.argtypes = [P, C.c_int, P, P, P, P, P, P, P]
        L.oracle_update_signal.restype = C.c_int
        L.oracle_update_signal_ent.argtypes = [P, C.c_int, P, P, P, P, P, P, P, P]
        L.oracle_update_signal_ent.restype = C.c_int
        L.oracle_entropy_sl.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, P]
        L.oracle_entropy_sl.restype = C.c_int
        L.oracle_next_sl.argtypes = [P, C.c_int, P, P, P, P, P]
        L.oracle_next_sl.restype = C.c_int
        L.oracle_cap_partial.argtypes = [C.c_int, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- C0 ---

def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def res53(a: int, b: int) -> float:
    return lib().oracle_res53(a, b)


def proposal_uniforms(seed: int, j: int) -> tuple[float, float]:
    """D23: (u_prop, u_keep) of proposal j >= 1 (Philox counter (j, 0, 0, 0))."""
    up, uk = C.c_double(), C.c_double()
    lib().oracle_proposal_uniforms(C.c_uint64(seed), C.c_uint32(j), C.byref(up), C.byref(uk))
    return up.value, uk.value


def uniforms(seed: int) -> tuple[float, float]:
    ua, us = C.c_double(), C.c_double()
    lib().oracle_uniforms(C.c_uint64(seed), C.byref(ua), C.byref(us))
    return ua.value, us.value


# ----------------------------------------------------------------- C1 ---

def row_kld(t, d) -> float:
    t = np.ascontiguousarray(t, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    assert t.shape == d.shape and t.ndim == 1
    return lib().oracle_row_kld(t.size, _p(t), _p(d))


def row_entropy(d) -> float:
    """H(softmax(d)) = -sum q log q."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    assert d.ndim == 1
    return lib().oracle_row_entropy(d.size, _p(d))


def draft_entropy(draft_logits, dtype: int) -> np.ndarray:
    """H(q) of every row of a [n, V] draft-logit array (fp32, or bf16 bit patterns as uint16)."""
    d = np.ascontiguousarray(draft_logits)
    out = np.empty(d.shape[0], dtype=np.float64)
    lib().oracle_draft_entropy(d.shape[0], d.shape[1], int(dtype), _p(d), d.shape[1], _p(out))
    return out


def row_log_ratio(t, d, x: int) -> float:
    t = np.ascontiguousarray(t, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    return lib().oracle_row_log_ratio(t.size, _p(t), _p(d), int(x))


@dataclass
class VerifyResult:
    accepted_len: np.ndarray   # [B] int32
    emitted: np.ndarray        # [sum k + B] int32, pad = -1
    kld: np.ndarray            # [sum k] float64
    log_ratio: np.ndarray      # [sum k] float64, log p(x) - log q(x)
    u_acc: np.ndarray          # [sum k + B]
    u_smp: np.ndarray          # [sum k + B]
    samp_diag: np.ndarray      # [B, 3]: R, lo, hi
    flags: np.ndarray          # [sum k + B]


def verify(cu_sl, draft_tokens, target_logits, draft_logits, seeds, dtype: int,
           nthreads: int = 1, greedy: bool = False, temperature=None,
           resample: int = 1) -> VerifyResult:
    """Batched verification. ``target_logits`` / ``draft_logits`` are 2-D numpy
    arrays of float32 (dtype=F32) or uint16 bf16 bit patterns (dtype=BF16);
    -inf entries are masked tokens (D21).
    greedy=True: T = 0 verification (accept iff x_j = argmax t_j, emit the
    target argmax).
    temperature: optional per-sequence temperatures [B] (D20): p = softmax(t/T),
    q = softmax(d/T); T = 0 makes that sequence greedy.
    resample: the recovery draw's reading — RESAMPLE_FULL (D7, default: the
    inverse CDF over max(0, p - q) with u_smp) or RESAMPLE_PROPOSAL (D23: up
    to PROPOSALS proposals v ~ p, each kept with probability
    max(0, p_v - q_v) / p_v, then the D7 draw)."""
    cu_sl = np.ascontiguousarray(cu_sl, dtype=np.int32)
    toks = np.ascontiguousarray(draft_tokens, dtype=np.int32)
    tl = np.ascontiguousarray(target_logits)
    dl = np.ascontiguousarray(draft_logits)
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    B = cu_sl.size - 1
    nk = int(cu_sl[-1])
    V = tl.shape[1]
    want = np.float32 if dtype == F32 else np.uint16
    assert tl.dtype == want and dl.dtype == want, (tl.dtype, want)
    assert tl.shape[0] >= nk + B and dl.shape[0] >= nk and seeds.size >= nk + B
    r = VerifyResult(
        accepted_len=np.zeros(B, np.int32), emitted=np.zeros(nk + B, np.int32),
        kld=np.zeros(nk, np.float64), log_ratio=np.zeros(nk, np.float64),
        u_acc=np.zeros(nk + B, np.float64), u_smp=np.zeros(nk + B, np.float64),
        samp_diag=np.zeros((B, 3), np.float64), flags=np.zeros(nk + B, np.int32))
    temps = None if temperature is None else np.ascontiguousarray(temperature, dtype=np.float64)
    assert temps is None or temps.size == B
    rc = lib().oracle_verify_temp(B, V, dtype, _p(cu_sl), _p(toks), _p(tl), tl.shape[1], _p(dl),
                                  dl.shape[1], _p(seeds), _p(r.accepted_len), _p(r.emitted), _p(r.kld),
                                  _p(r.log_ratio), _p(r.u_acc), _p(r.u_smp), _p(r.samp_diag),
                                  _p(r.flags), int(nthreads), int(bool(greedy)),
                                  None if temps is None else _p(temps), int(resample))
    if rc != 0:
        raise ValueError(f"oracle_verify failed: {rc}")
    return r


# ----------------------------------------------------------------- C2 ---

class _Cfg(C.Structure):
    _fields_ = [("delta", C.c_double), ("n_short", C.c_int), ("n_long", C.c_int),
                ("sl_min", C.c_int), ("sl_ceiling", C.c_int), ("epsilon", C.c_double),
                ("calib_steps", C.c_int), ("calib_sl", C.c_int), ("window_unit", C.c_int),
                ("cap_mode", C.c_int), ("entropy_mode", C.c_int), ("entropy_gamma", C.c_double)]


@dataclass
class Config:
    delta: float = 0.85
    n_short: int = 10
    n_long: int = 30
    sl_min: int = 2
    sl_ceiling: int = 8
    epsilon: float = 1e-6
    calib_steps: int = 5
    calib_sl: int = 4
    window_unit: int = 0
    cap_mode: int = 1
    entropy_mode: int = 0      # 1: min(SL^, SL_H) with the draft-entropy predictor (D22)
    entropy_gamma: float = 0.5

    def c(self) -> _Cfg:
        return _Cfg(self.delta, self.n_short, self.n_long, self.sl_min, self.sl_ceiling,
                    self.epsilon, self.calib_steps, self.calib_sl, self.window_unit,
                    self.cap_mode, self.entropy_mode, self.entropy_gamma)


def weighted_variance(values_recent_first, delta: float) -> float:
    v = np.ascontiguousarray(values_recent_first, dtype=np.float64)
    return lib().oracle_weighted_variance(_p(v), v.size, float(delta))


def scale_factor(mu_last: float) -> float:
    return lib().oracle_scale_factor(float(mu_last))


def calibrate(sl_a_max: int, mu_pre: float, kld_pre_max: float, sl_min: int = 2,
              sl_ceiling: int = 1 << 20, epsilon: float = 1e-6) -> tuple[int, float]:
    raw = C.c_double()
    r = lib().oracle_calibrate(int(sl_a_max), float(mu_pre), float(kld_pre_max), int(sl_min),
                               int(sl_ceiling), float(epsilon), C.byref(raw))
    return r, raw.value


def entropy_sl(h_mean: float, gamma: float, sl_max: int, sl_min: int = 2) -> tuple[int, float]:
    """D22: SL_H = clamp(rint(max(0, 1 - sqrt(gamma H)) (SL_max - SL_min) + SL_min))."""
    x = C.c_double()
    r = lib().oracle_entropy_sl(float(h_mean), float(gamma), int(sl_max), int(sl_min), C.byref(x))
    return r, x.value


def predict_sl(penalty: float, sl_max: int, sl_min: int = 2) -> tuple[int, float]:
    x = C.c_double()
    r = lib().oracle_predict_sl(float(penalty), int(sl_max), int(sl_min), C.byref(x))
    return r, x.value


class OracleState:
    """Per-sequence adapter state (history ring, calibration, SL_max)."""

    def __init__(self, cfg: Config, n: int):
        self.cfg = cfg
        self._cfg_c = cfg.c()
        self.n = n
        self._h = lib().oracle_state_new(C.byref(self._cfg_c), int(n))
        if not self._h:
            raise ValueError("invalid oracle config")

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.oracle_state_free(self._h)
            self._h = None

    def reset(self, slots):
        s = np.ascontiguousarray(slots, dtype=np.int32)
        lib().oracle_state_reset(self._h, _p(s), s.size)

    def update_signal(self, slots, cu_sl, kld, accepted_len, entropy=None):
        """entropy: optional draft entropy per draft position (cfg.entropy_mode, D22)."""
        slots = np.ascontiguousarray(slots, dtype=np.int32)
        cu_sl = np.ascontiguousarray(cu_sl, dtype=np.int32)
        kld = np.ascontiguousarray(kld, dtype=np.float64)
        acc = np.ascontiguousarray(accepted_len, dtype=np.int32)
        B = slots.size
        sl_hat = np.zeros(B, np.int32)
        calib = np.zeros(B, np.int32)
        diag = np.zeros((B, 8), np.float64)
        ent = None if entropy is None else np.ascontiguousarray(entropy, dtype=np.float64)
        rc = lib().oracle_update_signal_ent(self._h, B, _p(slots), _p(cu_sl), _p(kld), _p(acc),
                                            None if ent is None else _p(ent), _p(sl_hat), _p(calib), _p(diag))
        if rc != 0:
            raise ValueError("oracle_update_signal failed")
        return sl_hat, calib, diag

    def next_sl(self, sl_hat, calibrating, budget=None):
        return next_sl(self.cfg, sl_hat, calibrating, budget)


def next_sl(cfg: Config, sl_hat, calibrating, budget=None):
    sl_hat = np.ascontiguousarray(sl_hat, dtype=np.int32)
    calib = np.ascontiguousarray(calibrating, dtype=np.int32)
    B = sl_hat.size
    out = np.zeros(B, np.int32)
    cap = C.c_int32()
    cc = cfg.c()
    if budget is not None:
        budget = np.ascontiguousarray(budget, dtype=np.int32)
    lib().oracle_next_sl(C.byref(cc), B, _p(sl_hat), _p(calib),
                         _p(budget) if budget is not None else None, _p(out), C.byref(cap))
    return out, cap.value


def cap_partial(sl_hat, calibrating) -> tuple[int, int]:
    sl_hat = np.ascontiguousarray(sl_hat, dtype=np.int32)
    calib = np.ascontiguousarray(calibrating, dtype=np.int32)
    s, n = C.c_longlong(), C.c_longlong()
    lib().oracle_cap_partial(sl_hat.size, _p(sl_hat), _p(calib), C.byref(s), C.byref(n))
    return s.value, n.value
