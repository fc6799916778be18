"""Python binding of libdsde.so — the B200-native DSDE verification hot path.

Argument marshalling only: every step of the path (verify, signal, SL
prediction, cap) runs in the sm_100a kernels behind the C-ABI declared in
``include/dsde.h``. PyTorch supplies device memory and streams. There is no
CPU fallback: if ``libdsde.so`` is missing, importing the library raises.

Names follow the C-ABI: ``dsde_verify``, ``dsde_update_signal``,
``dsde_next_sl`` (plus the state / comm helpers). ``Step`` bundles the three
calls of one decoding step with its buffers (DSDE step).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, fields

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdsde.so")

DSDE_OK, DSDE_ERR_ARG, DSDE_ERR_CUDA, DSDE_ERR_NCCL, DSDE_ERR_STATE, DSDE_ERR_DEVICE = 0, -1, -2, -3, -4, -5
DSDE_F32, DSDE_BF16 = 0, 1
DSDE_PAD = -1
DSDE_MAX_SL = 16
DSDE_MAX_WINDOW = 64
FLAG_ACCEPT_NEAR_TIE, FLAG_SAMPLE_NEAR_TIE, FLAG_FALLBACK, FLAG_PROPOSAL_FALLBACK = 1, 2, 4, 8
RESAMPLE_PROPOSAL, RESAMPLE_FULL = 0, 1  # dsde_config.resample (D23 / D7)
DERR = {0: "none", 1: "bad_sl", 2: "bad_token", 3: "nonfinite", 4: "rows", 5: "bad_slot", 6: "vp_fallback"}

# Every function the header declares (checked against include/dsde.h by the tests).
EXPORTS = (
    "dsde_config_default", "dsde_status_string", "dsde_abi_version", "dsde_set_draft_entropy", "dsde_set_temperature",
    "dsde_state_create",
    "dsde_state_reset", "dsde_state_destroy", "dsde_state_bytes", "dsde_state_export",
    "dsde_state_import", "dsde_get_device_error", "dsde_clear_device_error",
    "dsde_verify_workspace_size", "dsde_verify", "dsde_update_signal", "dsde_next_sl", "dsde_step",
    "dsde_cap_value", "dsde_comm_unique_id", "dsde_comm_init", "dsde_comm_destroy",
    "dsde_profile_enable", "dsde_profile_read",
    "dsde_vp_sizes", "dsde_vp_stream", "dsde_vp_finalize", "dsde_vp_draw", "dsde_vp_select", "dsde_vp_place",
    "dsde_vp_workspace_size", "dsde_vp_verify",
)
# dsde_profile_read phases (include/dsde.h): the row stream k_stream_ldg (a1),
# then the tail k_tail (a2-a4, + a5-a7 in dsde_step); two spare slots
VERIFY_PHASES = ("stream", "tail", "", "")


class DsdeError(RuntimeError):
    pass


class Config(C.Structure):
    """dsde_config (include/dsde.h); defaults from dsde_config_default()."""
    _fields_ = [("delta", C.c_double), ("n_short", C.c_int), ("n_long", C.c_int),
                ("sl_min", C.c_int), ("sl_ceiling", C.c_int), ("epsilon", C.c_double),
                ("calib_steps", C.c_int), ("calib_sl", C.c_int), ("window_unit", C.c_int),
                ("cap_mode", C.c_int), ("greedy", C.c_int), ("device_rows", C.c_int),
                ("masked", C.c_int), ("entropy_mode", C.c_int), ("entropy_gamma", C.c_double),
                ("resample", C.c_int)]

    @classmethod
    def default(cls, **kw) -> "Config":
        c = cls()
        lib().dsde_config_default(C.byref(c))
        for k, v in kw.items():
            setattr(c, k, v)
        return c

    def as_dict(self) -> dict:
        return {f[0]: getattr(self, f[0]) for f in self._fields_}


_lib = None


def lib() -> C.CDLL:
    """Loads libdsde.so (built in-tree by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libdsde.so not built: {LIB_PATH} is missing "
                              "(run python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        P, I, I64, S = C.c_void_p, C.c_int, C.c_int64, C.c_size_t
        L.dsde_config_default.argtypes = [P]
        L.dsde_config_default.restype = None
        L.dsde_status_string.argtypes = [I]
        L.dsde_status_string.restype = C.c_char_p
        L.dsde_abi_version.restype = I
        L.dsde_set_draft_entropy.argtypes = [P, P]
        L.dsde_set_temperature.argtypes = [P, P]
        L.dsde_state_create.argtypes = [P, I, P]
        L.dsde_state_reset.argtypes = [P, P, I, P]
        L.dsde_state_destroy.argtypes = [P]
        L.dsde_state_bytes.argtypes = [P]
        L.dsde_state_bytes.restype = S
        L.dsde_state_export.argtypes = [P, P, S, P]
        L.dsde_state_import.argtypes = [P, P, S, P]
        L.dsde_get_device_error.argtypes = [P, P, P]
        L.dsde_clear_device_error.argtypes = [P, P]
        L.dsde_verify_workspace_size.argtypes = [I, I, I, I]
        L.dsde_verify_workspace_size.restype = S
        L.dsde_verify.argtypes = [I, I, I, I, P, P, P, I64, P, I64, P, P, P, P, P, P, S, P, P]
        L.dsde_vp_sizes.argtypes = [I, I, I, P, P, P]
        L.dsde_vp_stream.argtypes = [P, I, I, I, I, I, I, P, P, P, I64, P, I64, P, P, P]
        L.dsde_vp_finalize.argtypes = [P, I, I, I, I, I, P, P, P, P, P, P, P, P, P, P, P]
        L.dsde_vp_draw.argtypes = [P, I, I, I, I, I, P, P, I64, P, I64, P, P]
        L.dsde_vp_select.argtypes = [P, I, I, I, I, I, P, P, P, I64, P, I64, P, P]
        L.dsde_vp_place.argtypes = [P, I, P, P, P, P, P]
        L.dsde_vp_workspace_size.argtypes = [I, I, I, I, I]
        L.dsde_vp_workspace_size.restype = S
        L.dsde_vp_verify.argtypes = [P, I, I, I, I, P, P, P, I64, P, I64, P, P, P, P, P, P, S, P, P]
        L.dsde_update_signal.argtypes = [P, I, P, P, P, P, P, P, P]
        L.dsde_step.argtypes = [P, I, I, I, I, P, P, P, P, I64, P, I64, P, P, P, P, P, P, P, P, P, P,
                                P, S, P, P]
        L.dsde_next_sl.argtypes = [P, I, P, P, P, P, P, P, P]
        L.dsde_cap_value.argtypes = [P, I64, I64, I64]
        L.dsde_cap_value.restype = C.c_int32
        L.dsde_comm_unique_id.argtypes = [P]
        L.dsde_comm_init.argtypes = [P, I, I, P]
        L.dsde_comm_destroy.argtypes = [P]
        L.dsde_profile_enable.argtypes = [P, I]
        L.dsde_profile_read.argtypes = [P, P, P]
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != DSDE_OK:
        raise DsdeError(f"{what}: {lib().dsde_status_string(rc).decode()} ({rc})")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return DSDE_BF16
    if dt == torch.float32:
        return DSDE_F32
    raise DsdeError(f"unsupported logits dtype {dt}")


def cap_value(cfg: Config, sum_sl_hat: int, n_active: int, max_sl_hat: int) -> int:
    """The cap rule of dsde_next_sl on host integers (dsde_cap_value)."""
    return int(lib().dsde_cap_value(C.byref(cfg), int(sum_sl_hat), int(n_active), int(max_sl_hat)))


class State:
    """Owns a dsde_state (per-sequence KLD ring, calibration, SL_max)."""

    def __init__(self, cfg: Config | None = None, max_seqs: int = 1):
        self.cfg = cfg if cfg is not None else Config.default()
        h = C.c_void_p()
        _check(lib().dsde_state_create(C.byref(self.cfg), int(max_seqs), C.byref(h)), "dsde_state_create")
        self.h = h
        self.max_seqs = max_seqs

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().dsde_state_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self, slots: torch.Tensor, stream=None):
        _check(lib().dsde_state_reset(self.h, _ptr(slots), slots.numel(), _stream(stream)), "dsde_state_reset")

    def nbytes(self) -> int:
        return int(lib().dsde_state_bytes(self.h))

    def export(self, buf: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if buf is None:
            buf = torch.empty(self.nbytes(), dtype=torch.uint8, device="cuda")
        _check(lib().dsde_state_export(self.h, _ptr(buf), buf.numel() * buf.element_size(), _stream(stream)),
               "dsde_state_export")
        return buf

    def load(self, buf: torch.Tensor, stream=None):
        _check(lib().dsde_state_import(self.h, _ptr(buf), buf.numel() * buf.element_size(), _stream(stream)),
               "dsde_state_import")

    def device_error(self) -> tuple[int, int]:
        code, seq = C.c_int32(), C.c_int32()
        _check(lib().dsde_get_device_error(self.h, C.byref(code), C.byref(seq)), "dsde_get_device_error")
        return code.value, seq.value

    def clear_error(self, stream=None):
        _check(lib().dsde_clear_device_error(self.h, _stream(stream)), "dsde_clear_device_error")

    def set_draft_entropy(self, out=None):
        """dsde_set_draft_entropy: later verify / step calls also write H(q) of every
        draft row to ``out`` (float32 device tensor, >= sum k rows); None turns it off."""
        self._entropy_ref = out  # keep the buffer alive while the library holds its pointer
        _check(lib().dsde_set_draft_entropy(self.h, None if out is None else _ptr(out)), "dsde_set_draft_entropy")

    def set_temperature(self, temperature=None):
        """dsde_set_temperature (D20): per-sequence temperatures (float32 device
        tensor [B], batch order) for later verify / step calls; T = 0 makes that
        sequence greedy; None = T = 1 for every sequence."""
        self._temp_ref = temperature  # keep the buffer alive while the library holds its pointer
        _check(lib().dsde_set_temperature(self.h, None if temperature is None else _ptr(temperature)),
               "dsde_set_temperature")

    def profile(self, enable: bool = True):
        """Turns on/off per-kernel CUDA-event timing of dsde_verify calls on this state."""
        _check(lib().dsde_profile_enable(self.h, int(enable)), "dsde_profile_enable")

    def profile_read(self) -> tuple[dict, int]:
        """Summed ms per verify phase since the last read, and the call count."""
        ms = (C.c_float * len(VERIFY_PHASES))()
        calls = C.c_int()
        _check(lib().dsde_profile_read(self.h, ms, C.byref(calls)), "dsde_profile_read")
        out = {n: float(x) for n, x in zip(VERIFY_PHASES, ms) if n}
        return out, calls.value


class Comm:
    """An NCCL communicator for the batch-wide cap (one per rank)."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().dsde_comm_init(buf, int(nranks), int(rank), C.byref(h)), "dsde_comm_init")
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().dsde_comm_unique_id(buf), "dsde_comm_unique_id")
        return bytes(buf)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().dsde_comm_destroy(self.h)
            self.h = None


def workspace_size(B: int, total_draft_rows: int, V: int, dtype: torch.dtype) -> int:
    return int(lib().dsde_verify_workspace_size(B, total_draft_rows, V, dtype_code(dtype)))


def dsde_verify(state: State, V: int, total_draft_rows: int, cu_sl, draft_tokens, target_logits,
                draft_logits, seeds, accepted_len, emitted_tokens, kld, flags, workspace, stream=None):
    """dsde_verify (include/dsde.h): all tensors on the current CUDA device."""
    B = cu_sl.numel() - 1
    _check(lib().dsde_verify(
        B, int(V), dtype_code(target_logits.dtype), int(total_draft_rows), _ptr(cu_sl),
        _ptr(draft_tokens), _ptr(target_logits), target_logits.stride(0), _ptr(draft_logits),
        draft_logits.stride(0), _ptr(seeds), _ptr(accepted_len), _ptr(emitted_tokens), _ptr(kld),
        _ptr(flags), _ptr(workspace), workspace.numel(), state.h, _stream(stream)), "dsde_verify")


class VocabParallel:
    """Vocabulary-parallel verification (include/dsde.h
    dsde_vp_*): the target / draft logits of a batch split by columns over
    ``nshards`` shards. ``shard_slices(V)`` gives the column ranges. ``run_local``
    runs every stage of every shard in this process (the exchanges are plain
    device copies / reductions) — the single-GPU check that the sharded path
    reproduces dsde_verify; ``verify`` runs this rank's shard over a Comm (NCCL,
    dsde_vp_verify). Argument marshalling and buffer bookkeeping only."""

    def __init__(self, state: State, V: int, nshards: int, dtype: torch.dtype):
        self.state, self.V, self.n, self.dtype = state, int(V), int(nshards), dtype
        w, ns, nd = C.c_int(), C.c_int(), C.c_int()
        _check(lib().dsde_vp_sizes(self.V, self.n, dtype_code(dtype), C.byref(w), C.byref(ns), C.byref(nd)),
               "dsde_vp_sizes")
        self.W, self.ns_sh, self.nd_sh = w.value, ns.value, nd.value

    def shard_slices(self):
        return [(s * self.W, min(self.V, (s + 1) * self.W)) for s in range(self.n)]

    def run_local(self, cu_sl, draft_tokens, target_shards, draft_shards, seeds, accepted_len, emitted, kld,
                  flags=None, stream=None):
        """target_shards / draft_shards: per-shard [rows, >= Vs] tensors."""
        B, n = cu_sl.numel() - 1, self.n
        total = draft_tokens.numel()
        dev = cu_sl.device
        dt = dtype_code(self.dtype)
        L, st = lib(), self.state.h
        part = torch.empty((n, total * self.ns_sh * 32), dtype=torch.uint8, device=dev)
        xl = torch.zeros((n, total, 2), dtype=torch.float32, device=dev)
        for s in range(n):
            t, d = target_shards[s], draft_shards[s]
            _check(L.dsde_vp_stream(st, B, self.V, n, s, dt, total, _ptr(cu_sl), _ptr(draft_tokens), _ptr(t),
                                    t.stride(0), _ptr(d), d.stride(0), _ptr(part[s]), _ptr(xl[s]), _stream(stream)),
                   "dsde_vp_stream")
        xlog = xl.sum(0).contiguous()  # the all-reduce (sum): exactly one shard owns each x
        rec = torch.empty(B * 64, dtype=torch.uint8, device=dev)
        _check(L.dsde_vp_finalize(st, B, self.V, n, dt, total, _ptr(cu_sl), _ptr(draft_tokens), _ptr(part),
                                  _ptr(xlog), _ptr(seeds), _ptr(accepted_len), _ptr(emitted), _ptr(kld),
                                  _ptr(flags), _ptr(rec), _stream(stream)), "dsde_vp_finalize")
        mass = torch.empty((n, B * self.nd_sh * 16), dtype=torch.uint8, device=dev)
        for s in range(n):
            t, d = target_shards[s], draft_shards[s]
            _check(L.dsde_vp_draw(st, B, self.V, n, s, dt, _ptr(rec), _ptr(t), t.stride(0), _ptr(d), d.stride(0),
                                  _ptr(mass[s]), _stream(stream)), "dsde_vp_draw")
        toks = torch.empty((n, B), dtype=torch.int32, device=dev)
        for s in range(n):
            t, d = target_shards[s], draft_shards[s]
            _check(L.dsde_vp_select(st, B, self.V, n, s, dt, _ptr(rec), _ptr(mass), _ptr(t), t.stride(0), _ptr(d),
                                    d.stride(0), _ptr(toks[s]), _stream(stream)), "dsde_vp_select")
        tok = toks.max(0).values.contiguous()  # the all-reduce (max)
        _check(L.dsde_vp_place(st, B, _ptr(rec), _ptr(tok), _ptr(emitted), _ptr(flags), _stream(stream)),
               "dsde_vp_place")
        return tok

    def workspace(self, B: int, total: int, device="cuda"):
        n = lib().dsde_vp_workspace_size(B, total, self.V, self.n, dtype_code(self.dtype))
        if n == 0:
            raise DsdeError("dsde_vp_workspace_size: invalid shape")
        ws = torch.empty(n + 256, dtype=torch.uint8, device=device)
        return ws[(-ws.data_ptr()) % 256:]

    def verify(self, cu_sl, draft_tokens, target_shard, draft_shard, seeds, accepted_len, emitted, kld,
               flags, workspace, comm: "Comm | None" = None, stream=None):
        """dsde_vp_verify: this rank's shard (rank = the communicator's; comm
        None = one shard)."""
        B = cu_sl.numel() - 1
        _check(lib().dsde_vp_verify(
            self.state.h, B, self.V, dtype_code(self.dtype), draft_tokens.numel(), _ptr(cu_sl), _ptr(draft_tokens),
            _ptr(target_shard), target_shard.stride(0), _ptr(draft_shard), draft_shard.stride(0), _ptr(seeds),
            _ptr(accepted_len), _ptr(emitted), _ptr(kld), _ptr(flags), _ptr(workspace), workspace.numel(),
            comm.h if comm is not None else None, _stream(stream)), "dsde_vp_verify")


def dsde_update_signal(state: State, slots, cu_sl, kld, accepted_len, sl_hat, diag=None, stream=None):
    _check(lib().dsde_update_signal(state.h, slots.numel(), _ptr(slots), _ptr(cu_sl), _ptr(kld),
                                    _ptr(accepted_len), _ptr(sl_hat), _ptr(diag), _stream(stream)),
           "dsde_update_signal")


def dsde_next_sl(state: State, slots, sl_hat, budget, next_sl, cap, comm: Comm | None = None, stream=None):
    _check(lib().dsde_next_sl(state.h, slots.numel(), _ptr(slots), _ptr(sl_hat), _ptr(budget),
                              _ptr(next_sl), _ptr(cap), comm.h if comm is not None else None,
                              _stream(stream)), "dsde_next_sl")


def dsde_step(state: State, V: int, total_draft_rows: int, slots, cu_sl, draft_tokens, target_logits,
              draft_logits, seeds, budget, accepted_len, emitted_tokens, kld, flags, sl_hat, diag, next_sl,
              cap, workspace, comm: Comm | None = None, stream=None):
    """dsde_step (include/dsde.h): verify -> update_signal -> next_sl in one call."""
    B = cu_sl.numel() - 1
    _check(lib().dsde_step(
        state.h, B, int(V), dtype_code(target_logits.dtype), int(total_draft_rows), _ptr(slots), _ptr(cu_sl),
        _ptr(draft_tokens), _ptr(target_logits), target_logits.stride(0), _ptr(draft_logits),
        draft_logits.stride(0), _ptr(seeds), _ptr(budget), _ptr(accepted_len), _ptr(emitted_tokens), _ptr(kld),
        _ptr(flags), _ptr(sl_hat), _ptr(diag), _ptr(next_sl), _ptr(cap), _ptr(workspace), workspace.numel(),
        comm.h if comm is not None else None, _stream(stream)), "dsde_step")


@dataclass
class StepOut:
    accepted_len: torch.Tensor   # int32 [B]
    emitted: torch.Tensor        # int32 [sum k + B]
    kld: torch.Tensor            # float32 [sum k]
    flags: torch.Tensor          # uint8 [sum k + B]
    sl_hat: torch.Tensor         # int32 [B]
    next_sl: torch.Tensor        # int32 [B]
    cap: torch.Tensor            # int32 [1]
    diag: torch.Tensor | None    # float64 [B, 8]


class Step:
    """One DSDE decoding step on a batch: verify -> update_signal -> next_sl.

    Owns the workspace and output buffers for a maximum batch shape so a step
    allocates nothing (the launches can be captured in a CUDA graph)."""

    def __init__(self, state: State, B: int, V: int, dtype: torch.dtype, max_draft_rows: int | None = None,
                 with_diag: bool = False, comm: Comm | None = None, device="cuda"):
        self.state, self.B, self.V, self.dtype, self.comm = state, B, V, dtype, comm
        nmax = max_draft_rows if max_draft_rows is not None else B * DSDE_MAX_SL
        self.ws = torch.empty(workspace_size(B, nmax, V, dtype) + 256, dtype=torch.uint8, device=device)
        off = (-self.ws.data_ptr()) % 256
        self.ws = self.ws[off:]
        i32 = dict(dtype=torch.int32, device=device)
        self.accepted_len = torch.empty(B, **i32)
        self.emitted = torch.empty(nmax + B, **i32)
        self.kld = torch.empty(nmax, dtype=torch.float32, device=device)
        self.flags = torch.empty(nmax + B, dtype=torch.uint8, device=device)
        self.sl_hat = torch.empty(B, **i32)
        self.next_sl = torch.empty(B, **i32)
        self.cap = torch.empty(1, **i32)
        self.diag = torch.empty((B, 8), dtype=torch.float64, device=device) if with_diag else None
        self.slots = torch.arange(B, **i32)

    def _batch(self, cu_sl) -> int:
        B = cu_sl.numel() - 1
        if not 1 <= B <= self.B:
            raise DsdeError(f"batch of {B} sequences for a Step sized for {self.B}")
        return B

    def verify(self, cu_sl, draft_tokens, target, draft, seeds, total_draft_rows: int, stream=None):
        n, B = total_draft_rows, self._batch(cu_sl)
        dsde_verify(self.state, self.V, n, cu_sl, draft_tokens, target, draft, seeds,
                    self.accepted_len[:B], self.emitted[: n + B], self.kld[:n], self.flags[: n + B],
                    self.ws, stream)

    def signal_and_cap(self, cu_sl, budget=None, stream=None):
        """Batch B = cu_sl.numel() - 1 <= the Step's size: slots [0, B) (the same slots dsde_step uses)."""
        B = self._batch(cu_sl)
        dsde_update_signal(self.state, self.slots[:B], cu_sl, self.kld, self.accepted_len[:B], self.sl_hat[:B],
                           None if self.diag is None else self.diag[:B], stream)
        dsde_next_sl(self.state, self.slots[:B], self.sl_hat[:B], budget, self.next_sl[:B], self.cap, self.comm,
                     stream)

    def __call__(self, cu_sl, draft_tokens, target, draft, seeds, total_draft_rows: int, budget=None,
                 stream=None, fused: bool = True) -> StepOut:
        n, B = total_draft_rows, self._batch(cu_sl)
        diag = None if self.diag is None else self.diag[:B]
        if fused:  # one dsde_step call (+ the NCCL cap at N > 1)
            dsde_step(self.state, self.V, n, self.slots[:B], cu_sl, draft_tokens, target, draft, seeds, budget,
                      self.accepted_len[:B], self.emitted[: n + B], self.kld[:n], self.flags[: n + B],
                      self.sl_hat[:B], diag, self.next_sl[:B], self.cap, self.ws, self.comm, stream)
        else:
            self.verify(cu_sl, draft_tokens, target, draft, seeds, total_draft_rows, stream)
            self.signal_and_cap(cu_sl, budget, stream)
        return StepOut(self.accepted_len[:B], self.emitted[: n + B], self.kld[:n], self.flags[: n + B],
                       self.sl_hat[:B], self.next_sl[:B], self.cap, diag)
