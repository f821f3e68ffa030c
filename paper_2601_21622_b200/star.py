"""Star exchange + round scheduler binding (include/starsd.h sd_star_*).

PAPER.md Alg. 1: one draft instance (rank 0) serves N verifiers (ranks 1..N); each
(0, v) pair has its own channel.  The draft submits a round per (verifier, slot),
polls the global FIFO buffer Q_in for completed returns and drafts the next round
for whichever verifier came back first -- work-conserving, no synchronization barrier across
verifiers.  Marshalling only: the scheduler, transport and verify run in
libstarsd.so.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import StarsdError, check


def simulate(n_verifiers: int, n_slots: int, service_ms: float, return_ms: float,
             rounds: int) -> dict:
    """sd_star_simulate: the scheduler under a deterministic fake transport (host only).
    service_ms = S(d) (Eq. 5), return_ms = Z(d) = t_c + t_v (Eq. 6)."""
    st = _lib.StarStats()
    check(_lib.load().sd_star_simulate(n_verifiers, n_slots, float(service_ms), float(return_ms),
                                       rounds, ctypes.byref(st)), "sd_star_simulate")
    return _stats_dict(st)


def simulate_ex(service_ms, return_ms, n_slots: int, rounds: int) -> dict:
    """sd_star_simulate_ex: heterogeneous star (per-verifier S_v, Z_v) under the fake transport;
    adds the per-verifier services counted in the window."""
    import numpy as np
    S = np.ascontiguousarray(service_ms, np.float64)
    Z = np.ascontiguousarray(return_ms, np.float64)
    n = S.shape[0]
    per = np.zeros(n, np.uint64)
    st = _lib.StarStats()
    check(_lib.load().sd_star_simulate_ex(n, n_slots, S.ctypes.data, Z.ctypes.data, rounds,
                                          per.ctypes.data, ctypes.byref(st)), "sd_star_simulate_ex")
    d = _stats_dict(st)
    d["rounds_per_verifier"] = per.tolist()
    return d


def _pred_dict(p) -> dict:
    return {f: getattr(p, f) for f, _ in _lib.Prediction._fields_}


def analytics(beta, d: int, service_ms: float, return_ms: float, o_alone_per_ms: float) -> dict:
    """sd_star_analytics: Sec. 4 closed forms (Eqs. 3-11), N_full and the admission bound N_max."""
    import numpy as np
    b = np.ascontiguousarray(beta, np.float64)
    out = _lib.Prediction()
    check(_lib.load().sd_star_analytics(b.shape[0], b.ctypes.data, d, float(service_ms),
                                        float(return_ms), float(o_alone_per_ms),
                                        ctypes.byref(out)), "sd_star_analytics")
    return _pred_dict(out)


class Scheduler:
    """sd_sched_*: the star's host-side FIFO scheduler + online estimators, transport-free."""

    def __init__(self, n_verifiers: int, k: int):
        self._L = _lib.load()
        self._h = ctypes.c_void_p()
        check(self._L.sd_sched_create(ctypes.byref(self._h), n_verifiers, k), "sd_sched_create")

    def push(self, verifier: int, slot: int, round: int, t_ms: float):
        check(self._L.sd_sched_push(self._h, verifier, slot, round, float(t_ms)), "sd_sched_push")

    def pop(self, now_ms: float):
        v, s, r = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint64()
        rc = self._L.sd_sched_pop(self._h, float(now_ms), ctypes.byref(v), ctypes.byref(s),
                                  ctypes.byref(r))
        if rc == _lib.SD_ERR_NOT_READY:
            return None
        check(rc, "sd_sched_pop")
        return v.value, s.value, r.value

    def service(self, verifier: int, t0_ms: float, t1_ms: float):
        check(self._L.sd_sched_service(self._h, verifier, float(t0_ms), float(t1_ms)),
              "sd_sched_service")

    def observe(self, verifier: int, return_ms: float, accept_len=None):
        import numpy as np
        a = np.ascontiguousarray(accept_len if accept_len is not None else [], np.int32)
        check(self._L.sd_sched_observe(self._h, verifier, float(return_ms),
                                       a.ctypes.data if a.size else None, a.size),
              "sd_sched_observe")

    def stats(self) -> dict:
        st = _lib.StarStats()
        check(self._L.sd_sched_stats(self._h, ctypes.byref(st)), "sd_sched_stats")
        return _stats_dict(st)

    def predict(self, o_alone_per_ms: float) -> dict:
        out = _lib.Prediction()
        check(self._L.sd_sched_predict(self._h, float(o_alone_per_ms), ctypes.byref(out)),
              "sd_sched_predict")
        return _pred_dict(out)

    def close(self):
        if self._h:
            self._L.sd_sched_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stats_dict(st) -> dict:
    return {"busy_fraction": st.busy_fraction, "mean_idle_ms": st.mean_idle_ms,
            "mean_wait_ms": st.mean_wait_ms, "window_ms": st.window_ms, "rounds": st.rounds}


def predicted(n_verifiers: int, service_ms: float, return_ms: float) -> dict:
    """Closed forms of Sec. 4.1 (Eqs. 7-10) for one slot per verifier:
    T_idle = max(0, Z - (N-1) S), T_gamma = N S + T_idle, busy = N S / T_gamma,
    N_full = ceil(Z / S) + 1 (the smallest N with T_idle = 0)."""
    import math
    n, s, z = n_verifiers, service_ms, return_ms
    t_idle = max(0.0, z - (n - 1) * s)
    return {"t_idle_ms": t_idle, "t_gamma_ms": n * s + t_idle,
            "busy_fraction": n * s / (n * s + t_idle), "n_full": math.ceil(z / s) + 1}


def unique_ids(world: int) -> bytes:
    """Two communicator ids per (0, v) pair (draft -> verifier, verifier -> draft)."""
    buf = ctypes.create_string_buffer(2 * _lib.SD_STAR_ID_BYTES * (world - 1))
    check(_lib.load().sd_star_unique_ids(world, buf), "sd_star_unique_ids")
    return buf.raw


def exchange_ids(rank: int, world: int, group=None) -> bytes:
    """The one-time handshake: rank 0 creates one communicator id per (0, v) pair
    and broadcasts them over the already-initialised torch.distributed group."""
    import torch.distributed as dist
    obj = [unique_ids(world) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ids = obj[0]
    if not isinstance(ids, bytes) or len(ids) != 2 * _lib.SD_STAR_ID_BYTES * (world - 1):
        raise StarsdError("exchange_ids: malformed id blob")
    return ids


def _dt(dtype: torch.dtype) -> int:
    if dtype == torch.float32:
        return _lib.SD_DTYPE_F32
    if dtype == torch.bfloat16:
        return _lib.SD_DTYPE_BF16
    raise TypeError(f"dtype must be float32 or bfloat16, got {dtype}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Star:
    """One rank's handle.  transport="nccl": rank 0 = draft, ranks 1..world-1 = verifiers, one
    process per GPU, `ids` from exchange_ids().  transport="loopback": a single process plays
    the draft and world-1 virtual verifiers on one device (the exchange is a D2D copy; the
    draft's submit() then carries the verifier's target logits)."""

    def __init__(self, rank: int, world: int, max_batch: int, k: int, vocab: int,
                 temperature: float, seed: int = 0, n_slots: int = 2,
                 dtype: torch.dtype = torch.float32, device=None, ids: bytes | None = None,
                 transport: str = "nccl", timeout_ms: int = 60000, target_ms: float = 0.0):
        dev = torch.device(device if device is not None else "cuda")
        if dev.type != "cuda":
            raise StarsdError("Star needs a CUDA device")
        self.rank, self.world, self.k, self.vocab = rank, world, k, vocab
        self.temperature = float(temperature)
        self.device = dev
        self._L = _lib.load()
        tcode = {"nccl": _lib.SD_STAR_NCCL, "loopback": _lib.SD_STAR_LOOPBACK}[transport]
        cfg = _lib.StarConfig(rank, world, n_slots,
                              _lib.Shape(max_batch, k, vocab, vocab, vocab, _dt(dtype)),
                              self.temperature, seed, timeout_ms,
                              dev.index if dev.index is not None else torch.cuda.current_device(),
                              tcode, float(target_ms))
        self._h = ctypes.c_void_p()
        idbuf = None if ids is None else ctypes.create_string_buffer(ids, len(ids))
        check(self._L.sd_star_create(ctypes.byref(self._h), ctypes.byref(cfg), idbuf),
              "sd_star_create")

    def _stream(self, stream):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def submit(self, verifier: int, slot: int, round: int, ids: torch.Tensor,
               q: torch.Tensor | None, accept_len: torch.Tensor, tokens: torch.Tensor,
               request_id_base: int = 0, p: torch.Tensor | None = None, stream=None):
        """Draft: send (ids [B,k], q [B,k,V]) to `verifier` for `slot` and post the receive of
        (accept_len [B], tokens [B,k+1]).  Returns immediately; completion shows up in poll()."""
        d = _lib.RoundDesc(verifier, slot, round, ids.shape[0], request_id_base, _ptr(p),
                           _ptr(ids), _ptr(q), _ptr(accept_len), _ptr(tokens))
        check(self._L.sd_star_round(self._h, ctypes.byref(d), self._stream(stream)),
              "sd_star_round")

    def serve(self, slot: int, round: int, batch: int, p: torch.Tensor,
              accept_len: torch.Tensor, tokens: torch.Tensor, request_id_base: int = 0,
              stream=None):
        """Verifier: receive the round's (ids, q), verify against p [B,k+1,V], send results."""
        d = _lib.RoundDesc(self.rank, slot, round, batch, request_id_base, _ptr(p), None, None,
                           _ptr(accept_len), _ptr(tokens))
        check(self._L.sd_star_round(self._h, ctypes.byref(d), self._stream(stream)),
              "sd_star_round")

    def poll(self, timeout_us: int = 0):
        """Draft: next completed (verifier, slot, round) in FIFO order, or None.  Verifier: the
        oldest round whose results have been sent, or None."""
        v, s, r = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint64()
        rc = self._L.sd_star_poll(self._h, ctypes.byref(v), ctypes.byref(s), ctypes.byref(r),
                                  timeout_us)
        if rc in (_lib.SD_ERR_NOT_READY, _lib.SD_ERR_TIMEOUT):
            return None
        check(rc, "sd_star_poll")
        return v.value, s.value, r.value

    def draft_begin(self, stream=None, verifier: int = 0):
        check(self._L.sd_star_draft_begin_v(self._h, verifier, self._stream(stream)),
              "sd_star_draft_begin")

    def draft_end(self, stream=None):
        check(self._L.sd_star_draft_end(self._h, self._stream(stream)), "sd_star_draft_end")

    def stats(self) -> dict:
        st = _lib.StarStats()
        check(self._L.sd_star_stats(self._h, ctypes.byref(st)), "sd_star_stats")
        return _stats_dict(st)

    def observe(self, verifier: int, accept_len_host):
        """Draft: feed a returned round's accept lengths (host) into the online beta estimate."""
        import numpy as np
        a = np.ascontiguousarray(accept_len_host, np.int32)
        check(self._L.sd_star_observe(self._h, verifier, a.ctypes.data, a.size), "sd_star_observe")

    def predict(self, o_alone_per_ms: float) -> dict:
        """Draft: Sec. 4 closed forms on the online S(d), Z(d), beta; N_full and N_max."""
        out = _lib.Prediction()
        check(self._L.sd_star_predict(self._h, float(o_alone_per_ms), ctypes.byref(out)),
              "sd_star_predict")
        return _pred_dict(out)

    def close(self):
        if self._h:
            check(self._L.sd_star_destroy(self._h), "sd_star_destroy")
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
