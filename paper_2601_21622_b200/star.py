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
                 transport: str = "nccl", timeout_ms: int = 60000, target_ms: float = 0.0,
                 payload: str = "full"):
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
                              tcode, float(target_ms),
                              {"full": _lib.SD_STAR_PAYLOAD_FULL, "qmeta": _lib.SD_STAR_PAYLOAD_QMETA}[payload])
        self._h = ctypes.c_void_p()
        idbuf = None if ids is None else ctypes.create_string_buffer(ids, len(ids))
        check(self._L.sd_star_create(ctypes.byref(self._h), ctypes.byref(cfg), idbuf),
              "sd_star_create")

    def _stream(self, stream):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def submit(self, verifier: int, slot: int, round: int, ids: torch.Tensor,
               q: torch.Tensor | None, accept_len: torch.Tensor, tokens: torch.Tensor,
               request_id_base: int = 0, p: torch.Tensor | None = None, stream=None,
               qmeta: torch.Tensor | None = None):
        """Draft: send (ids [B,k], q [B,k,V]) -- or, with payload="qmeta", ids + qmeta [B,k,3]
        (sd_qmeta records from draft_sample / draft_qmeta; q must then stay valid until the round
        returns) -- to `verifier` for `slot` and post the receive of (accept_len [B],
        tokens [B,k+1]).  Returns immediately; completion shows up in poll()."""
        d = _lib.RoundDesc(verifier, slot, round, ids.shape[0], request_id_base, _ptr(p),
                           _ptr(ids), _ptr(q), _ptr(accept_len), _ptr(tokens), _ptr(qmeta))
        check(self._L.sd_star_round(self._h, ctypes.byref(d), self._stream(stream)),
              "sd_star_round")

    def serve(self, slot: int, round: int, batch: int, p: torch.Tensor,
              accept_len: torch.Tensor, tokens: torch.Tensor, request_id_base: int = 0,
              stream=None):
        """Verifier: receive the round's (ids, q), verify against p [B,k+1,V], send results."""
        d = _lib.RoundDesc(self.rank, slot, round, batch, request_id_base, _ptr(p), None, None,
                           _ptr(accept_len), _ptr(tokens), None)
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


def simulate_trace(trace: dict, service_ms: float, return_ms: float, beta, k: int,
                   n_slots: int = 2, max_active: int = 128, seed: int = 0,
                   window_ms: float = 1000.0, until_ms: float | None = None) -> dict:
    """Trace-driven star (BASELINE config 5, bursty arrivals): the draft's FIFO scheduler (the same
    sd_sched_* the NCCL star runs) serves rounds of per-verifier cohorts whose membership follows
    the request trace.  trace: {v: [(arrival_ms, length_tokens), ...]} (workload.bursty_trace).
    A verifier keeps <= max_active requests in n_slots cohorts; a cohort with at least one active
    request issues its next round when its previous one returned (closed loop); a round costs
    the draft service_ms (S(d), Eq. 5, independent of the batch) and returns return_ms later
    (Z(d), Eq. 6); each request emits L + 1 tokens per round, L ~ truncated geometric with per-
    verifier acceptance beta[v-1] (Lemma 1, i.i.d. acceptance).  Returns the busy fraction overall
    and per window, per-verifier tokens/s, mean T_wait and completed requests.  Runs until every
    request completed, or until the draft clock reaches until_ms."""
    import heapq

    import numpy as np
    rng = np.random.default_rng(seed)
    nv = len(trace)
    beta = np.broadcast_to(np.asarray(beta, np.float64), (nv,))
    sched = Scheduler(nv, k)
    arrivals = {v: list(trace[v]) for v in trace}
    nxt = {v: 0 for v in trace}
    active = {(v, s): [] for v in trace for s in range(n_slots)}     # [remaining, length]
    count = {v: 0 for v in trace}
    waiting_stream = {(v, s): True for v in trace for s in range(n_slots)}  # no round in flight
    tokens = np.zeros(nv)
    done_req = 0
    events = []        # (t, kind, v, s): kind 0 = return, 1 = arrival wake-up
    for v in trace:
        if arrivals[v]:
            heapq.heappush(events, (arrivals[v][0][0], 1, v, -1))
    t = 0.0
    busy = []
    last_t = max((r[-1][0] for r in arrivals.values() if r), default=0.0)

    def admit(v, now):
        while nxt[v] < len(arrivals[v]) and arrivals[v][nxt[v]][0] <= now and count[v] < max_active:
            ln = arrivals[v][nxt[v]][1]
            s = nxt[v] % n_slots
            active[(v, s)].append([ln, ln])
            count[v] += 1
            nxt[v] += 1

    def ready(v, now):
        for s in range(n_slots):
            if waiting_stream[(v, s)] and active[(v, s)]:
                waiting_stream[(v, s)] = False
                sched.push(v, s, 0, now)
        if nxt[v] < len(arrivals[v]) and count[v] < max_active:
            heapq.heappush(events, (max(now, arrivals[v][nxt[v]][0]), 1, v, -1))

    while True:
        # move every event due by t into the queue
        while events and events[0][0] <= t:
            te, kind, v, s = heapq.heappop(events)
            if kind == 0:                                   # a round of (v, s) returned
                reqs = active[(v, s)]
                L = np.minimum(rng.geometric(1.0 - beta[v - 1], len(reqs)) - 1, k) \
                    if beta[v - 1] < 1.0 else np.full(len(reqs), k)
                keep = []
                for rq, l in zip(reqs, L):
                    emit = min(int(l) + 1, rq[0])
                    tokens[v - 1] += emit
                    rq[0] -= emit
                    if rq[0] > 0:
                        keep.append(rq)
                    else:
                        done_req += 1
                        count[v] -= 1
                active[(v, s)] = keep
                waiting_stream[(v, s)] = True
                sched.observe(v, return_ms, L.astype(np.int32))
            admit(v, te)
            ready(v, te)
        if until_ms is not None and t >= until_ms:
            break
        got = sched.pop(t)
        if got is None:
            if not events:
                break
            t = events[0][0]                                # the draft idles (T_idle)
            continue
        v, s, _ = got
        sched.service(v, t, t + service_ms)
        busy.append((t, t + service_ms))
        t += service_ms
        heapq.heappush(events, (t + return_ms, 0, v, s))
        if t > last_t + 1e6:
            break
    st = sched.stats()
    horizon = max(b[1] for b in busy) if busy else 0.0
    nw = int(np.ceil(horizon / window_ms)) if horizon > 0 else 0
    per_win = np.zeros(nw)
    for a, b in busy:
        w0, w1 = int(a // window_ms), int(min(b, horizon - 1e-9) // window_ms)
        for w in range(w0, w1 + 1):
            lo, hi = max(a, w * window_ms), min(b, (w + 1) * window_ms)
            if hi > lo:
                per_win[w] += hi - lo
    out = {"busy_fraction": float(sum(b - a for a, b in busy) / horizon) if horizon else 0.0,
           "busy_per_window": (per_win / window_ms).tolist(),
           "tokens_per_s": (tokens / (horizon / 1000.0)).tolist() if horizon else [0.0] * nv,
           "mean_wait_ms": st["mean_wait_ms"], "rounds": st["rounds"],
           "completed_requests": done_req, "horizon_ms": horizon}
    sched.close()
    return out
