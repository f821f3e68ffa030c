"""CPU oracle for the StarSD verify step (ctypes wrapper over ``oracle/starsd_ref.c``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2601_21622_b200``) never imports it, and it imports nothing from the product path.

The arithmetic lives in plain C99/fp64 (``starsd_ref.c``); this file only marshals numpy
arrays.  Citations for every function are in the C source (Alg. 2, and
the readings C-1..C-17 listed in DESIGN.md).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "starsd_ref.c")
_LIB_PATH = os.path.join(_HERE, "libstarsd_ref.so")
KMAX = 31

FAULT_BAD_DRAFT_ID = 1
FAULT_NONFINITE = 2
FAULT_EMPTY_ROW = 4
FAULT_ZERO_Q = 8
FAULT_ZERO_RESIDUAL = 16
HARD_FAULTS = FAULT_BAD_DRAFT_ID | FAULT_NONFINITE | FAULT_EMPTY_ROW


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math: fp64 semantics are the point)."""
    hdr = os.path.join(_HERE, "starsd_ref.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(_SRC), os.path.getmtime(hdr))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-fno-fast-math", "-ffp-contract=off",
                           "-D_POSIX_C_SOURCE=200809L", "-Wall", "-Wextra", "-fPIC", "-shared",
                           "-o", tmp, _SRC, "-lm", "-lpthread"])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Trace(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int32), ("token", ctypes.c_int32), ("status", ctypes.c_int32),
                ("n_tested", ctypes.c_int32),
                ("lam_p", ctypes.c_double * (KMAX + 1)), ("lam_q", ctypes.c_double * KMAX),
                ("ell", ctypes.c_double * KMAX), ("a", ctypes.c_double * KMAX),
                ("u_acc", ctypes.c_double * KMAX),
                ("R", ctypes.c_double), ("u_smp", ctypes.c_double), ("theta", ctypes.c_double),
                ("C_prev", ctypes.c_double), ("C_tok", ctypes.c_double),
                ("mu_a", ctypes.c_double), ("mu_s", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        vp, i32, i64, u64, dbl = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                  ctypes.c_uint64, ctypes.c_double)
        L.sd_ref_verify.argtypes = [vp, vp, vp, i32, i32, i32, i64, i64, i32, dbl, u64, u64, u64,
                                    vp, vp, vp, vp, i32]
        L.sd_ref_verify.restype = ctypes.c_int
        L.sd_ref_sample_check.argtypes = [vp, vp, vp, i32, i32, i32, i64, i64, i32, dbl, u64, u64,
                                          u64, i32, i32, vp, vp, vp, vp]
        L.sd_ref_sample_check.restype = ctypes.c_int
        L.sd_ref_accept_probs.argtypes = [vp, vp, vp, i32, i32, i32, i64, i64, i32, dbl, u64,
                                          u64, u64, vp, vp]
        L.sd_ref_accept_probs.restype = ctypes.c_int
        L.sd_ref_outcome_dist.argtypes = [vp, vp, vp, i32, i32, i32, i64, i64, i32, dbl, vp]
        L.sd_ref_outcome_dist.restype = ctypes.c_int
        L.sd_ref_draft_sample.argtypes = [vp, i32, i32, i32, i64, i32, dbl, u64, u64, u64, vp, vp,
                                          vp, vp]
        L.sd_ref_draft_sample.restype = ctypes.c_int
        L.sd_ref_tree_verify.argtypes = [vp, vp, vp, i32, i32, i32, i32, i64, i64, i32, dbl, u64,
                                         u64, u64, vp, vp, vp, vp, vp]
        L.sd_ref_tree_verify.restype = ctypes.c_int
        L.sd_ref_tree_outcome_dist.argtypes = [vp, vp, vp, i32, i32, i32, i32, i64, i64, i32, dbl,
                                               vp]
        L.sd_ref_tree_outcome_dist.restype = ctypes.c_int
        L.sd_ref_beta.argtypes = [vp, vp, i32, dbl]
        L.sd_ref_beta.restype = dbl
        L.sd_ref_softmax.argtypes = [vp, i32, dbl, vp]
        L.sd_ref_softmax.restype = None
        L.sd_ref_philox4x32_10.argtypes = [vp, vp, vp]
        L.sd_ref_philox4x32_10.restype = None
        L.sd_ref_uniforms.argtypes = [u64, ctypes.c_uint32, u64, u64, vp, vp]
        L.sd_ref_uniforms.restype = None
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _logits(a, name):
    """Accept float32 arrays (fp32 logits) or uint16 arrays (raw bf16 bits)."""
    if a is None:
        return None, None
    a = np.ascontiguousarray(a)
    if a.dtype == np.float32:
        return a, 0
    if a.dtype == np.uint16:
        return a, 1
    raise TypeError(f"{name}: expected float32 or uint16 (bf16 bits), got {a.dtype}")


def verify(p, q, ids, T, seed=0, round=0, rid_base=0, V=None, trace=False, n_threads=1):
    """Lazy step-by-step verify of a batch.

    p: [B, k+1, ld_p] logits, q: [B, k, ld_q] (None allowed iff T == 0), ids: [B, k] int32.
    Returns (L [B], tokens [B, k+1], status [B]) and, if ``trace``, a list of ``Trace``.
    """
    p, dt = _logits(p, "p")
    q, dq = _logits(q, "q")
    if q is not None and dq != dt:
        raise TypeError("p and q must have the same dtype")
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    B, k = ids.shape
    ld_p = p.shape[-1]
    ld_q = q.shape[-1] if q is not None else 0
    V = ld_p if V is None else V
    L = np.zeros(B, np.int32)
    tok = np.zeros((B, k + 1), np.int32)
    st = np.zeros(B, np.int32)
    tr = (Trace * B)() if trace else None
    rc = lib().sd_ref_verify(_ptr(p), _ptr(q), _ptr(ids), B, k, V, ld_p, ld_q, dt, float(T),
                             seed, round, rid_base, _ptr(L), _ptr(tok), _ptr(st),
                             ctypes.addressof(tr) if tr is not None else None, n_threads)
    if rc != 0:
        raise ValueError("sd_ref_verify: invalid argument")
    if trace:
        return L, tok, st, list(tr)
    return L, tok, st


def sample_check(p, q, ids, b, L, t, T, seed=0, round=0, rid_base=0, V=None):
    """C(t-1), C(t), R, theta of the sampling distribution at a forced stop position L."""
    p, dt = _logits(p, "p")
    q, _ = _logits(q, "q")
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    k = ids.shape[1]
    V = p.shape[-1] if V is None else V
    out = [ctypes.c_double() for _ in range(4)]
    rc = lib().sd_ref_sample_check(_ptr(p), _ptr(q), _ptr(ids), b, k, V, p.shape[-1],
                                   q.shape[-1], dt, float(T), seed, round, rid_base, L, t,
                                   *[ctypes.byref(o) for o in out])
    if rc != 0:
        raise ValueError("sd_ref_sample_check: invalid argument")
    return tuple(o.value for o in out)


def accept_probs(p, q, ids, b, T, seed=0, round=0, rid_base=0, V=None):
    """(a_j, u_acc(j)) for every position j of request b (no early stop)."""
    p, dt = _logits(p, "p")
    q, _ = _logits(q, "q")
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    k = ids.shape[1]
    V = p.shape[-1] if V is None else V
    a = np.zeros(k)
    u = np.zeros(k)
    rc = lib().sd_ref_accept_probs(_ptr(p), _ptr(q), _ptr(ids), b, k, V, p.shape[-1],
                                   q.shape[-1], dt, float(T), seed, round, rid_base, _ptr(a),
                                   _ptr(u))
    if rc != 0:
        raise ValueError("sd_ref_accept_probs: invalid argument")
    return a, u


def outcome_dist(p, q, ids, T, V=None):
    """Exact Pr(L = j, token = y) per request, shape [B, k+1, V] (uniforms integrated out)."""
    p, dt = _logits(p, "p")
    q, _ = _logits(q, "q")
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    B, k = ids.shape
    V = p.shape[-1] if V is None else V
    out = np.zeros((B, k + 1, V), np.float64)
    rc = lib().sd_ref_outcome_dist(_ptr(p), _ptr(q), _ptr(ids), B, k, V, p.shape[-1],
                                   q.shape[-1] if q is not None else 0, dt, float(T), _ptr(out))
    if rc != 0:
        raise ValueError("sd_ref_outcome_dist: invalid argument")
    return out


def draft_sample(q, T, seed=0, round=0, rid_base=0, V=None):
    """sd_ref_draft_sample on q [B, k, ld] (fp32, or uint16 raw bf16).  Returns (ids [B,k] int32,
    log q(x) [B,k], CDF margin mu [B,k], status [B,k])."""
    q = np.ascontiguousarray(q)
    dtype = 1 if q.dtype == np.uint16 else 0
    if dtype == 0:
        q = np.ascontiguousarray(q, np.float32)
    B, k, ld = q.shape
    V = ld if V is None else V
    ids = np.zeros((B, k), np.int32)
    logq = np.zeros((B, k), np.float64)
    mu = np.zeros((B, k), np.float64)
    st = np.zeros((B, k), np.int32)
    rc = lib().sd_ref_draft_sample(_ptr(q), B, k, V, ld, dtype, float(T), seed & (2**64 - 1),
                                   round & (2**64 - 1), rid_base & (2**64 - 1), _ptr(ids),
                                   _ptr(logq), _ptr(mu), _ptr(st))
    if rc != 0:
        raise ValueError("sd_ref_draft_sample: invalid argument")
    return ids, logq, mu, st


def tree_nodes(m, d):
    """(N, N_internal) of a full m-ary tree of depth d."""
    N = sum(m ** t for t in range(d + 1))
    return N, N - m ** d


def tree_verify(p, q, tok, m, d, T, seed=0, round=0, rid_base=0, V=None):
    """sd_ref_tree_verify: p [B, N, ld], q [B, N_int, ld] (None at T == 0), tok [B, N] int32.
    Returns (L [B], tokens [B, d+1], status [B], stop node [B], margin mu [B])."""
    p = np.ascontiguousarray(p)
    dtype = 1 if p.dtype == np.uint16 else 0
    if dtype == 0:
        p = np.ascontiguousarray(p, np.float32)
    if q is not None:
        q = np.ascontiguousarray(q, p.dtype)
    tok = np.ascontiguousarray(tok, np.int32)
    B, N, ld = p.shape
    V = ld if V is None else V
    L = np.zeros(B, np.int32)
    toks = np.zeros((B, d + 1), np.int32)
    st = np.zeros(B, np.int32)
    node = np.zeros(B, np.int32)
    mu = np.zeros(B, np.float64)
    rc = lib().sd_ref_tree_verify(_ptr(p), _ptr(q), _ptr(tok), B, m, d, V, ld,
                                  q.shape[-1] if q is not None else ld, dtype, float(T),
                                  seed & (2**64 - 1), round & (2**64 - 1), rid_base & (2**64 - 1),
                                  _ptr(L), _ptr(toks), _ptr(st), _ptr(node), _ptr(mu))
    if rc != 0:
        raise ValueError("sd_ref_tree_verify: invalid argument")
    return L, toks, st, node, mu


def tree_outcome_dist(p, q, tok, m, d, T):
    """sd_ref_tree_outcome_dist: [B, N, V] exact Pr(stop at node n, emit y)."""
    p = np.ascontiguousarray(p, np.float32)
    q = np.ascontiguousarray(q, np.float32)
    tok = np.ascontiguousarray(tok, np.int32)
    B, N, V = p.shape
    out = np.zeros((B, N, V), np.float64)
    rc = lib().sd_ref_tree_outcome_dist(_ptr(p), _ptr(q), _ptr(tok), B, m, d, V, V, V, 0,
                                        float(T), _ptr(out))
    if rc != 0:
        raise ValueError("sd_ref_tree_outcome_dist: invalid argument")
    return out


def beta(zp, zq, T=1.0):
    zp = np.ascontiguousarray(zp, np.float32)
    zq = np.ascontiguousarray(zq, np.float32)
    return lib().sd_ref_beta(_ptr(zp), _ptr(zq), zp.shape[-1], float(T))


def softmax(z, T=1.0):
    z = np.ascontiguousarray(z, np.float32)
    out = np.zeros(z.shape[-1], np.float64)
    lib().sd_ref_softmax(_ptr(z), z.shape[-1], float(T), _ptr(out))
    return out


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().sd_ref_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def uniforms(seed, j, round, rid):
    ua, us = ctypes.c_double(), ctypes.c_double()
    lib().sd_ref_uniforms(seed, j, round, rid, ctypes.byref(ua), ctypes.byref(us))
    return ua.value, us.value
