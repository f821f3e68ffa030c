"""ctypes prototypes of include/starsd.h.  Loading fails loudly if libstarsd.so is missing:
there is no CPU fallback anywhere on the product path."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstarsd.so")

SD_OK = 0
STATUS_NAMES = {0: "SD_OK", 1: "SD_ERR_INVALID_ARGUMENT", 2: "SD_ERR_UNSUPPORTED",
                3: "SD_ERR_CUDA", 4: "SD_ERR_NCCL", 5: "SD_ERR_TIMEOUT", 6: "SD_ERR_NOT_READY",
                7: "SD_ERR_INTERNAL"}
SD_DTYPE_F32, SD_DTYPE_BF16 = 0, 1
SD_ERR_TIMEOUT, SD_ERR_NOT_READY = 5, 6
SD_STAR_ID_BYTES = 128
STAR_ID_BYTES = 128

# every symbol the header declares (tests check the library exports all of them)
EXPORTS = ["sd_verify", "sd_verify_workspace_size", "sd_philox_uniforms", "sd_star_unique_ids",
           "sd_star_create", "sd_star_round", "sd_star_poll", "sd_star_draft_begin",
           "sd_star_draft_end", "sd_star_stats", "sd_star_destroy", "sd_status_string",
           "sd_last_error", "sd_version", "sd_profile_events", "sd_profile_timestamps", "sd_debug_trace",
           "sd_star_simulate", "sd_verify_plan", "sd_verify_trace", "sd_star_simulate_ex",
           "sd_star_analytics", "sd_star_observe", "sd_star_predict", "sd_star_draft_begin_v",
           "sd_sched_create", "sd_sched_push", "sd_sched_pop", "sd_sched_service",
           "sd_sched_observe", "sd_sched_stats", "sd_sched_predict", "sd_sched_destroy",
           "sd_draft_workspace_size", "sd_draft_sample", "sd_draft_qmeta", "sd_verify_qmeta",
           "sd_tree_verify", "sd_verify_staged"]


class Shape(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("k", ctypes.c_int32), ("vocab", ctypes.c_int32),
                ("ld_p", ctypes.c_int64), ("ld_q", ctypes.c_int64), ("dtype", ctypes.c_int32)]


class Plan(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("launches", ctypes.c_int32),
                ("cluster", ctypes.c_int32), ("slice", ctypes.c_int32), ("ctas", ctypes.c_int64),
                ("tail_ctas", ctypes.c_int64), ("tagged", ctypes.c_int32), ("options", ctypes.c_int32)]


PLAN_OPTIONS = {2: "early"}


VARIANT_NAMES = {1: "two_launch"}


class StarConfig(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("n_slots", ctypes.c_int32),
                ("max_shape", Shape), ("temperature", ctypes.c_float), ("seed", ctypes.c_uint64),
                ("timeout_ms", ctypes.c_int32), ("device", ctypes.c_int32),
                ("transport", ctypes.c_int32), ("target_ms", ctypes.c_float),
                ("payload", ctypes.c_int32)]


SD_STAR_NCCL, SD_STAR_LOOPBACK = 0, 1
SD_STAR_PAYLOAD_FULL, SD_STAR_PAYLOAD_QMETA = 0, 1


class RoundDesc(ctypes.Structure):
    _fields_ = [("verifier", ctypes.c_int32), ("slot", ctypes.c_int32), ("round", ctypes.c_uint64),
                ("batch", ctypes.c_int32), ("request_id_base", ctypes.c_uint64),
                ("p_logits", ctypes.c_void_p), ("draft_ids", ctypes.c_void_p),
                ("q_logits", ctypes.c_void_p), ("out_accept_len", ctypes.c_void_p),
                ("out_tokens", ctypes.c_void_p), ("q_meta", ctypes.c_void_p)]


class StarStats(ctypes.Structure):
    _fields_ = [("busy_fraction", ctypes.c_double), ("mean_idle_ms", ctypes.c_double),
                ("mean_wait_ms", ctypes.c_double), ("window_ms", ctypes.c_double),
                ("rounds", ctypes.c_uint64)]


class Prediction(ctypes.Structure):
    _fields_ = [("expected_accepted", ctypes.c_double), ("t_idle_ms", ctypes.c_double),
                ("t_gamma_ms", ctypes.c_double), ("throughput_per_ms", ctypes.c_double),
                ("per_target_min_per_ms", ctypes.c_double), ("busy_fraction", ctypes.c_double),
                ("n_full", ctypes.c_int32), ("n_max", ctypes.c_int32),
                ("service_ms", ctypes.c_double), ("return_ms", ctypes.c_double)]


class StarsdError(RuntimeError):
    pass


_lib = None


def load():
    """Load libstarsd.so (built by paper_2601_21622_b200.build / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise StarsdError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (the CUDA extension is required; there is no fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, u32, i64, u64, sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32,
                                  ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t)
    st = ctypes.c_int
    L.sd_verify.argtypes = [vp, vp, vp, ctypes.POINTER(Shape), ctypes.c_float, u64, u64, u64,
                            vp, vp, vp, vp, sz, vp]
    L.sd_verify.restype = st
    L.sd_verify_workspace_size.argtypes = [ctypes.POINTER(Shape), ctypes.c_float,
                                           ctypes.POINTER(sz)]
    L.sd_verify_workspace_size.restype = st
    L.sd_verify_plan.argtypes = [ctypes.POINTER(Shape), ctypes.c_float, ctypes.POINTER(Plan)]
    L.sd_verify_plan.restype = st
    L.sd_verify_qmeta.argtypes = [vp, vp, vp, vp, ctypes.POINTER(Shape), ctypes.c_float, u64, u64,
                                  u64, vp, vp, vp, vp, sz, vp]
    L.sd_verify_qmeta.restype = st
    L.sd_verify_staged.argtypes = [vp, vp, vp, ctypes.POINTER(Shape), ctypes.c_float, u64, u64, u64,
                                   vp, vp, vp, vp, sz, vp, vp, vp]
    L.sd_verify_staged.restype = st
    L.sd_draft_workspace_size.argtypes = [ctypes.POINTER(Shape), ctypes.c_float, ctypes.POINTER(sz)]
    L.sd_draft_workspace_size.restype = st
    L.sd_draft_sample.argtypes = [vp, ctypes.POINTER(Shape), ctypes.c_float, u64, u64, u64, vp, vp,
                                  vp, vp, sz, vp]
    L.sd_draft_sample.restype = st
    L.sd_draft_qmeta.argtypes = [vp, vp, ctypes.POINTER(Shape), ctypes.c_float, vp, vp, sz, vp]
    L.sd_draft_qmeta.restype = st
    L.sd_tree_verify.argtypes = [vp, vp, vp, ctypes.POINTER(Shape), i32, ctypes.c_float, u64, u64,
                                 u64, vp, vp, vp, vp, vp]
    L.sd_tree_verify.restype = st
    L.sd_verify_trace.argtypes = [ctypes.POINTER(Shape), ctypes.c_float, vp, vp, vp, vp, vp, vp, vp]
    L.sd_verify_trace.restype = st
    L.sd_philox_uniforms.argtypes = [u64, u64, vp, vp, i32, vp, vp]
    L.sd_philox_uniforms.restype = st
    L.sd_star_unique_ids.argtypes = [i32, vp]
    L.sd_star_unique_ids.restype = st
    L.sd_star_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(StarConfig), vp]
    L.sd_star_create.restype = st
    L.sd_star_round.argtypes = [vp, ctypes.POINTER(RoundDesc), vp]
    L.sd_star_round.restype = st
    L.sd_star_poll.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32),
                               ctypes.POINTER(u64), i32]
    L.sd_star_poll.restype = st
    L.sd_star_draft_begin.argtypes = [vp, vp]
    L.sd_star_draft_begin.restype = st
    L.sd_star_draft_end.argtypes = [vp, vp]
    L.sd_star_draft_end.restype = st
    L.sd_star_stats.argtypes = [vp, ctypes.POINTER(StarStats)]
    L.sd_star_stats.restype = st
    L.sd_star_destroy.argtypes = [vp]
    L.sd_star_destroy.restype = st
    L.sd_star_simulate.argtypes = [i32, i32, ctypes.c_double, ctypes.c_double, i32,
                                   ctypes.POINTER(StarStats)]
    L.sd_star_simulate.restype = st
    dbl = ctypes.c_double
    pd = ctypes.POINTER(dbl)
    L.sd_star_simulate_ex.argtypes = [i32, i32, vp, vp, i32, vp, ctypes.POINTER(StarStats)]
    L.sd_star_simulate_ex.restype = st
    L.sd_star_analytics.argtypes = [i32, vp, i32, dbl, dbl, dbl, ctypes.POINTER(Prediction)]
    L.sd_star_analytics.restype = st
    L.sd_star_observe.argtypes = [vp, i32, vp, i32]
    L.sd_star_observe.restype = st
    L.sd_star_predict.argtypes = [vp, dbl, ctypes.POINTER(Prediction)]
    L.sd_star_predict.restype = st
    L.sd_star_draft_begin_v.argtypes = [vp, i32, vp]
    L.sd_star_draft_begin_v.restype = st
    L.sd_sched_create.argtypes = [ctypes.POINTER(vp), i32, i32]
    L.sd_sched_create.restype = st
    L.sd_sched_push.argtypes = [vp, i32, i32, u64, dbl]
    L.sd_sched_push.restype = st
    L.sd_sched_pop.argtypes = [vp, dbl, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(u64)]
    L.sd_sched_pop.restype = st
    L.sd_sched_service.argtypes = [vp, i32, dbl, dbl]
    L.sd_sched_service.restype = st
    L.sd_sched_observe.argtypes = [vp, i32, dbl, vp, i32]
    L.sd_sched_observe.restype = st
    L.sd_sched_stats.argtypes = [vp, ctypes.POINTER(StarStats)]
    L.sd_sched_stats.restype = st
    L.sd_sched_predict.argtypes = [vp, dbl, ctypes.POINTER(Prediction)]
    L.sd_sched_predict.restype = st
    L.sd_sched_destroy.argtypes = [vp]
    L.sd_sched_destroy.restype = st
    L.sd_profile_events.argtypes = [vp, i32]
    L.sd_profile_events.restype = st
    L.sd_profile_timestamps.argtypes = [vp, i32]
    L.sd_profile_timestamps.restype = st
    L.sd_debug_trace.argtypes = [vp]
    L.sd_debug_trace.restype = st
    L.sd_status_string.argtypes = [st]
    L.sd_status_string.restype = ctypes.c_char_p
    L.sd_last_error.argtypes = []
    L.sd_last_error.restype = ctypes.c_char_p
    L.sd_version.argtypes = []
    L.sd_version.restype = ctypes.c_char_p
    _lib = L
    return L


def check(rc: int, what: str):
    if rc != SD_OK:
        L = load()
        raise StarsdError(f"{what}: {STATUS_NAMES.get(rc, rc)}: "
                          f"{L.sd_last_error().decode(errors='replace')}")
    return rc
