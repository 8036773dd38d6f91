"""ctypes mirror of ``include/semsched_b200.h`` (the C-ABI structs).

Kept separate from the loader so the test-side oracle binding can reuse the
same struct layouts without touching the product library.
"""

from __future__ import annotations

import ctypes as C

SS_OK = 0
SS_ERR_INVALID_ARG = 1
SS_ERR_CUDA = 2
SS_ERR_TRACE_FAILED = 3
SS_ERR_NO_DEVICE = 4
SS_ERR_UNSUPPORTED = 5

SS_TRACE_OK = 0
SS_TRACE_LIVELOCK = 1
SS_TRACE_ROUND_CAP = 2
SS_TRACE_LOG_OVERFLOW = 3
SS_TRACE_INTERNAL = 4
SS_TRACE_REF_ERROR = 6
TRACE_STATUS_NAMES = {0: "ok", 1: "livelock", 2: "round_cap", 3: "log_overflow", 4: "internal",
                      6: "reference_error"}

SS_POLICY = {"semantic": 0, "fcfs": 1, "sjf": 2, "hpjf": 3}
SS_FLAG_ROUND_LOG = 1
SS_FLAG_DIGEST = 2
SS_FLAG_FORCE_CHUNKED = 4
SS_FLAG_FORCE_PERROUND = 8
SS_MAX_BATCH = 32
SS_MAX_LEVELS = 16
SS_MAX_TRACE_REQS = 1 << 24
SS_BULK_MIN_DEFAULT = 1024
SS_EPILOGUE_MIN_DEFAULT = 16384

SS_STAGE_WAITING = 0
SS_STAGE_DECODING = 2
SS_STAGE_COMPLETED = 5
SS_STAGE_UNSERVABLE = 6

SS_LOG_HEADER_WORDS = 8
SS_LOG_DECISION_WORDS = 9
SS_KIND_DECODE, SS_KIND_PREFILL, SS_KIND_NONE = 0, 1, 2


class ss_profile(C.Structure):
    _fields_ = [("alpha1", C.c_double), ("alpha2", C.c_double), ("gamma1", C.c_double),
                ("gamma2", C.c_double), ("beta_load", C.c_double), ("beta_save", C.c_double)]


class ss_params(C.Structure):
    _fields_ = [("profile", ss_profile), ("memory_capacity", C.c_int64),
                ("batch_size", C.c_int32), ("policy", C.c_int32),
                ("dependency_rule", C.c_int32), ("decode_cost_sum", C.c_int32),
                ("levels", C.c_int32), ("flags", C.c_uint32), ("max_rounds", C.c_int64),
                ("bulk_min", C.c_int64), ("epilogue_min", C.c_int64)]


class ss_trace_batch(C.Structure):
    _fields_ = [("n_traces", C.c_int32), ("_pad", C.c_int32), ("n_requests", C.c_int64),
                ("trace_offsets", C.c_void_p), ("ready_time", C.c_void_p),
                ("arrival_time", C.c_void_p), ("prompt_len", C.c_void_p),
                ("true_output_len", C.c_void_p), ("pred_len", C.c_void_p),
                ("pred_urgency", C.c_void_p), ("true_urgency", C.c_void_p),
                ("tie_rank", C.c_void_p)]


class ss_trace_stats(C.Structure):
    _fields_ = [("digest", C.c_uint64), ("rounds", C.c_int64), ("evictions", C.c_int64),
                ("mem_used_peak", C.c_int64), ("log_words", C.c_int64),
                ("completed", C.c_int32), ("unservable", C.c_int32), ("status", C.c_int32),
                ("lost_evictions", C.c_int32), ("anomalies", C.c_int32), ("_pad", C.c_int32),
                ("sum_pool", C.c_int64), ("sum_granted", C.c_int64), ("sum_victims", C.c_int64),
                ("sum_resident_evict", C.c_int64), ("final_clock", C.c_double), ("sum_wait", C.c_double),
                ("sum_norm_wait", C.c_double), ("level_norm_sum", C.c_double * SS_MAX_LEVELS),
                ("level_count", C.c_int32 * SS_MAX_LEVELS)]


class ss_request_out(C.Structure):
    _fields_ = [("first_scheduled", C.c_void_p), ("finish_time", C.c_void_p),
                ("generated", C.c_void_p), ("evictions", C.c_void_p),
                ("f_t", C.c_void_p), ("state", C.c_void_p)]


class ss_outputs(C.Structure):
    _fields_ = [("req", ss_request_out), ("stats", C.c_void_p),
                ("unservable_slots", C.c_void_p), ("round_log", C.c_void_p),
                ("log_offsets", C.c_void_p)]


STATS_DTYPE = None


def stats_dtype():
    """numpy structured dtype matching ss_trace_stats (for bulk reads)."""
    global STATS_DTYPE
    if STATS_DTYPE is None:
        import numpy as np

        STATS_DTYPE = np.dtype([
            ("digest", "<u8"), ("rounds", "<i8"), ("evictions", "<i8"), ("mem_used_peak", "<i8"),
            ("log_words", "<i8"), ("completed", "<i4"), ("unservable", "<i4"), ("status", "<i4"),
            ("lost_evictions", "<i4"), ("anomalies", "<i4"), ("_pad", "<i4"),
            ("sum_pool", "<i8"), ("sum_granted", "<i8"), ("sum_victims", "<i8"), ("sum_resident_evict", "<i8"),
            ("final_clock", "<f8"), ("sum_wait", "<f8"), ("sum_norm_wait", "<f8"),
            ("level_norm_sum", "<f8", (SS_MAX_LEVELS,)), ("level_count", "<i4", (SS_MAX_LEVELS,)),
        ])
        assert STATS_DTYPE.itemsize == C.sizeof(ss_trace_stats)
    return STATS_DTYPE
