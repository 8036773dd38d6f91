"""Test-side binding of the CPU oracle (oracle/semsched_oracle.c).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may use this module.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2506_12204_b200 import _abi as A
from paper_2506_12204_b200.results import alloc_host_outputs, collect, log_capacity_words

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(REPO, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "build", "libsemsched_oracle.so")
_lib = None


def build_oracle() -> str:
    deps = [os.path.join(ORACLE_DIR, "semsched_oracle.c"), os.path.join(REPO, "include", "semsched_b200.h")]
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < max(os.path.getmtime(d) for d in deps):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
    return ORACLE_SO


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_oracle())
        _lib.so_run_traces.restype = C.c_int
        _lib.so_run_traces.argtypes = [C.POINTER(A.ss_params), C.POINTER(A.ss_trace_batch),
                                       C.c_void_p, C.POINTER(A.ss_outputs), C.c_int]
        for name, res, args in (
            ("so_prefill_time", C.c_double, [C.c_int64]),
            ("so_decode_step_time", C.c_double, [C.c_int64, C.c_int64]),
            ("so_decode_total_time", C.c_double, [C.c_int64, C.c_int64]),
            ("so_optimal_save_tokens", C.c_int64, [C.c_int64, C.c_int64]),
            ("so_resume_cost", C.c_double, [C.c_int64, C.c_int64, C.c_int64]),
            ("so_should_cache_prefill", C.c_int, [C.c_int64]),
            ("so_estimate_remaining_time", C.c_double, [C.c_int64] * 5),
        ):
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args + [C.POINTER(A.ss_profile)]
        _lib.so_audit.restype = None
        _lib.so_audit.argtypes = [C.c_int32] + [C.c_void_p] * 6
        _lib.so_pysum.restype = C.c_double
        _lib.so_pysum.argtypes = [C.c_void_p, C.c_int64]
    return _lib


def _ptr(a):
    return a.ctypes.data if a.size else None


def host_batch_struct(batch) -> A.ss_trace_batch:
    b = A.ss_trace_batch()
    b.n_traces = batch.n_traces
    b.n_requests = batch.n_requests
    b.trace_offsets = _ptr(batch.offsets)
    b.ready_time = _ptr(batch.ready)
    b.arrival_time = _ptr(batch.arrival)
    b.prompt_len = _ptr(batch.prompt)
    b.true_output_len = _ptr(batch.true_out)
    b.pred_len = _ptr(batch.pred_len)
    b.pred_urgency = _ptr(batch.pred_urg)
    b.true_urgency = _ptr(batch.true_urg)
    b.tie_rank = _ptr(batch.tie)
    return b


def run_oracle(params: A.ss_params, batch, threads: int = 1, use_ids: bool = True):
    """Run the oracle on a TraceBatch; returns a RunResult."""
    outs = alloc_host_outputs(batch.n_requests, batch.n_traces)
    log = log_off = None
    o = A.ss_outputs()
    if params.flags & A.SS_FLAG_ROUND_LOG:
        log_off = log_capacity_words(batch, params)
        log = np.zeros(max(int(log_off[-1]), 1), np.uint32)
        o.round_log = log.ctypes.data
        o.log_offsets = log_off.ctypes.data
    o.req = A.ss_request_out(outs["first_scheduled"].ctypes.data, outs["finish_time"].ctypes.data,
                             outs["generated"].ctypes.data, outs["evictions"].ctypes.data,
                             outs["f_t"].ctypes.data, outs["state"].ctypes.data)
    o.stats = outs["stats"].ctypes.data
    o.unservable_slots = outs["unservable"].ctypes.data
    hb = host_batch_struct(batch)
    ids = np.ascontiguousarray(batch.ids, np.int64) if use_ids else None
    rc = lib().so_run_traces(C.byref(params), C.byref(hb), _ptr(ids) if ids is not None else None,
                             C.byref(o), int(threads))
    res = collect(batch, outs, log, log_off)
    res.extra["rc"] = rc
    return res


def audit_oracle(offsets, finish, arrival, rank):
    """Eq. 2 counts per trace from the C restatement (test infrastructure)."""
    T = len(offsets) - 1
    arr = lambda x, dt: np.ascontiguousarray(np.asarray(x, dt))
    off, fin, av, rk = arr(offsets, np.int64), arr(finish, np.float64), arr(arrival, np.float64), arr(rank, np.int32)
    v = np.zeros(max(T, 1), np.int64)
    c = np.zeros(max(T, 1), np.int64)
    lib().so_audit(T, _ptr(off), _ptr(fin), _ptr(av), _ptr(rk), v.ctypes.data, c.ctypes.data)
    return v[:T], c[:T]
