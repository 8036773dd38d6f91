"""Bulk trace preparation through the native generator (``csrc/ss_tracegen.cpp``).

``generate_batch`` returns the same ``TraceBatch`` that
``soa.prepare_trace(workload.generate(spec), cfg)`` builds per seed, for
thousands of seeds at a time on all host cores (the Python path costs
~13 ms per 1k-request trace; config E has 65,536 of them)."""

from __future__ import annotations

import ctypes as C
import os
from typing import Sequence

import numpy as np

from .predictors import ErrorModel, PredictorConfig, Strategy
from .soa import TraceBatch
from .workload import WorkloadSpec


class ss_gen_spec(C.Structure):
    _fields_ = [("total_requests", C.c_int64), ("gap_s", C.c_double), ("concurrent", C.c_int32),
                ("concurrent_fixed", C.c_int32), ("levels", C.c_int32), ("buckets", C.c_int32),
                ("urgency_weights", C.c_void_p), ("prompt_lo", C.c_int64), ("prompt_hi", C.c_int64),
                ("out_lo", C.c_int64), ("out_hi", C.c_int64), ("max_output_len", C.c_int64),
                ("bucket_reps", C.c_void_p), ("latency_s", C.c_double), ("pred_batch", C.c_int32),
                ("full_batching", C.c_int32), ("urgency_error", C.c_double), ("length_error", C.c_double),
                ("urgency_disp", C.c_int64), ("length_disp", C.c_int64)]


class ss_gen_out(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg",
                                          "true_urg", "tie", "ids", "record_pos")]


def _lib():
    from .native import lib

    L = lib()
    if not getattr(L, "_gen_typed", False):
        L.ss_generate_traces.restype = C.c_int
        L.ss_generate_traces.argtypes = [C.POINTER(ss_gen_spec), C.c_int64, C.c_void_p, C.c_void_p,
                                         C.POINTER(ss_gen_out), C.c_int]
        L._gen_typed = True
    return L


def _gen_spec(spec: WorkloadSpec, predictor: PredictorConfig):
    """ss_gen_spec for ``spec`` + ``predictor``; returns (spec, keep-alive arrays)."""
    # representative length of every bucket index (workload.py:48-60)
    width = spec.max_output_len / spec.buckets
    reps = np.array([int(round((i + 0.5) * width)) for i in range(spec.buckets)], np.uint32)
    weights = None
    if spec.urgency_weights:
        weights = np.ascontiguousarray(np.asarray(spec.urgency_weights, np.float64))
    s = ss_gen_spec()
    s.total_requests = int(spec.total_requests)
    s.gap_s = spec.gap_s
    s.concurrent = spec.concurrent
    s.concurrent_fixed = 1 if spec.concurrent_mode == "fixed" else 0
    s.levels = spec.levels
    s.buckets = spec.buckets
    s.urgency_weights = weights.ctypes.data if weights is not None else None
    s.prompt_lo, s.prompt_hi = spec.prompt_len_range
    s.out_lo, s.out_hi = spec.output_len_range
    s.max_output_len = spec.max_output_len
    s.bucket_reps = reps.ctypes.data
    s.latency_s = predictor.latency_s
    s.pred_batch = predictor.batch_size
    s.full_batching = 1 if predictor.strategy is Strategy.FULL_BATCHING else 0
    s.urgency_error = predictor.urgency_error
    s.length_error = predictor.length_error
    s.urgency_disp = ErrorModel(predictor.urgency_error, spec.levels).displacement
    s.length_disp = ErrorModel(predictor.length_error, spec.max_output_len).displacement
    return s, (reps, weights)


def _typed(L, name, argtypes):
    f = getattr(L, name)
    if not getattr(f, "_ss_typed", False):
        f.restype = C.c_int
        f.argtypes = argtypes
        f._ss_typed = True
    return f


def native_arrivals(spec: WorkloadSpec):
    """workload.generate's draws for one spec (ss_generate_arrivals): arrival,
    prompt, true output and true urgency arrays in generation order."""
    n = int(spec.total_requests)
    s, keep = _gen_spec(spec, PredictorConfig())
    out = (np.empty(n, np.float64), np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.uint8))
    f = _typed(_lib(), "ss_generate_arrivals", [C.POINTER(ss_gen_spec), C.c_int64] + [C.c_void_p] * 4)
    if f(C.byref(s), int(spec.seed), *[a.ctypes.data if n else None for a in out]):
        raise ValueError("invalid workload spec for the native generator")
    return out


def native_predict(rng, what: int, levels: int, buckets: int, max_output_len: int, urgency_error: float = 0.0,
                   length_error: float = 0.0, latency_s: float = 0.0, pred_batch: int = 64,
                   full_batching: bool = False, arrival=None, true_out=None, true_urg=None, n: int = 0):
    """The predictor draws of ss_predict, continuing (and advancing) the
    CPython ``random.Random`` ``rng``: returns (pred_urg, pred_bucket, ready)."""
    version, words, gauss = rng.getstate()
    state = np.array(words, dtype=np.uint32)
    s = ss_gen_spec()
    s.levels, s.buckets, s.max_output_len = int(levels), int(buckets), int(max_output_len)
    s.urgency_error, s.length_error = float(urgency_error), float(length_error)
    s.urgency_disp = ErrorModel(urgency_error, levels).displacement if what & 1 else 1
    s.length_disp = ErrorModel(length_error, max_output_len).displacement if what & 2 else 1
    s.latency_s, s.pred_batch, s.full_batching = float(latency_s), int(pred_batch), 1 if full_batching else 0
    arr = lambda x, dt: np.ascontiguousarray(np.asarray(x, dt)) if x is not None else None
    a, o, u = arr(arrival, np.float64), arr(true_out, np.uint32), arr(true_urg, np.uint8)
    pu, pb, rd = np.zeros(n, np.uint8), np.zeros(n, np.uint32), np.zeros(n, np.float64)
    ptr = lambda x: x.ctypes.data if x is not None and x.size else None
    f = _typed(_lib(), "ss_predict", [C.POINTER(ss_gen_spec), C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p])
    if f(C.byref(s), n, ptr(a), ptr(o), ptr(u), int(what), state.ctypes.data, ptr(pu), ptr(pb), ptr(rd)):
        raise ValueError("invalid predictor arguments")
    rng.setstate((version, tuple(int(w) for w in state), gauss))
    return pu, pb, rd


def generate_batch_device(spec: WorkloadSpec, seeds: Sequence[int], predictor: PredictorConfig = PredictorConfig(),
                          pred_seeds: Sequence[int] = None, device="cuda"):
    """``generate_batch`` on the GPU (``ss_generate_traces_device``, one thread
    per trace): returns a ``native.DeviceBatch`` whose inputs never leave
    HBM, identical to ``DeviceBatch(generate_batch(...))``."""
    import torch

    from .native import DeviceBatch, NativeUnavailable

    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
    pseeds = seeds if pred_seeds is None else np.ascontiguousarray(np.asarray(pred_seeds, dtype=np.int64))
    T, N = len(seeds), int(spec.total_requests)
    s, keep = _gen_spec(spec, predictor)
    db = DeviceBatch.allocate(T, N, device, with_ids=True)
    t = db.t
    o = ss_gen_out(*[t[k].data_ptr() if t[k].numel() else None for k in
                     ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie",
                      "ids", "record_pos")])
    L = _lib()
    if not getattr(L, "_gen_dev_typed", False):
        L.ss_generate_traces_device.restype = C.c_int
        L.ss_generate_traces_device.argtypes = [C.POINTER(ss_gen_spec), C.c_int64, C.c_void_p, C.c_void_p,
                                                C.POINTER(ss_gen_out), C.c_void_p]
        L._gen_dev_typed = True
    rc = L.ss_generate_traces_device(C.byref(s), T, seeds.ctypes.data, pseeds.ctypes.data, C.byref(o),
                                     C.c_void_p(torch.cuda.current_stream(device).cuda_stream))
    if rc == 1:
        raise ValueError("invalid workload spec for the native generator")
    if rc == 2:
        raise NativeUnavailable("CUDA error in ss_generate_traces_device")
    if rc == 3:
        raise RuntimeError("prediction-ready order differs from generation order")
    return db


def generate_batch(spec: WorkloadSpec, seeds: Sequence[int], predictor: PredictorConfig = PredictorConfig(),
                   pred_seeds: Sequence[int] = None, threads: int = 0, pinned: bool = False) -> TraceBatch:
    """Traces for ``seeds`` (workload seeds); ``pred_seeds`` default to the same
    values (``run_scenario`` uses ``cfg.seed`` for both)."""
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
    pseeds = seeds if pred_seeds is None else np.ascontiguousarray(np.asarray(pred_seeds, dtype=np.int64))
    T, N = len(seeds), int(spec.total_requests)
    n = T * N
    s, keep = _gen_spec(spec, predictor)

    def buf(dt):
        if pinned:
            import torch

            tdt = {np.float64: torch.float64, np.uint32: torch.int32, np.uint8: torch.uint8,
                   np.int64: torch.int64}[dt]
            return torch.empty(max(n, 1), dtype=tdt, pin_memory=True).numpy().view(dt)[:n]
        return np.empty(n, dt)

    arrs = dict(ready=buf(np.float64), arrival=buf(np.float64), prompt=buf(np.uint32), true_out=buf(np.uint32),
                pred_len=buf(np.uint32), pred_urg=buf(np.uint8), true_urg=buf(np.uint8), tie=buf(np.uint32),
                ids=np.empty(n, np.int64), record_pos=np.empty(n, np.int64))
    o = ss_gen_out(*[arrs[k].ctypes.data if n else None for k in
                     ("ready", "arrival", "prompt", "true_out", "pred_len", "pred_urg", "true_urg", "tie",
                      "ids", "record_pos")])
    rc = _lib().ss_generate_traces(C.byref(s), T, seeds.ctypes.data, pseeds.ctypes.data, C.byref(o),
                                   int(threads or os.cpu_count() or 1))
    if rc:
        raise ValueError("invalid workload spec for the native generator")
    offsets = np.arange(T + 1, dtype=np.int64) * N
    return TraceBatch(offsets=offsets, **arrs)
