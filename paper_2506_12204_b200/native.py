"""Loader and callers of the in-tree CUDA extension (C-ABI via ctypes).

There is no CPU fallback: if the shared library or a CUDA device is missing
every entry point raises ``NativeUnavailable``. Device memory comes from
PyTorch (``torch.empty(..., device="cuda")``) purely as an allocator and
stream provider; the C-ABI sees raw pointers only.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _abi as A
from .results import RunResult, alloc_host_outputs, collect, log_capacity_words

LIB_PATH = os.environ.get("SS_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                         "libsemsched_b200.so")
_lib = None


class NativeUnavailable(RuntimeError):
    """The CUDA extension or the device is missing (no fallback exists)."""


class SchedulerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"semsched_b200 error {code}: {msg}")
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} not built; run `python -m paper_2506_12204_b200.build` "
                "(or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        L.ss_last_error.restype = C.c_char_p
        L.ss_device_info.argtypes = [C.POINTER(C.c_int)] * 4
        L.ss_workspace_bytes.argtypes = [C.POINTER(A.ss_params), C.c_int32, C.c_int64, C.POINTER(C.c_size_t)]
        L.ss_kernel_config.argtypes = [C.POINTER(A.ss_params), C.c_int32, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ss_run_traces.argtypes = [C.POINTER(A.ss_params), C.POINTER(A.ss_trace_batch),
                                    C.POINTER(A.ss_outputs), C.c_void_p, C.c_size_t, C.c_void_p,
                                    C.POINTER(C.c_float)]
        L.ss_run_traces_host.argtypes = [C.POINTER(A.ss_params), C.POINTER(A.ss_trace_batch),
                                         C.POINTER(A.ss_outputs), C.c_void_p, C.POINTER(C.c_float)]
        L.ss_last_timings.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float)]
        for f in ("ss_device_info", "ss_workspace_bytes", "ss_kernel_config", "ss_run_traces",
                  "ss_run_traces_host", "ss_last_timings"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


EXPORTED = ("ss_last_error", "ss_device_info", "ss_workspace_bytes", "ss_run_traces",
            "ss_run_traces_host", "ss_kernel_config", "ss_last_timings", "ss_select_batch", "ss_evict",
            "ss_step_last_error", "ss_audit_host", "ss_audit_last_error",
            "ss_audit_last_kernel_ms", "ss_generate_traces", "ss_generate_traces_device")


# kernels one ss_run_traces call launches (ss_prepass.cu + the scheduler +
# ss_epilogue.cu): detect, eoff scan, init, bulk keys, histogram, plan,
# 16 x (count, scan, scatter), final copy, sched_kernel, the end-of-trace
# kernels. The bulk stages exit at once when no trace admits a bulk group.
def launches_per_run(params=None, max_trace_len=None) -> int:
    bulk = params is None or params.bulk_min >= 0
    if params is not None and max_trace_len is not None:
        bulk = _bulk_possible(params, max_trace_len)
    # detect, scan, init, select (+ the bulk sort) + the scheduler: semantic runs
    # launch the three variants (chunked without eviction, chunked, per-round); the
    # unselected ones exit at once
    sched = 3 if params is None or params.policy == A.SS_POLICY["semantic"] else 1
    # the short-trace epilogue (outputs + exact sums, one warp per trace) always runs;
    # the two grid-wide long-trace kernels only when a trace is long enough
    epi = 1 + (2 if params is None or _epilogue_possible(params, max_trace_len) else 0)
    return 4 + (3 + 16 * 3 + 1 if bulk else 0) + sched + epi


def _epilogue_threshold(params) -> int:
    return A.SS_EPILOGUE_MIN_DEFAULT if params.epilogue_min == 0 else max(int(params.epilogue_min), 0)


def _epilogue_possible(params, max_trace_len=None) -> bool:
    """Whether any trace is long enough for the grid-wide end of trace."""
    thr = _epilogue_threshold(params)
    return thr > 0 and (max_trace_len is None or max_trace_len >= thr)


def _bulk_possible(params, max_trace_len: int) -> bool:
    """Whether any trace could admit a bulk group (ss_params.bulk_min)."""
    if params.bulk_min < 0:
        return False
    thr = params.bulk_min if params.bulk_min > 0 else A.SS_BULK_MIN_DEFAULT
    return max_trace_len >= thr


def _with_bulk(params, max_trace_len):
    """A copy of params with the bulk-sort stage and the grid-wide end of trace
    disabled when no trace is long enough to need them (saves their empty
    launches; results are identical)."""
    if max_trace_len is None:
        return params
    no_bulk = not _bulk_possible(params, max_trace_len) and params.bulk_min >= 0
    no_epi = not _epilogue_possible(params, max_trace_len) and params.epilogue_min >= 0
    if not (no_bulk or no_epi):
        return params
    q = A.ss_params()
    C.pointer(q)[0] = params
    if no_bulk:
        q.bulk_min = -1
    if no_epi:
        q.epilogue_min = -1
    return q


def last_timings():
    """(prepass_ms, kernel_ms) of this thread's last timed ss_run_traces."""
    pm, km = C.c_float(), C.c_float()
    lib().ss_last_timings(C.byref(pm), C.byref(km))
    return pm.value, km.value


def last_error() -> str:
    return lib().ss_last_error().decode()


def device_info():
    d, sms, ma, mi = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    rc = lib().ss_device_info(C.byref(d), C.byref(sms), C.byref(ma), C.byref(mi))
    if rc == A.SS_ERR_NO_DEVICE:
        raise NativeUnavailable("no CUDA device: the scheduler has no CPU path")
    if rc:
        raise SchedulerError(rc, last_error())
    return {"device": d.value, "sm_count": sms.value, "cc": (ma.value, mi.value)}


def kernel_config(params, n_traces: int):
    b, w, s = C.c_int(), C.c_int(), C.c_int()
    rc = lib().ss_kernel_config(C.byref(params), int(n_traces), C.byref(b), C.byref(w), C.byref(s))
    if rc:
        raise SchedulerError(rc, last_error())
    return {"blocks": b.value, "warps_per_block": w.value, "smem_per_block": s.value}


def _p(a) -> Optional[int]:
    return a.ctypes.data if a is not None and a.size else None


def host_batch(batch) -> A.ss_trace_batch:
    hb = A.ss_trace_batch()
    hb.n_traces = batch.n_traces
    hb.n_requests = batch.n_requests
    hb.trace_offsets = _p(batch.offsets)
    for f, name in (("ready", "ready_time"), ("arrival", "arrival_time"), ("prompt", "prompt_len"),
                    ("true_out", "true_output_len"), ("pred_len", "pred_len"),
                    ("pred_urg", "pred_urgency"), ("true_urg", "true_urgency"), ("tie", "tie_rank")):
        setattr(hb, name, _p(getattr(batch, f)))
    return hb


def _check(rc: int, allow_trace_failed: bool):
    if rc == A.SS_OK or (rc == A.SS_ERR_TRACE_FAILED and allow_trace_failed):
        return
    if rc == A.SS_ERR_NO_DEVICE:
        raise NativeUnavailable(last_error())
    if rc == A.SS_ERR_INVALID_ARG:
        raise ValueError(last_error())
    raise SchedulerError(rc, last_error())


def run_host(params, batch, want_log: bool = False, stream: int = 0, allow_trace_failed: bool = True,
             log_scale: int = 1) -> RunResult:
    """Host buffers in, host buffers out (the plugin call). Copies are inside."""
    batch.validate()
    outs = alloc_host_outputs(batch.n_requests, batch.n_traces)
    o = A.ss_outputs()
    o.req = A.ss_request_out(_p(outs["first_scheduled"]), _p(outs["finish_time"]), _p(outs["generated"]),
                             _p(outs["evictions"]), _p(outs["f_t"]), _p(outs["state"]))
    o.stats = _p(outs["stats"])
    o.unservable_slots = _p(outs["unservable"])
    log = log_off = None
    if want_log:
        params.flags |= A.SS_FLAG_ROUND_LOG
        log_off = log_capacity_words(batch, params, log_scale)
        log = np.zeros(max(int(log_off[-1]), 1), np.uint32)
        o.round_log = _p(log)
        o.log_offsets = _p(log_off)
    else:
        params.flags &= ~A.SS_FLAG_ROUND_LOG
    hb = host_batch(batch)
    ms = C.c_float(0.0)
    rc = lib().ss_run_traces_host(C.byref(params), C.byref(hb), C.byref(o), C.c_void_p(stream), C.byref(ms))
    _check(rc, allow_trace_failed)
    res = collect(batch, outs, log, log_off, kernel_ms=ms.value)
    # a trace whose log outgrew the first guess runs again with 4x the space; a trace the
    # reference would never finish (livelock) overflows any log, so the retries are bounded
    if want_log and (res.stats["status"] == A.SS_TRACE_LOG_OVERFLOW).any() and log_scale < 64:
        return run_host(params, batch, want_log, stream, allow_trace_failed, log_scale * 4)
    return res


class DeviceBatch:
    """A TraceBatch resident in HBM (torch tensors as the allocator)."""

    FIELDS = (("ready", "ready_time"), ("arrival", "arrival_time"), ("prompt", "prompt_len"),
              ("true_out", "true_output_len"), ("pred_len", "pred_len"), ("pred_urg", "pred_urgency"),
              ("true_urg", "true_urgency"), ("tie", "tie_rank"))

    def __init__(self, batch, device="cuda"):
        import torch

        self.batch = batch
        self.n_traces = batch.n_traces
        self.n_requests = batch.n_requests
        self.max_trace_len = int(np.diff(batch.offsets).max()) if batch.n_traces else 0
        self.t = {"offsets": torch.from_numpy(np.ascontiguousarray(batch.offsets)).to(device)}
        for f, _ in self.FIELDS:
            self.t[f] = torch.from_numpy(np.ascontiguousarray(getattr(batch, f))).to(device)

    @classmethod
    def allocate(cls, n_traces: int, per_trace: int, device="cuda", with_ids: bool = False):
        """Uninitialised inputs for ``n_traces`` equal-length traces (filled
        on the device, e.g. by ``tracegen.generate_batch_device``)."""
        import torch

        self = cls.__new__(cls)
        self.batch = None
        self.n_traces = n_traces
        self.max_trace_len = per_trace
        n = n_traces * per_trace
        self.n_requests = n
        dts = {"ready": torch.float64, "arrival": torch.float64, "prompt": torch.int32, "true_out": torch.int32,
               "pred_len": torch.int32, "pred_urg": torch.uint8, "true_urg": torch.uint8, "tie": torch.int32}
        self.t = {"offsets": torch.arange(n_traces + 1, dtype=torch.int64, device=device) * per_trace}
        for f, dt in dts.items():
            self.t[f] = torch.empty(max(n, 1), dtype=dt, device=device)
        for f in ("ids", "record_pos"):
            self.t[f] = torch.empty(max(n, 1) if with_ids else 0, dtype=torch.int64, device=device)
        return self

    def struct(self) -> A.ss_trace_batch:
        db = A.ss_trace_batch()
        db.n_traces = self.n_traces
        db.n_requests = self.n_requests
        db.trace_offsets = self.t["offsets"].data_ptr()
        for f, name in self.FIELDS:
            setattr(db, name, self.t[f].data_ptr() if self.t[f].numel() else None)
        return db


class DeviceOutputs:
    def __init__(self, n_requests: int, n_traces: int, device="cuda", with_state: bool = True):
        import torch

        n = max(n_requests, 1)
        self.t = {
            "first_scheduled": torch.empty(n, dtype=torch.float64, device=device),
            "finish_time": torch.empty(n, dtype=torch.float64, device=device),
            "generated": torch.empty(n, dtype=torch.int32, device=device),
            "evictions": torch.empty(n, dtype=torch.int32, device=device),
            "f_t": torch.empty(n, dtype=torch.float64, device=device) if with_state else None,
            "state": torch.empty(n, dtype=torch.int32, device=device) if with_state else None,
            "stats": torch.empty(n_traces * C.sizeof(A.ss_trace_stats), dtype=torch.uint8, device=device),
            "unservable": torch.empty(n, dtype=torch.int32, device=device),
        }

    def struct(self) -> A.ss_outputs:
        o = A.ss_outputs()
        g = lambda k: self.t[k].data_ptr() if self.t[k] is not None else None
        o.req = A.ss_request_out(g("first_scheduled"), g("finish_time"), g("generated"), g("evictions"),
                                 g("f_t"), g("state"))
        o.stats = g("stats")
        o.unservable_slots = g("unservable")
        return o

    def stats_numpy(self) -> np.ndarray:
        return self.t["stats"].cpu().numpy().view(A.stats_dtype())


class Workspace:
    def __init__(self, params, n_traces: int, n_requests: int, device="cuda"):
        import torch

        nb = C.c_size_t()
        rc = lib().ss_workspace_bytes(C.byref(params), int(n_traces), int(n_requests), C.byref(nb))
        _check(rc, False)
        self.nbytes = nb.value
        self.t = torch.empty(self.nbytes, dtype=torch.uint8, device=device)


def run_device(params, dbatch: DeviceBatch, douts: DeviceOutputs, ws: Workspace, stream=None,
               time_kernel: bool = False) -> Optional[float]:
    """Inputs/outputs already in HBM; launches on `stream` (torch stream or None)."""
    import torch

    params.flags &= ~A.SS_FLAG_ROUND_LOG
    params = _with_bulk(params, getattr(dbatch, "max_trace_len", None))
    s = stream if stream is not None else torch.cuda.current_stream()
    ms = C.c_float(0.0)
    db, do = dbatch.struct(), douts.struct()
    rc = lib().ss_run_traces(C.byref(params), C.byref(db), C.byref(do), C.c_void_p(ws.t.data_ptr()),
                             C.c_size_t(ws.nbytes), C.c_void_p(s.cuda_stream),
                             C.byref(ms) if time_kernel else None)
    _check(rc, False)
    return ms.value if time_kernel else None
