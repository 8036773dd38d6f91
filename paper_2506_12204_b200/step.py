"""ctypes callers of the per-step C-ABI (``ss_select_batch``, ``ss_evict``;
``include/semsched_b200.h``, ``csrc/ss_step.cu``).

Keys cross the boundary as four float64 per tuple (``ss_key4``): the
reference's key tuples hold ints (rank, id) and floats (f_t, arrival); their
float64 images compare exactly like Python compares the ints and floats
(|ints| < 2**53), and shorter tuples are padded with -inf so that a tuple's
prefix sorts first, as in Python.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import _abi as A
from .native import NativeUnavailable, SchedulerError, lib

SS_SELECT_TOP_B, SS_SELECT_STAGE_AWARE, SS_SELECT_PREEMPTIVE, SS_SELECT_FCFS = 0, 1, 2, 3


class ss_victim(C.Structure):
    _fields_ = [("index", C.c_int32), ("action", C.c_int32), ("decode_saved", C.c_int64),
                ("decode_discarded", C.c_int64), ("freed_slots", C.c_int64), ("prefilled", C.c_int64),
                ("kv_host", C.c_int64), ("f_t_before", C.c_double), ("f_t_after", C.c_double),
                ("_pad", C.c_int64)]


VICTIM_DTYPE = np.dtype([("index", "<i4"), ("action", "<i4"), ("decode_saved", "<i8"),
                         ("decode_discarded", "<i8"), ("freed_slots", "<i8"), ("prefilled", "<i8"),
                         ("kv_host", "<i8"), ("f_t_before", "<f8"), ("f_t_after", "<f8"), ("_pad", "<i8")])
assert VICTIM_DTYPE.itemsize == C.sizeof(ss_victim)

_bound = False


def _lib():
    global _bound
    L = lib()
    if not _bound:
        vp, i32p, i64p = C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64)
        L.ss_select_batch.restype = C.c_int
        L.ss_select_batch.argtypes = [vp, vp, vp, C.c_int64, vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                      vp, i32p, vp, i32p, i32p, i32p, vp]
        L.ss_evict.restype = C.c_int
        L.ss_evict.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                               C.POINTER(A.ss_profile), C.c_int32, C.c_int32, vp, i64p, vp, i64p, i32p, vp]
        L.ss_step_last_error.restype = C.c_char_p
        _bound = True
    return L


def _check(rc: int) -> None:
    if rc == A.SS_OK:
        return
    msg = _lib().ss_step_last_error().decode()
    if rc == A.SS_ERR_INVALID_ARG:
        raise ValueError(msg)
    if rc == A.SS_ERR_NO_DEVICE:
        raise NativeUnavailable(msg)
    raise SchedulerError(rc, msg)


def pack_keys(keys: Sequence[tuple]) -> np.ndarray:
    """Key tuples -> (n, 4) float64, padded with -inf."""
    out = np.full((len(keys), 4), -np.inf, np.float64)
    for i, k in enumerate(keys):
        if len(k) > 4:
            raise ValueError("keys longer than 4 components are not supported")
        out[i, :len(k)] = k
    return out


def _p(a: np.ndarray):
    return a.ctypes.data if a is not None and a.size else None


def select_batch(stored: np.ndarray, current, pool_decoding: np.ndarray, ongoing: np.ndarray,
                 ongoing_decoding: np.ndarray, b: int, mode: int):
    """-> (cand, merged, n_selected, kind). See ``ss_select_batch``."""
    L = _lib()
    n_pool, n_ong = len(stored), len(ongoing)
    stored = np.ascontiguousarray(stored, np.float64)
    cur = None if current is None else np.ascontiguousarray(current, np.float64)
    pd = np.ascontiguousarray(pool_decoding, np.uint8)
    on = np.ascontiguousarray(ongoing, np.float64).reshape(n_ong, 4)
    od = np.ascontiguousarray(ongoing_decoding, np.uint8)
    cand = np.zeros(32, np.int32)
    merged = np.zeros(64, np.int32)
    nc, nm, ns, kind = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    rc = L.ss_select_batch(_p(stored), _p(cur), _p(pd), n_pool, _p(on), _p(od), n_ong, int(b), int(mode),
                           cand.ctypes.data, C.byref(nc), merged.ctypes.data, C.byref(nm), C.byref(ns),
                           C.byref(kind), None)
    _check(rc)
    return cand[:nc.value].copy(), merged[:nm.value].copy(), ns.value, kind.value


def evict(ev_keys, prompt, prefilled, decoded, kv_device, pred_len, f_t, protected, demand: int, used: int,
          capacity: int, profile, dependency_rule: bool, select: bool):
    """-> (victims structured array, skipped indices, failed). See ``ss_evict``."""
    L = _lib()
    n = len(prompt)
    arr = lambda x, dt: np.ascontiguousarray(np.asarray(x), dt)
    keys = arr(ev_keys, np.float64).reshape(n, 4) if select else np.zeros((0, 4))
    pr, pf, de = arr(prompt, np.uint32), arr(prefilled, np.uint32), arr(decoded, np.uint32)
    kv, pl, ft = arr(kv_device, np.uint32), arr(pred_len, np.uint32), arr(f_t, np.float64)
    pt = arr(protected, np.uint8) if select else np.zeros(0, np.uint8)
    out = np.zeros(max(n, 1), VICTIM_DTYPE)
    sk = np.zeros(max(n, 1), np.int32)
    nv, ns, failed = C.c_int64(), C.c_int64(), C.c_int32()
    prof = A.ss_profile(profile.alpha1, profile.alpha2, profile.gamma1, profile.gamma2, profile.beta_load,
                        profile.beta_save)
    rc = L.ss_evict(_p(keys), _p(pr), _p(pf), _p(de), _p(kv), _p(pl), _p(ft), _p(pt), n, int(demand), int(used),
                    int(capacity), C.byref(prof), 1 if dependency_rule else 0, 1 if select else 0,
                    out.ctypes.data, C.byref(nv), sk.ctypes.data, C.byref(ns), C.byref(failed), None)
    _check(rc)
    return out[:nv.value].copy(), sk[:ns.value].copy(), bool(failed.value)
