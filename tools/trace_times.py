"""Dev tool: per-trace start and duration on the GPU (libss_ttime.so, built with
-DSS_DEBUG_TRACE_TIME: %globaltimer at trace start in sum_pool, duration in _pad).
Usage: trace_times.py <workload> [traces]"""
import os, sys
os.environ["SS_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2506_12204_b200", "_lib", "libss_ttime.so")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import bench
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
W = sys.argv[1]
wl = bench.WORKLOADS[W]
T = int(sys.argv[2]) if len(sys.argv) > 2 else wl["traces"]
batch = bench.native_batch(W, wl, np.arange(T), pinned=False)
prm = make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST)
import torch
dbatch = native.DeviceBatch(batch, "cuda")
douts = native.DeviceOutputs(batch.n_requests, T, "cuda", with_state=False)
ws = native.Workspace(prm, T, batch.n_requests, "cuda")
native.run_device(prm, dbatch, douts, ws)  # warm-up
kms = native.run_device(prm, dbatch, douts, ws, time_kernel=True)
torch.cuda.synchronize()
st = douts.t["stats"].cpu().numpy().view(A.stats_dtype())

class _R:
    kernel_ms = kms
res = _R()
t0 = st["sum_pool"].astype(np.int64)
dur = st["_pad"].astype(np.int64) / 1e6
start = (t0 - t0.min()) / 1e6
end = start + dur
rounds = st["rounds"].astype(np.int64)
print(f"{W}: {T} traces, kernel {res.kernel_ms:.2f} ms, makespan {end.max():.2f} ms")
print(f"  duration ms: mean {dur.mean():.2f} min {dur.min():.2f} p50 {np.median(dur):.2f} p99 {np.percentile(dur, 99):.2f} max {dur.max():.2f}")
print(f"  ns per round: mean {1e6 * dur.sum() / rounds.sum():.1f}; corr(duration, rounds) {np.corrcoef(dur, rounds)[0, 1]:.3f}")
first = start < 0.05
print(f"  first wave: {first.sum()} traces, duration mean {dur[first].mean():.2f}, max {dur[first].max():.2f}; later: {(~first).sum()} traces, mean {dur[~first].mean() if (~first).any() else 0:.2f}")
for q in (0.0, 0.25, 0.5, 0.75, 1.0):
    tq = q * end.max()
    print(f"  t={tq:6.2f} ms: {int(((start <= tq) & (end > tq)).sum())} traces running")
sm = st["sum_victims"].astype(np.int64)
print(f"  SMs used {len(np.unique(sm))}, traces per SM min {np.bincount(sm).min() if len(sm) else 0} max {np.bincount(sm).max()}")
for die, sel in (("SM < 74", sm < 74), ("SM >= 74", sm >= 74)):
    if sel.any():
        print(f"  {die}: {sel.sum()} traces, start min {start[sel].min():.2f} max {start[sel].max():.2f}, end max {end[sel].max():.2f}, "
              f"busy {dur[sel].sum() / (end[sel].max() - start[sel].min()):.0f} traces in flight on average")
hist, edges = np.histogram(start, bins=12)
print("  start-time histogram:", list(hist), "edges ms", [round(e, 2) for e in edges])
