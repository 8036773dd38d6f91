"""Dev tool: per-trace warp-cycles by kernel section (libss_dbgtime.so,
-DSS_DEBUG_TIMING): which sections explain the spread of trace durations.
Usage: trace_sections.py [traces]"""
import ctypes as C, os, sys
os.environ["SS_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2506_12204_b200", "_lib", "libss_dbgtime.so")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import bench
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
wl = bench.WORKLOADS["B"]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
batch = bench.native_batch("B", wl, np.arange(T), pinned=False)
prm = make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST)
lib = native.lib()
dbatch = native.DeviceBatch(batch, "cuda")
douts = native.DeviceOutputs(batch.n_requests, T, "cuda", with_state=False)
ws = native.Workspace(prm, T, batch.n_requests, "cuda")
native.run_device(prm, dbatch, douts, ws)  # one launch: trace indices are global
buf = (C.c_ulonglong * (32 * T))()
lib.ss_debug_trace_cycles(buf, T)
v = np.frombuffer(buf, dtype=np.uint64).reshape(T, 32).astype(np.float64)
names = ["init/admission/top", "fast per-round body", "chunk", "g: composition", "outputs", "stretch entry", "stretch vote",
         "stretch order", "g: KV admission", "g: batch duration", "g: progress", "g: record", "g: ongoing rebuild",
         "g: queue rebuild", "g: evict_one calls", "refill"]
tot = v[:, :16].sum(1)
print(f"{T} traces: cycles per trace mean {tot.mean():.3g} std {tot.std():.3g} min {tot.min():.3g} max {tot.max():.3g}")
for i, n in enumerate(names):
    x = v[:, i]
    if x.sum() == 0:
        continue
    cov = np.cov(x, tot)[0, 1] / tot.var()
    print(f"  {n:22s} mean {x.mean():10.3g}  std {x.std():10.3g}  share of variance {cov:6.3f}  corr {np.corrcoef(x, tot)[0, 1]:.3f}")
c = v[:, 16:]
print("  counts mean: chunks %.0f, chunk rounds %.0f, per-round %.0f, general %.0f, refills %.1f" % tuple(c[:, [0, 1, 2, 3, 5]].mean(0)))
for j, n in ((0, "chunks"), (2, "per-round"), (3, "general"), (5, "refills")):
    print(f"  corr(cycles, {n}) {np.corrcoef(c[:, j], tot)[0, 1]:.3f}")
np.save("gpurun_out/trace_sections.npy", v)
