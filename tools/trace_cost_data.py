"""Dev tool: per-trace GPU duration (libss_ttime.so) or per-trace stats (the
product library) for config-B seeds 0..T-1, saved to gpurun_out/ for offline
analysis of what predicts a trace's cost. Usage: trace_cost_data.py dur|stats T"""
import os, sys
mode, T = sys.argv[1], int(sys.argv[2])
if mode == "dur":
    os.environ["SS_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2506_12204_b200", "_lib",
                                             "libss_ttime.so")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import bench
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
wl = bench.WORKLOADS["B"]
prm = make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST)
batch = bench.native_batch("B", wl, np.arange(T), pinned=False)
dbatch = native.DeviceBatch(batch, "cuda")
douts = native.DeviceOutputs(batch.n_requests, T, "cuda", with_state=False)
ws = native.Workspace(prm, T, batch.n_requests, "cuda")
native.run_device(prm, dbatch, douts, ws)
native.run_device(prm, dbatch, douts, ws)
torch.cuda.synchronize()
st = douts.t["stats"].cpu().numpy().view(A.stats_dtype())
np.save(f"gpurun_out/trace_{mode}_{T}.npy", st)
print(mode, T, "saved")
