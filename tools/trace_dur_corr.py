"""Dev tool: is a trace's GPU duration intrinsic to the trace? Runs the same
traces in two orders (one wave) with libss_ttime.so and correlates per-trace
durations; also against per-trace features from the stats."""
import os, sys
os.environ["SS_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2506_12204_b200", "_lib", "libss_ttime.so")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import bench
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
wl = bench.WORKLOADS["B"]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
prm = make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST)


def run(seeds):
    batch = bench.native_batch("B", wl, seeds, pinned=False)
    dbatch = native.DeviceBatch(batch, "cuda")
    douts = native.DeviceOutputs(batch.n_requests, len(seeds), "cuda", with_state=False)
    ws = native.Workspace(prm, len(seeds), batch.n_requests, "cuda")
    native.run_device(prm, dbatch, douts, ws)
    kms = native.run_device(prm, dbatch, douts, ws, time_kernel=True)
    torch.cuda.synchronize()
    st = douts.t["stats"].cpu().numpy().view(A.stats_dtype())
    return st["_pad"].astype(np.float64) / 1e6, st, kms


seeds = np.arange(T)
d1, st, k1 = run(seeds)
d2r, _, k2 = run(seeds[::-1].copy())
d2 = d2r[::-1]
perm = np.random.default_rng(1).permutation(T)
d3p, _, k3 = run(seeds[perm])
d3 = np.empty(T); d3[perm] = d3p
print(f"kernels {k1:.2f} {k2:.2f} {k3:.2f} ms; corr(order, reversed) {np.corrcoef(d1, d2)[0, 1]:.3f}, corr(order, shuffled) {np.corrcoef(d1, d3)[0, 1]:.3f}")
feats = {k: st[k].astype(np.float64) for k in ("rounds", "sum_granted", "sum_pool", "completed", "mem_used_peak")}
dm = (d1 + d2 + d3) / 3
for k, v in feats.items():
    print(f"  corr(mean duration, {k}) {np.corrcoef(dm, v)[0, 1]:.3f}")
np.save("gpurun_out/trace_durations.npy", np.stack([d1, d2, d3]))
