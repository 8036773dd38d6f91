"""Dev tool: wall time of the pipelined host call vs its kernel span (config B)."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import bench
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
wl = bench.WORKLOADS["B"]
batch, T = bench.build_batch(wl, 0, None, pinned=True)
prm = lambda: make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST)
for i in range(5):
    t0 = time.perf_counter()
    res = native.run_host(prm(), batch)
    t1 = time.perf_counter()
    print(f"wall {1e3 * (t1 - t0):.2f} ms (incl. Python output allocation), kernel span {res.kernel_ms:.2f} ms")
