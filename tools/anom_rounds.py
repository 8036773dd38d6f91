"""Dev tool: general-path rounds with and without the stale-entry flag
(libss_dbganom.so, -DSS_DEBUG_ANOM) on a bench workload sample."""
import os, sys
os.environ["SS_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2506_12204_b200", "_lib", "libss_dbganom.so")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
import bench
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.results import make_params
W, T = sys.argv[1], int(sys.argv[2])
wl = bench.WORKLOADS[W]
batch, T = bench.build_batch(wl, 0, T, pinned=False)
res = native.run_host(make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST), batch)
anom = res.stats["_pad"].astype(np.int64)
print(f"{W}: rounds {res.stats['rounds'].sum()}, rounds run with the stale-entry flag {anom.sum()}; "
      f"traces with such rounds {(anom > 0).sum()}/{T}")
