"""Dev tool: GPU vs oracle digests over many traces of tight-memory and ample configs.
    python tools/parity_sweep.py <traces> [auto|chunked|perround]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np
from oracle_binding import run_oracle
from paper_2506_12204_b200 import _abi as A, native
from paper_2506_12204_b200.costs import get_profile
from paper_2506_12204_b200.dist import shard_seeds
from paper_2506_12204_b200.results import make_params
from paper_2506_12204_b200.scenarios import MIXED_PROFILE
from paper_2506_12204_b200.tracegen import generate_batch
from paper_2506_12204_b200.workload import WorkloadSpec

T = int(sys.argv[1])
VAR = {"auto": 0, "chunked": A.SS_FLAG_FORCE_CHUNKED, "perround": A.SS_FLAG_FORCE_PERROUND}[
    sys.argv[2] if len(sys.argv) > 2 else "auto"]
bad_total = 0
from paper_2506_12204_b200.predictors import PredictorConfig

ERR = PredictorConfig(length_error=0.5, urgency_error=0.1)
for prof_name, cap, levels, n, b, pred in (("a100_qwen7b", 2295, 3, 1000, 16, None), ("a5000_qwen7b", 2295, 3, 1000, 16, None),
                                           ("mixed", 2295, 3, 1000, 16, None), ("a100_qwen7b", 1200, 5, 800, 16, None),
                                           ("a100_qwen7b", 700, 4, 500, 16, None), ("a100_qwen7b", 10**9, 5, 1000, 16, None),
                                           ("a100_qwen7b", 10**9, 5, 1000, 32, None), ("a5000_qwen7b", 10**9, 3, 2000, 8, None),
                                           ("a100_qwen7b", 10**9, 5, 1000, 16, ERR), ("a100_qwen7b", 3000, 4, 800, 16, ERR)):
    prof = MIXED_PROFILE if prof_name == "mixed" else get_profile(prof_name)
    batch = generate_batch(WorkloadSpec(total_requests=n, levels=levels), shard_seeds(T, 0, seed0=17),
                           pred or PredictorConfig())
    p = lambda f=0: make_params(prof, b, cap, levels=levels, flags=A.SS_FLAG_DIGEST | f)
    g = native.run_host(p(VAR), batch)
    c = run_oracle(p(), batch, threads=os.cpu_count())
    ok = c.stats["status"] == 0
    bad = (g.stats["status"] != c.stats["status"]) | (g.stats["rounds"] != c.stats["rounds"]) | \
          (ok & (g.stats["digest"] != c.stats["digest"]))
    bad_total += int(bad.sum())
    print(f"{prof_name} cap {cap} levels {levels} n {n} b {b}{' predictor errors' if pred else ''}: {T} traces, {int((~ok).sum())} ref errors, "
          f"anomalies {int(c.stats['anomalies'].sum())}, mismatches {int(bad.sum())} {list(np.nonzero(bad)[0][:8])}")
print("TOTAL MISMATCHES", bad_total)
