"""Dev tool: warp-cycles per scheduler-kernel section (libss_dbgtime.so, built with
-DSS_DEBUG_TIMING) on a bench workload. Usage: section_timing.py <workload> [traces]"""
import ctypes as C, os, sys
os.environ["SS_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2506_12204_b200", "_lib", os.environ.get("SS_DBG_LIB", "libss_dbgtime.so"))
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
force = {"auto": 0, "chunked": A.SS_FLAG_FORCE_CHUNKED, "perround": A.SS_FLAG_FORCE_PERROUND}[os.environ.get("SS_BENCH_VARIANT", "auto")]
prm = make_params(get_profile(wl["profile"]), 16, wl["capacity"], levels=wl["levels"], flags=A.SS_FLAG_DIGEST | force)
lib = native.lib()
buf = (C.c_ulonglong * 32)()
native.run_host(prm, batch)  # warm-up
lib.ss_debug_cycles(buf)
res = native.run_host(prm, batch)
lib.ss_debug_cycles(buf)
v = list(buf)
tot = sum(v[:16]) or 1
names = ["init/admission/top", "fast per-round body", "chunk", "g: composition", "outputs", "stretch entry", "stretch vote", "stretch order",
         "g: KV admission", "g: batch duration", "g: progress", "g: record", "g: ongoing rebuild", "g: queue rebuild", "g: evict_one calls", "refill"]
rounds = int(res.stats["rounds"].sum())
print(f"{W}: {T} traces, {rounds} rounds, kernel {res.kernel_ms:.2f} ms")
for i, n in enumerate(names):
    print(f"  {n:20s} {100 * v[i] / tot:5.1f}%  {v[i] / max(rounds, 1):8.1f} warp-cycles/round")
c = v[16:]
print(f"  chunks {c[0]}, chunk rounds {c[1]} ({c[1] / max(c[0], 1):.1f}/chunk), per-round fast {c[2]}, general {c[3]}")
if c[5]: print(f"  refills {c[5]}, cycles per refill {v[15] / c[5]:.0f}")
if c[4]: print(f"  evict_one calls {c[4]}, cycles per call {v[14] / c[4]:.0f}")
if c[0]: print(f"  cycles/chunk {v[2] / c[0]:.0f}, per chunk round {v[2] / max(c[1], 1):.0f}, order screen settled {100 * c[6] / c[0]:.1f}% of chunks, exact loop {c[7] / c[0]:.2f} members per chunk")
if c[2]: print(f"  cycles per per-round fast round {v[1] / c[2]:.0f}")
print(f"  stretch entries with a queued decoding candidate below the full batch: {c[8]}")
print(f"  stretch vote exits: admission {c[9]}, p* queued {c[10]}, completion rounds {c[11]}; reorders {c[15]}")
if os.environ.get("SS_DEBUG_D"):
    print(f"  stretch entry refused (queued decoding candidate) {c[12]}; eviction breaks {c[13]}, of which before any round {c[14]}")
else:
    print(f"  chunk ends: at L (completion / 32) {c[12]}, admission {c[13]}, order / p* {c[14]}")
if c[3]: print(f"  cycles per general round (composition .. queue rebuild) {sum(v[i] for i in (3, 8, 9, 10, 11, 12, 13)) / c[3]:.0f}")
