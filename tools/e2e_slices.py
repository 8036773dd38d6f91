"""Dev tool: host-entry (e2e) time per slice count (SS_HOST_SLICES); W=<workload> (default B)."""
import ctypes as C, os, subprocess, sys, json
W = os.environ.get("W", "B")
for sl in sys.argv[1:] or ["1", "2", "4", "6", "8"]:
    env = dict(os.environ, SS_HOST_SLICES=sl)
    out = subprocess.run([sys.executable, "bench.py", "--workload", W, "--steps", "3", "--warmup", "3", "--no-cpu"],
                         capture_output=True, text=True, env=env).stdout
    d = json.loads([l for l in out.splitlines() if l.startswith("{")][-1])
    print(f"slices {sl}: device {d['ms_per_step']:.2f} ms, e2e {d['e2e']['ms_per_step']:.2f} ms", flush=True)
