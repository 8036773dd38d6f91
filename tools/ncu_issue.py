"""Issue-rate profile of the scheduler kernel for bench.py's roofline.

Run on the GPU box (under gpurun), one workload at a time:

    python tools/ncu_issue.py B [D E A ...]

For each workload it runs ``bench.py --workload W --steps 1 --warmup 0`` under
``ncu --clock-control none`` restricted to the scheduler launches of the
first run (the three variants ``sched_kernel<...>``; the unselected ones exit
at their first instruction) and writes ``gpurun_out/ncu_issue_<W>.json`` (committed as ``profiles/ncu_issue_<W>.json``):
warp instructions executed, DRAM bytes read+written and duration of the
selected (longest) variant, plus the decisions and traces of that launch, so
bench.py can divide the instruction count by its own live kernel time.
A number measured under ncu is never reported as a bench value.
"""

import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
           "smsp__warps_active.avg.per_cycle_active", "launch__registers_per_thread"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def profile(w: str) -> dict:
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    logf = os.path.join(REPO, "gpurun_out", f"ncu_issue_{w}.csv")
    cmd = ["ncu", "--clock-control", "none", "--metrics", ",".join(METRICS), "-k", "regex:sched_kernel", "-c", "3",
           "--csv", "--log-file", logf, sys.executable, "bench.py", "--workload", w, "--steps", "1", "--warmup", "1",
           "--no-e2e", "--no-cpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=REPO)
    line = next(json.loads(x) for x in out.stdout.splitlines() if x.startswith("{"))
    text = open(logf).read()
    rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))  # skip ==PROF== lines
    kern = {}
    for r in rows:
        k = kern.setdefault(r["ID"], {"kernel": r["Kernel Name"]})
        v = r["Metric Value"].replace(",", "")
        try:
            k[r["Metric Name"]] = float(v) * SCALE.get(r["Metric Unit"], 1.0)
        except ValueError:
            pass
    sel = max(kern.values(), key=lambda k: k.get("gpu__time_duration.sum", 0))
    res = {"workload": w, "kernel": sel["kernel"], "decisions": line["decisions_per_step"],
           "traces": line["config"]["traces_per_gpu"], "inst_executed": sel["smsp__inst_executed.sum"],
           "dram_bytes": sel["dram__bytes_read.sum"] + sel["dram__bytes_write.sum"],
           "duration_ms_under_ncu": 1e3 * sel["gpu__time_duration.sum"],
           "issue_active_pct": sel["smsp__issue_active.avg.pct_of_peak_sustained_active"],
           "sm_cycles_elapsed": sel["sm__cycles_elapsed.avg"],
           "warps_active_per_smsp": sel["smsp__warps_active.avg.per_cycle_active"],
           "registers": sel["launch__registers_per_thread"],
           "all_variants": [{"kernel": k["kernel"], "ms": 1e3 * k.get("gpu__time_duration.sum", 0)}
                            for k in kern.values()],
           "command": " ".join(cmd[:9] + ["<log>", "python"] + cmd[11:])}
    res["warp_instr_per_decision"] = res["inst_executed"] / res["decisions"]
    # gpurun merges gpurun_out/ back; copy the file to profiles/ to commit it
    with open(os.path.join(REPO, "gpurun_out", f"ncu_issue_{w}.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    return res


if __name__ == "__main__":
    for w in sys.argv[1:] or ["B"]:
        print(json.dumps(profile(w)))
