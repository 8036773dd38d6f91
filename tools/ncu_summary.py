"""Summarise an ncu report into profiles/: key metrics, stall mix, hot lines."""
import csv, io, json, subprocess, sys

rep, out_json = sys.argv[1], sys.argv[2]
decisions = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
summary = {k: {"value": d.get(k), "unit": u.get(k)} for k in keys}
stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for h, v in d.items()
          if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and v not in ("", "n/a")}
tot = sum(stalls.values()) or 1.0
summary["stall_mix_pct"] = {k: round(100 * v / tot, 2) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v}
def mb(x):
    return float(x) * (1e6 if u.get("dram__bytes_read.sum", "").startswith("M") else 1e9 if u.get("dram__bytes_read.sum", "").startswith("G") else 1)
rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
if rd and wr:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    summary["dram_bytes_per_launch"] = float(rd) * scale[u["dram__bytes_read.sum"]] + float(wr) * scale[u["dram__bytes_write.sum"]]
if decisions:
    summary["warp_instructions_per_decision"] = float(d["smsp__inst_executed.sum"]) / decisions
json.dump(summary, open(out_json, "w"), indent=1)
print(json.dumps(summary, indent=1))
