"""Top source lines of an ncu report by stall samples and instructions
(ncu --page source --print-source=cuda,sass). Usage: ncu_lines.py rep [N]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
hdr = None
agg = defaultdict(lambda: [0, 0, defaultdict(int), ""])
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        f = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0] or not row[0].isdigit():
        continue
    d = dict(zip(hdr[2:], row[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ins = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    a = agg[(f, int(row[0]))]
    a[0] += s
    a[1] += ins
    a[3] = row[1][:90]
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "-"):
            a[2][k[6:]] += int(v)
tot_s = sum(a[0] for a in agg.values()) or 1
tot_i = sum(a[1] for a in agg.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for (f, ln), a in sorted(agg.items(), key=lambda x: -x[1][0])[:N]:
    top = ",".join(f"{k}:{v}" for k, v in sorted(a[2].items(), key=lambda x: -x[1])[:3])
    print(f"{100*a[0]/tot_s:5.1f}% {100*a[1]/tot_i:5.1f}%i {f}:{ln:<5d} {a[3]:<90s} {top}")
