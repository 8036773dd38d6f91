"""Stall samples of an ncu report grouped by the scheduler kernel's sections
('// ----' markers and function starts in ss_kernel.cu); inlined helpers from
other files are attributed to the section whose code called them only when
ncu reports the call site, so they are listed on their own."""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
src = open(sys.argv[2] if len(sys.argv) > 2 else "paper_2506_12204_b200/csrc/ss_kernel.cu").read().split("\n")
secs = [(i + 1, l.strip()[:72]) for i, l in enumerate(src)
        if "// ----" in l or l.startswith("__device__") or l.startswith("template") or "SS_EVICT_INLINE bool" in l]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
hdr = None
agg = defaultdict(int)
ins = defaultdict(int)
tot = 0
toti = 0
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        f = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit():
        continue
    d = dict(zip(hdr[2:], row[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        n_i = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    tot += s
    toti += n_i
    ln = int(row[0])
    if f == "ss_kernel.cu":
        name = None
        for a, n in secs:
            if a <= ln:
                name = (a, n)
        agg[name] += s
        ins[name] += n_i
    else:
        agg[(0, f)] += s
        ins[(0, f)] += n_i
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:30]:
    print(f"{100 * v / tot:5.1f}% samples {100 * ins[k] / max(toti, 1):5.1f}% instr  {k}")
