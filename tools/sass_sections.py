"""Dev tool: instructions executed and stall samples of one scheduler kernel
per KERNEL-LEVEL source section (inlined helpers charged to their call site).

    python tools/sass_sections.py <ncu source csv (--print-source sass,cuda)> <cubin> <mangled kernel> [ranges]

The ncu source page attributes an inlined helper's SASS to the helper's own
line; nvdisasm -gi prints each instruction's inline chain, whose outermost
ss_kernel.cu line is the kernel statement that expanded it. Noinline callees
(q_insert32, refill, queue_has_stale, ...) are separate functions and are
reported by name.
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

# kernel line ranges (ss_kernel.cu) -> section name; edit to the file's layout
SECTIONS = [
    ("trace init", 834, 956),
    ("admission/refill/anom", 957, 1032),
    ("stretch entry+setup+vote", 1033, 1171),
    ("per-round fast body", 1172, 1294),
    ("chunk: clock chain", 1295, 1337),
    ("chunk: order screen", 1338, 1378),
    ("chunk: exact loop", 1379, 1397),
    ("chunk: stop vote", 1398, 1416),
    ("chunk: digest", 1417, 1427),
    ("chunk: log", 1428, 1446),
    ("chunk: commit", 1447, 1464),
    ("stretch order/exit", 1465, 1512),
    ("g: composition", 1513, 1664),
    ("g: KV admission", 1665, 1827),
    ("g: batch duration", 1828, 1868),
    ("g: progress", 1869, 1956),
    ("g: record+digest", 1957, 2003),
    ("g: ongoing rebuild", 2004, 2045),
    ("g: queue rebuild", 2046, 2070),
    ("outputs/stats", 2071, 2131),
]


def kernel_lines(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-gi", cubin], capture_output=True, text=True).stdout.splitlines()
    start = out.index(f".text.{kernel}:")
    off_line, funcs = {}, {}
    cur = None
    sec = kernel
    for ln in out[start:]:
        if ln.startswith(".text.") and ln.endswith(":"):
            sec = ln[6:-1]
        if ln.startswith(".nv.constant0") or (ln.startswith(".text.") and sec != kernel and "sched_kernel" in sec):
            break
        m = re.match(r'\s*//## File "(.*)", line (\d+)$', ln)
        if m and m.group(1).endswith("ss_kernel.cu"):
            cur = int(m.group(2))
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m and sec == kernel:
            off_line[int(m.group(1), 16)] = (cur, m.group(2).strip(" ;"))
    return off_line


def main():
    csv_path, cubin, kernel = sys.argv[1:4]
    off_line = kernel_lines(cubin, kernel)
    size = max(off_line) + 16
    rows = []
    hdr = None
    for row in csv.reader(io.StringIO(open(csv_path).read())):
        if row and row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < 8 or not row[2].startswith("0x"):
            continue
        d = dict(zip(hdr, row))
        rows.append((int(row[2], 16), row[3].strip(), int(d["Instructions Executed"] or 0),
                     int(d["Warp Stall Sampling (All Samples)"] or 0)))
    # the kernel's base: the address whose instruction stream matches offset 0
    first = off_line[0][1].split()[0]
    cands = sorted({a for a, s, _, _ in rows if s.split()[0] == first})
    by_addr = {a: s for a, s, _, _ in rows}
    base = next(b for b in cands if all(by_addr.get(b + o, "").split()[:1] == off_line[o][1].split()[:1]
                                        for o in list(off_line)[:200:7] if (b + o) in by_addr))
    agg = defaultdict(lambda: [0, 0])
    for a, s, ins, smp in rows:
        o = a - base
        if 0 <= o < size and o in off_line:
            ln = off_line[o][0] or 0
            name = next((n for n, lo, hi in SECTIONS if lo <= ln <= hi), f"line {ln}")
        else:
            name = "noinline callees"
        agg[name][0] += ins
        agg[name][1] += smp
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"{kernel}: {ti:.4g} warp-instructions, {ts} samples")
    for n, (i, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {n:32s} instr {100 * i / ti:5.1f}%  samples {100 * s / ts:5.1f}%")


if __name__ == "__main__":
    main()
