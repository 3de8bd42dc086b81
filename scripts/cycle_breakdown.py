"""Per-launch times of one full cycle from an ncu launch list of
scripts/ncu_target.py (TMG_NO_SOLVE_GRAPH=1):  python scripts/cycle_breakdown.py l.csv"""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
sc = {"ns": 1e-3, "us": 1, "ms": 1e3, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
seq = []
for r in rows:
    name = r[ki]
    m = re.search(r"stream_kernel<\w+, (?:\(int\))?(\d+), (?:\(int\))?(\d+), (?:\(bool\))?(\d), (?:\(int\))?(\d+), "
                  r"(?:\(int\))?(\d+)>", name)
    short = f"stream NT={m.group(1)} NU={m.group(2)} kind={m.group(4)}" if m else re.sub(r"\(.*", "", name)[-40:]
    seq.append((short, float(r[vi].replace(",", "")) * sc[r[ui]], r[gi] if gi else ""))
idx = [i for i, (n, _, _) in enumerate(seq) if "kind=4" in n]
a, b = idx[-3], idx[-2]
print(f"one cycle: {b - a} launches, {sum(t for _, t, _ in seq[a:b]):.1f} us")
for n, t, g in seq[a:b]:
    print(f"  {t:9.1f} us {g:>14} {n}")
