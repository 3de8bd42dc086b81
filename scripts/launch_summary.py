"""Summarise an ncu --metrics gpu__time_duration.sum launch list: one warm
batched solve (between the 2nd and 3rd residual-norm kernels) by kernel."""
import collections
import csv
import re
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
seq = [(re.sub(r"\(.*", "", r[ki])[:72], float(r[vi].replace(",", "")) * scale[r[ui]]) for r in rows]
r0 = [i for i, (n, _) in enumerate(seq) if re.search(r"stream_kernel<double, \d, 0, 1, 0, 0>", n)]
a, b = r0[1], r0[2]
tot, cnt = collections.defaultdict(float), collections.Counter()
for n, v in seq[a:b]:
    tot[n] += v
    cnt[n] += 1
T = sum(tot.values())
print(f"one warm solve: {T / 1e3:.3f} ms of kernel time, {b - a} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e3:9.3f} ms {100 * v / T:5.1f}% {cnt[k]:4d}  {k}")
print("first cycle, per launch (us):")
for n, v in seq[a:a + 2 + 2 * 24]:
    print(f"{v:9.1f}  {n}")
