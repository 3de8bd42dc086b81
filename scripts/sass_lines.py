"""Attribute an ncu SASS source page (--page source --csv --print-source sass)
to CUDA source lines using `nvdisasm -g -c` of the same cubin.

    python scripts/sass_lines.py all.dis <mangled kernel> hot_sass.csv [top]
"""
import collections
import csv
import re
import sys

dis, fn, sass = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
cur, insts = ("?", 0), []
for l in lines[start + 1:]:
    if l.startswith("//----") or l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        insts.append((cur, m.group(2).strip()))
rows = list(csv.reader(open(sass)))
hdr, rows = rows[1], rows[2:]
si, ie, src = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"),
               hdr.index("Source"))
assert len(rows) == len(insts), (len(rows), len(insts))
bad = sum(1 for r, (_, t) in zip(rows, insts) if r[src].split()[0] != t.split()[0])
samp, ex = collections.Counter(), collections.Counter()
for r, (loc, _) in zip(rows, insts):
    samp[loc] += float(r[si])
    ex[loc] += float(r[ie])
T, E = sum(samp.values()), sum(ex.values())
print(f"{len(insts)} instructions, opcode mismatches {bad}; samples {T:.0f}, executed {E:.0f}")
for loc, v in samp.most_common(top):
    print(f"{100 * v / T:5.1f}% samples {100 * ex[loc] / E:5.1f}% inst  {loc[0]}:{loc[1]}")
