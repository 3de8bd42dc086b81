"""Key metrics of an ncu --set full report (raw page) and instruction mix."""
import collections
import csv
import io
import re
import subprocess
import sys

# argument: a .ncu-rep, or the prefix of the <prefix>_raw.csv / <prefix>_sass.csv
# exports that scripts/profile_round.sh brings back from the GPU box
rep = sys.argv[1]
if rep.endswith(".ncu-rep"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
else:
    raw = open(rep + "_raw.csv").read()
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]
for d in data:
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k:62s} {d[i]} {units[i]}")
    print("  --")
if rep.endswith(".ncu-rep"):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout.splitlines()
else:
    src = open(rep + "_sass.csv").read().splitlines()
rows = list(csv.reader(src[1:]))
hdr = rows[0]
si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
op = collections.Counter()
tot = 0.0
for r in rows[1:]:
    if len(r) < len(hdr) or r[0] == "Kernel Name":
        break
    try:
        v = float(r[ei] or 0)
    except ValueError:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[si])
    if m:
        op[m.group(2)] += v
        tot += v
print(f"  instructions (first kernel): {tot:.0f}")
for k, v in op.most_common(24):
    print(f"  {k:10s} {100 * v / tot:6.2f}%")
