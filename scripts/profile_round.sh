#!/bin/bash
# GPU-box profiling recipe for the headline (BASELINE config 3), one GPU:
#   1. (bench.py itself runs in scripts/gpu_round.sh)
#   2. ncu launch list of bench.py (gpu__time_duration per launch, serialised)
#   3. ncu --set full of the two dominant kernels of one solve (the finest
#      level's vertically fused pass, stream_kernel_v<..., FINEST>; the largest
#      coarse down pair, stream_kernel_d), located from a launch list of
#      scripts/ncu_target.py
# Usage (from the repo root, under gpurun):  bash scripts/profile_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu \
    > $OUT/${TAG}_ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches_target.csv python scripts/ncu_target.py > $OUT/${TAG}_ncu_target.log 2>&1
echo "target launch list rc=$?"
# index (among launches of the same kernel name) of the longest K_UP2DOWN (finest, fused) and K_UP2 (level 1) launch
read SKIP4 SKIP5 < <(python - "$OUT/${TAG}_launches_target.csv" <<'EOF'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
norm = lambda k: k.replace("(int)", "").replace("(bool)", "").replace("true", "1")
def best(tag):
    seq = [float(r[vi].replace(",", "")) for r in rows if tag in norm(r[ki])]
    return max(range(len(seq)), key=lambda i: seq[i]) if seq else 0
print(best("stream_kernel_v<double, 2, 1, 1, 2, 1>"), best("stream_kernel_d<double, 2, 1, 1,"))
EOF
)
echo "skip kind4=$SKIP4 kind5=$SKIP5"
for K in v d; do
    S=$([ $K = v ] && echo $SKIP4 || echo $SKIP5)
    if [ $K = v ]; then RX="regex:stream_kernel_v<double, (\\(int\\))?2, (\\(int\\))?1, (\\(bool\\))?(1|true), (\\(int\\))?2, (\\(bool\\))?(1|true)>";
    else RX="regex:stream_kernel_d<"; fi
    timeout 900 ncu --set full --import-source on --clock-control none \
        --kernel-name-base demangled \
        -k "$RX" --launch-skip $S --launch-count 1 \
        -o /tmp/${TAG}_ncu_kind$K -f python scripts/ncu_target.py > $OUT/${TAG}_ncu_kind$K.log 2>&1
    echo "ncu full kind$K rc=$?"
    # reports are ~30 MB each: bring back the raw metrics and the SASS source page only
    ncu -i /tmp/${TAG}_ncu_kind$K.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_kind${K}_raw.csv 2>/dev/null
    ncu -i /tmp/${TAG}_ncu_kind$K.ncu-rep --page source --csv --print-source sass \
        > $OUT/${TAG}_ncu_kind${K}_sass.csv 2>/dev/null
done
