set -u
OUT=gpurun_out; TAG=${1:-s5}
RX="regex:stream_kernel_v<double, (\\(int\\))?2, (\\(int\\))?1, (\\(bool\\))?(1|true), (\\(int\\))?2, (\\(bool\\))?(1|true)>"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "$RX" --launch-skip 5 --launch-count 1 -o /tmp/${TAG}_v -f python scripts/ncu_target.py > $OUT/${TAG}_ncu_v.log 2>&1
echo rc=$?
ncu -i /tmp/${TAG}_v.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_v_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_v.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_ncu_v_sass.csv 2>/dev/null
