set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "w_f_cycle or f_cycle or w_cycle or tail or cycles" > gpurun_out/r02z_pytest_f.txt 2>&1
tail -3 gpurun_out/r02z_pytest_f.txt
python - > gpurun_out/r02z_fcycle.txt 2>&1 <<'PY'
import sys, time
sys.path.insert(0, ".")
sys.argv = ["x"]
import scripts.bench_suite as bs
for cyc, kw in (("V", {}), ("F", {}), ("W", dict(coarsest=1024, coarse="scan"))):
    for nu in (1, 2):
        r = bs.solve_case(2, 1 << 20, 1.0, nu, cyc, reps=3, **kw)
        print(cyc, nu, r, flush=True)
PY
cat gpurun_out/r02z_fcycle.txt
