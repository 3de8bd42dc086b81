timeout 900 python -m pytest tests/test_gpu_scale_and_edges.py -q -m gpu -k "stream" > gpurun_out/r02u_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02u_pytest.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r02u_bench.json 2> gpurun_out/r02u_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/r02u_bench.err
