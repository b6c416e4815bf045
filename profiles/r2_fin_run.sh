# finalize: chunked staging of the candidate slots (pair scans: > 320 slots per query)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_tc_bound.py -q -x > gpurun_out/fin_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fin_tests.log
for B in 256 1024 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/fin_b$B.log 2>&1; done
echo done
