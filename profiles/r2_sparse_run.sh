# finer segments for sparse tensor-core batches: parity / node-split / compat suites, C5 latency, C1 line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_subsearch.py tests/test_c5_stream.py tests/test_compat.py tests/test_cpp_adapter.py tests/test_gpu_wide.py tests/test_gpu_limits.py -q -x > gpurun_out/sp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sp_tests.log
timeout 900 python bench.py --config c5sched > gpurun_out/sp_c5sched.log 2>&1
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/sp_c1.log 2>&1
bash profiles/r2_c5_launches.sh
echo done
