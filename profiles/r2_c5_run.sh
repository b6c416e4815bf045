# node-split path: subsearch/compat tests, C5 sub-stage latency, sub-stage kernel launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_subsearch.py tests/test_c5_stream.py tests/test_compat.py tests/test_cpp_adapter.py -q -x > gpurun_out/c5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c5_tests.log
timeout 900 python bench.py --config c5sched > gpurun_out/c5_sched.log 2>&1
bash profiles/r2_c5_launches.sh
echo done
