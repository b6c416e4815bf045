# stage-block MMA issue: parity subset + C3 bench lines across batch sizes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py tests/test_gpu_subsearch.py -q -x > gpurun_out/s8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s8_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s8_b256.log 2>&1
for B in 1024 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/s8_b$B.log 2>&1; done
HIVF_TC_PAIR_PPL=-1 timeout 600 python bench.py --batch 4096 --steps 10 --warmup 3 --no-cpu > gpurun_out/s8_w128_b4096.log 2>&1
HIVF_TC_PAIR_PPL=0 timeout 600 python bench.py --batch 2048 --steps 10 --warmup 3 --no-cpu > gpurun_out/s8_pair_b2048.log 2>&1
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu > gpurun_out/s8_c2.log 2>&1
echo done
