# out-of-line insertion path for <= 3 (128-query) / <= 8 (pair) candidates per tile: wide tests + dense C3 batches
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/ins2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ins2_tests.log
for B in 1024 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/ins2_b$B.log 2>&1; done
HIVF_TC_PAIR_PPL=-1 timeout 600 python bench.py --batch 4096 --steps 10 --warmup 3 --no-cpu > gpurun_out/ins2_w128_b4096.log 2>&1
echo done
