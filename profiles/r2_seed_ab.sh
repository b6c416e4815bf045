# drop-bound seed A/B on C3 dense batches (one box, alternating), + wide parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/seed_tests.log 2>&1; echo "rc=$?" >> gpurun_out/seed_tests.log
for r in 1 2; do
  for B in 1024 4096; do
    HIVF_OPTS="seed_rows=0" timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/seed_off_r${r}_b$B.log 2>&1
    timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/seed_on_r${r}_b$B.log 2>&1
  done
done
HIVF_OPTS="seed_rows=64" timeout 600 python bench.py --batch 4096 --steps 10 --warmup 3 --no-cpu > gpurun_out/seed_64_b4096.log 2>&1
timeout 600 python bench.py --batch 2048 --steps 10 --warmup 3 --no-cpu > gpurun_out/seed_on_b2048.log 2>&1
HIVF_TC_PAIR_PPL=-1 timeout 600 python bench.py --batch 4096 --steps 10 --warmup 3 --no-cpu > gpurun_out/seed_on_w128_b4096.log 2>&1
echo done
