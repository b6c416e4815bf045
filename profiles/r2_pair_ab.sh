# A/B of the CTA-pair scan (k_scan_pair) on one box: C3 dense batches, alternating runs
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/r2_pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pair_tests.log
for r in 1 2; do
  for B in 2048 4096; do
    HIVF_TC_PAIR_PPL=-1 timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_ab${r}_w128_b$B.log 2>&1
    HIVF_TC_PAIR_PPL=0 timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_ab${r}_pair_b$B.log 2>&1
  done
done
HIVF_TC_PAIR_PPL=0 HIVF_TCPROF=gpurun_out/tcprof_pair_b4096.npy timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > gpurun_out/r2_tcprof_pair_b4096.log 2>&1
echo done
