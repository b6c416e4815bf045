mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_wide.py -q -x -k pairs256 > gpurun_out/r2_pair_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pair_tests2.log
for r in 1 2; do
  for B in 4096; do
    HIVF_TC_PAIR_PPL=-1 timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_ab2${r}_w128_b$B.log 2>&1
    HIVF_TC_PAIR_PPL=0 timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_ab2${r}_pair_b$B.log 2>&1
  done
done
echo done
