# Final round-2 evidence at HEAD (after the tensor-core coarse pass, set-mode select,
# rank placement, two-lane tiered indexes): GPU suite, smoke, bench lines, reference arm,
# C3z two-lane, dense batches, C5 through the reference scheduler
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f4_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/f4_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f4_smoke.log
timeout 900 python bench.py > gpurun_out/f4_bench_c3.log 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/f4_bench_c2.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/f4_bench_c1.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/f4_ref_c3.log 2>&1
timeout 900 python bench.py --config c3z --hbm-budget-gb 16 --steps 10 > gpurun_out/f4_c3z16.log 2>&1
for B in 1024 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 > gpurun_out/f4_b$B.log 2>&1; done
timeout 900 python bench.py --config c5sched > gpurun_out/f4_c5sched_gpu.log 2>&1
echo done
