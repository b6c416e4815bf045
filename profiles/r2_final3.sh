# Final round-2 evidence at HEAD: smoke, bench lines C3/C2/C1 (+CPU baseline), reference arm, C5 live, dense batches
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f3_smoke.log
timeout 900 python bench.py > gpurun_out/f3_bench_c3.log 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/f3_bench_c2.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/f3_bench_c1.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/f3_ref_c3.log 2>&1
timeout 900 python bench.py --config c5sched > gpurun_out/f3_c5sched_gpu.log 2>&1
for B in 1024 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 > gpurun_out/f3_b$B.log 2>&1; done
echo done
