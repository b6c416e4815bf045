# Round-2 evidence refresh at HEAD (one box): GPU suite, smoke, C1/C2/C3 bench lines, C3 reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2g_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_smoke.log
timeout 900 python bench.py > gpurun_out/r2g_bench_c3.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/r2g_bench_c1.log 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/r2g_bench_c2.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r2g_ref_c3.log 2>&1
echo done
