# Round-2 evidence at HEAD (one box): GPU suite, smoke, bench lines, reference arm, launch list, ncu capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2f_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2f_bench_c3.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r2f_ref_c3.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/r2f_bench_c1.log 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/r2f_bench_c2.log 2>&1
timeout 900 python bench.py --config c5sched > gpurun_out/r2f_c5sched_gpu.log 2>&1
timeout 1200 python bench.py --config c5sched --impl reference > gpurun_out/r2f_c5sched_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -s 170 -c 200 --csv --log-file gpurun_out/r2f_launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 2 -c 1 -o gpurun_out/r2f_scan_c3 python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
echo done
