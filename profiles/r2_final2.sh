# Round-2 evidence at HEAD (fp16 filter copy + stage-block MMA issue), one box
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f2_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/f2_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f2_smoke.log
timeout 900 python bench.py > gpurun_out/f2_bench_c3.log 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/f2_bench_c2.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/f2_bench_c1.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/f2_ref_c3.log 2>&1
timeout 900 python bench.py --config c5sched > gpurun_out/f2_c5sched_gpu.log 2>&1
HIVF_NCU_RANGE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/f2_launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 2 -c 1 -o gpurun_out/f2_scan_c3 python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 1800 python bench.py --shard all/8 > gpurun_out/f2_shard_c3.log 2>&1
timeout 2400 python bench.py --config c4 --shard all/8 > gpurun_out/f2_shard_c4.log 2>&1
echo done
