# fp16 filter copy: GPU suite, C3/C2/C1 bench lines, C3 launch list + one ncu --set full of the scan
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/h16_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/h16_gputest.log
timeout 900 python bench.py > gpurun_out/h16_bench_c3.log 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/h16_bench_c2.log 2>&1
timeout 600 python bench.py --config c1 > gpurun_out/h16_bench_c1.log 2>&1
HIVF_NCU_RANGE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/h16_launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 2 -c 1 -o gpurun_out/h16_scan_c3 python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
echo done
