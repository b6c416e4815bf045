# CTA-pair scan with a 4-slot TMEM ring (tiles of <= 128 queries 4-deep): pair parity (forced), dense C3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x > gpurun_out/t4_wide.log 2>&1; echo "rc=$?" >> gpurun_out/t4_wide.log
HIVF_TC_PAIR_PPL=0 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t4_suite_pairs.log 2>&1; echo "rc=$?" >> gpurun_out/t4_suite_pairs.log
for B in 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/t4_b$B.log 2>&1; done
HIVF_TC_PAIR_PPL=0 timeout 600 python bench.py --batch 2048 --steps 10 --warmup 3 --no-cpu > gpurun_out/t4_pair_b2048.log 2>&1
HIVF_TCPROF=gpurun_out/tcprof_t4_pair_b4096.npy timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
echo done
