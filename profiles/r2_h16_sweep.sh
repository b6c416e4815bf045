# fp16 filter copy: C3 batch sweep (default kernel choice + alternatives), stall counters
mkdir -p gpurun_out
for B in 512 1024 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/h16s_b$B.log 2>&1; done
HIVF_TC_PAIR_PPL=-1 timeout 600 python bench.py --batch 4096 --steps 10 --warmup 3 --no-cpu > gpurun_out/h16s_w128_b4096.log 2>&1
HIVF_TC_PAIR_PPL=0 timeout 600 python bench.py --batch 2048 --steps 10 --warmup 3 --no-cpu > gpurun_out/h16s_pair_b2048.log 2>&1
HIVF_TC_WIDE2_PPL=-1 timeout 600 python bench.py --batch 1024 --steps 10 --warmup 3 --no-cpu > gpurun_out/h16s_w64_b1024.log 2>&1
HIVF_TCPROF=gpurun_out/tcprof_h16_b256.npy timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu > gpurun_out/h16s_prof_b256.log 2>&1
HIVF_TCPROF=gpurun_out/tcprof_h16_b4096.npy timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > gpurun_out/h16s_prof_b4096.log 2>&1
echo done
