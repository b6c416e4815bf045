mkdir -p gpurun_out
HIVF_TC_PAIR_PPL=-1 HIVF_TCPROF=gpurun_out/tcprof_s8_w128_b4096.npy timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
HIVF_TCPROF=gpurun_out/tcprof_s8_pair_b4096.npy timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
HIVF_TCPROF=gpurun_out/tcprof_s8_b256.npy timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu > /dev/null 2>&1
for v in 32 36; do HIVF_TC_PAIR_PPL=0 HIVF_OPTS="scan_kernel=3,tc_variant=$v" timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > gpurun_out/s8_pv_$v.log 2>&1; done
echo done
