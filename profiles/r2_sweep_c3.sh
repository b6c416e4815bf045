mkdir -p gpurun_out
for B in 256 512 1024 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_sweep_b$B.log 2>&1; done
for B in 512 1024; do HIVF_TC_WIDE2_PPL=0 timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_sweep_w128_b$B.log 2>&1; done
for B in 2048 4096; do HIVF_TC_WIDE2_PPL=-1 timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_sweep_w64_b$B.log 2>&1; done
echo done
