# C3 batch sweep at HEAD (fp16 filter copy, tensor-core coarse pass, set-mode select)
mkdir -p gpurun_out
for B in 64 128 256 512 1024 2048 4096; do timeout 600 python bench.py --batch $B --steps 10 --warmup 3 --no-cpu > gpurun_out/hs_b$B.log 2>&1; done
echo done
