# e2e with pinned host queries (C1/C2/C3), and the drop-bound seed at C3 B=256
mkdir -p gpurun_out
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/sm_c1.log 2>&1
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/sm_c2.log 2>&1
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/sm_c3.log 2>&1
HIVF_OPTS="seed_ppl=0" timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/sm_c3_seed.log 2>&1
HIVF_OPTS="seed_ppl=0" timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/sm_c2_seed.log 2>&1
echo done
