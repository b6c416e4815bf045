# Pair scan bottleneck split at C3 B=4096 (debug variants, results inexact, timing only):
# 0 = full kernel, 4 = no MMAs, 32 = no tile epilogue, 36 = neither (load pipeline + handshakes only)
mkdir -p gpurun_out
for v in 0 4 32 36; do
  HIVF_TC_PAIR_PPL=0 HIVF_OPTS="scan_kernel=3,tc_variant=$v" timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > gpurun_out/r2_pv_$v.log 2>&1
done
for v in 0 4; do
  HIVF_TC_PAIR_PPL=-1 HIVF_OPTS="scan_kernel=3,tc_variant=$v" timeout 600 python bench.py --batch 4096 --steps 4 --warmup 3 --no-cpu > gpurun_out/r2_wv_$v.log 2>&1
done
echo done
