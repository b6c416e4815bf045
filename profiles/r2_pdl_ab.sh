# A/B of programmatic dependent launch on the search path (HIVF_PDL=0 vs default), one box, alternating
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gputest_pdl.log 2>&1; echo "rc=$?" >> gpurun_out/r2_gputest_pdl.log
for r in 1 2; do
  for c in c1 c2; do
    HIVF_PDL=0 timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r2_pdl${r}_off_$c.log 2>&1
    timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r2_pdl${r}_on_$c.log 2>&1
  done
done
echo done
