# GPU suite on both filter paths: the fp16 filter copy (default) and the fp32 lists (HIVF_FILTER_H16=0)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/suite_h16.log 2>&1; echo "rc=$?" >> gpurun_out/suite_h16.log
HIVF_FILTER_H16=0 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/suite_fp32.log 2>&1; echo "rc=$?" >> gpurun_out/suite_fp32.log
echo done
