# Round-2 multi-GPU and fp32-path evidence at HEAD: every shard of the 8-GPU C3 and
# Zipf C4 jobs timed on one B200 (per-shard parity), the N=2 bench path simulated on
# one GPU (gloo), and the GPU suite with every scan on the fp32 lists
mkdir -p gpurun_out
timeout 1800 python bench.py --shard all/8 > gpurun_out/f5_shard_c3.log 2>&1
HIVF_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/f5_sim_n2.log 2>&1; echo "rc=$?" >> gpurun_out/f5_sim_n2.log
HIVF_FILTER_H16=0 timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f5_gputest_fp32_lists.log 2>&1; echo "rc=$?" >> gpurun_out/f5_gputest_fp32_lists.log
timeout 2400 python bench.py --config c4 --shard all/8 > gpurun_out/f5_shard_c4.log 2>&1
echo done
