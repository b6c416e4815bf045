# N-rank bench path at HEAD, functional simulation on one GPU (gloo host transport; not a reported number)
mkdir -p gpurun_out
HIVF_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/sim_n2.log 2>&1; echo "rc=$?" >> gpurun_out/sim_n2.log
echo done
