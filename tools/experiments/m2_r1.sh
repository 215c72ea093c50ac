mkdir -p gpurun_out
timeout 300 python bench.py --mode m2 --steps 6 --warmup 2 > gpurun_out/m2_1.log 2>&1; tail -3 gpurun_out/m2_1.log
for AR in fused nccl; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --mode m2 --steps 6 --warmup 2 --allreduce $AR > gpurun_out/m2_2_$AR.log 2>&1; tail -1 gpurun_out/m2_2_$AR.log
done
