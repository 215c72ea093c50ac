mkdir -p gpurun_out
nvidia-smi topo -m | head -5
python -m pytest tests/test_gpu_multi.py -q -s 2>&1 | tail -30
NCCL_DEBUG=INFO python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench2.log 2>&1
grep -E "NVLS|Algo|algorithm|Channel 00" gpurun_out/bench2.log | head -10
tail -1 gpurun_out/bench2.log
