mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench2b.log 2>&1
tail -1 gpurun_out/bench2b.log
python bench.py --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench1b.log 2>&1; tail -1 gpurun_out/bench1b.log
