mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --trace gpurun_out/trace_w1.jsonl > /dev/null 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29593 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --trace gpurun_out/trace_w2.jsonl > gpurun_out/trace_w2_bench.log 2>&1
tail -1 gpurun_out/trace_w2_bench.log | cut -c1-300
ls gpurun_out | grep trace
