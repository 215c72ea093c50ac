timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "primitive" 2>&1 | tail -2
for N in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2967$N tools/ar_bench.py 2>/dev/null | grep world
done
