mkdir -p gpurun_out
python -m pytest tests/test_gpu_multi.py -q -s 2>&1 | grep -E "ok|FAIL|passed|failed|ulp" | tail -20
for N in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > gpurun_out/bench${N}_c.log 2>&1
tail -1 gpurun_out/bench${N}_c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($N, d['ms_per_step'], d.get('exposed_comm'), d.get('allreduce'))"
done
