mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -q -s -x 2>&1 | grep -E "ok|FAIL|passed|failed|Error|error" | tail -20
for AR in fused nccl; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --allreduce $AR > gpurun_out/bench2_$AR.log 2>&1
tail -1 gpurun_out/bench2_$AR.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$AR', d['ms_per_step'], d.get('exposed_comm',{}).get('ms'), d.get('allreduce'))" || tail -5 gpurun_out/bench2_$AR.log
done
