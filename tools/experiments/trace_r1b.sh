mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29593 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --trace gpurun_out/trace2_w2.jsonl > gpurun_out/trace2_w2_bench.log 2>&1
tail -1 gpurun_out/trace2_w2_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('exposed_comm',{}); a=d.get('allreduce',{}); print('W=2 ms=%.3f exposed=%.3f (%.1f%%) ar_bus=%.0f' % (d['ms_per_step'], e.get('ms',0), 100*e.get('frac_of_update',0), a.get('bus_gbs',0)))"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29594 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --allreduce nccl > gpurun_out/trace2_w2n_bench.log 2>&1
tail -1 gpurun_out/trace2_w2n_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('exposed_comm',{}); a=d.get('allreduce',{}); print('W=2 nccl ms=%.3f exposed=%.3f (%.1f%%) ar_bus=%.0f' % (d['ms_per_step'], e.get('ms',0), 100*e.get('frac_of_update',0), a.get('bus_gbs',0)))"
