mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -s -x 2>&1 | grep -E "ok|FAIL|passed|failed|Error|error" | tail -12
for N in 2 4; do for AR in fused nccl; do for MIB in 16 64 150; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --allreduce $AR --bucket-mib $MIB > gpurun_out/sweep_${N}_${AR}_${MIB}.log 2>&1
tail -1 gpurun_out/sweep_${N}_${AR}_${MIB}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('exposed_comm',{}); a=d.get('allreduce',{}); print('W=$N $AR ${MIB}MiB nb=%d ms=%.3f exposed=%.3f (%.1f%%) ar_bus=%.0f' % (d['config']['n_buckets'], d['ms_per_step'], e.get('ms',0), 100*e.get('frac_of_update',0), a.get('bus_gbs',0)))" || tail -3 gpurun_out/sweep_${N}_${AR}_${MIB}.log
done; done; done
