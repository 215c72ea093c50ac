timeout 1700 python -m pytest tests/test_gpu_multi.py -q -s -x -k c3 2>&1 | grep -E "C3|FAIL|passed|failed|update|Error" | tail -15
for N in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > /tmp/b$N.log 2>&1
tail -1 /tmp/b$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d.get('exposed_comm',{}); a=d.get('allreduce',{}); print('W=$N ms=%.3f value=%.3e exposed=%.3f (%.1f%%) ar_bus=%.0f impl=%s' % (d['ms_per_step'], d['value'], e.get('ms',0), 100*e.get('frac_of_update',0), a.get('bus_gbs',0), a.get('impl')))"
done
