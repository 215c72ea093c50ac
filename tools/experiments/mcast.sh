for MC in 0 1; do
echo "== SMPU_AR_MCAST=$MC"
SMPU_AR_MCAST=$MC timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "primitive or world4_real_fused or world2 and fused and not graph" 2>&1 | tail -1
for N in 2 4; do
SMPU_AR_MCAST=$MC timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969$N tools/ar_bench.py 2>/dev/null | grep fused
SMPU_AR_MCAST=$MC timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['exposed_comm']; print('W=$N ms=%.3f exposed=%.3f (%.1f%%) bus=%.0f' % (d['ms_per_step'], e['ms'], 100*e['frac_of_update'], d['allreduce']['bus_gbs']))"
done; done
