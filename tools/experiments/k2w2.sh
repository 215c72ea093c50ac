for K2 in 0 2 3; do
SMPU_K2_CTAS_PER_SM=$K2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['exposed_comm']; print('K2cps=$K2 ms=%.3f t1=%.3f exposed=%.3f (%.1f%%) bus=%.0f' % (d['ms_per_step'], e['t_world1_ms'], e['ms'], 100*e['frac_of_update'], d['allreduce']['bus_gbs']))"
done
