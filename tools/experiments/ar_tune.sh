for V in 0 1; do for C in 1 2 4; do
SMPU_AR_VEC32=$V SMPU_AR_CTAS_PER_SM=$C timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > /tmp/b2.log 2>&1; tail -1 /tmp/b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('vec32=$V ctas=$C ms=%.3f calls=%.3f exposed=%.3f bus=%.0f' % (d['ms_per_step'], d['graph']['ms_per_step_calls'], d['exposed_comm']['ms'], d['allreduce']['bus_gbs']))"
done; done
SMPU_AR_VEC32=1 timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "world2 and fused" 2>&1 | tail -1
