for N in 2 4; do for C in 37 74 148; do
SMPU_AR_VEC32=1 SMPU_AR_CTAS=$C timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > /tmp/b2.log 2>&1; tail -1 /tmp/b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=$N ctas=$C ms=%.3f calls=%.3f exposed=%.3f bus=%.0f resident=%.3f' % (d['ms_per_step'], d['graph']['ms_per_step_calls'], d['exposed_comm']['ms'], d['allreduce']['bus_gbs'], d['graph']['resident_microbatches']['ms_per_step']))"
done; done
