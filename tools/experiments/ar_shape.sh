for cfg in "1 256" "2 256" "1 512" "2 512"; do set -- $cfg
for N in 2 4; do
SMPU_AR_UNROLL=$1 SMPU_AR_THREADS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2971$N tools/ar_bench.py 2>/dev/null | grep fused | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('U=$1 T=$2 W=$N standalone bus %.0f' % d['bus_gbs'])"
SMPU_AR_UNROLL=$1 SMPU_AR_THREADS=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['exposed_comm']; print('   step ms=%.3f exposed=%.3f (%.1f%%) bus=%.0f' % (d['ms_per_step'], e['ms'], 100*e['frac_of_update'], d['allreduce']['bus_gbs']))"
done; done
SMPU_AR_UNROLL=2 timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "primitive or world4_real_fused" 2>&1 | tail -1
