mkdir -p gpurun_out/sweep2
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 2>&1 | tail -9
for N in 2 4; do for MIB in 4 16 64 150 256; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N bench.py --gpus $N --steps 20 --warmup 5 --no-e2e --bucket-mib $MIB > gpurun_out/sweep2/w${N}_${MIB}.log 2>&1
tail -1 gpurun_out/sweep2/w${N}_${MIB}.log > gpurun_out/sweep2/w${N}_${MIB}.json
python -c "import json; d=json.load(open('gpurun_out/sweep2/w${N}_${MIB}.json')); e=d['exposed_comm']; a=d['allreduce']; print('W=$N ${MIB}MiB nb=%d ms=%.3f exposed=%.3f (%.1f%%) bus=%.0f' % (d['config']['n_buckets'], d['ms_per_step'], e['ms'], 100*e['frac_of_update'], a['bus_gbs']))" || tail -2 gpurun_out/sweep2/w${N}_${MIB}.log
done; done
