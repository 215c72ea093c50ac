mkdir -p gpurun_out/var
for i in 1 2 3; do
python bench.py --no-e2e --no-cpu-baseline > gpurun_out/var/n1_$i.json 2>/dev/null
done
for N in 2 4; do for i in 1 2; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2968$N bench.py --gpus $N --no-e2e > gpurun_out/var/n${N}_$i.log 2>&1; tail -1 gpurun_out/var/n${N}_$i.log > gpurun_out/var/n${N}_$i.json
done; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/var/*.json')):
    d = json.load(open(f))
    e = d.get('exposed_comm', {})
    print(f.split('/')[-1], round(d['ms_per_step'], 4), '%.4e' % d['value'], round(d['roofline']['frac'], 3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), round(e.get('frac_of_update', 0), 3), d['graph']['resident_microbatches']['ms_per_step'])
PY
