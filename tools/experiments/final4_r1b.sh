mkdir -p gpurun_out/final
timeout 2700 python -m pytest tests -m gpu -q -x --durations=6 2>&1 | tail -10
python bench.py > gpurun_out/final/n1.json 2> gpurun_out/final/n1.err; tail -1 gpurun_out/final/n1.json | cut -c1-200
for N in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2965$N bench.py --gpus $N > gpurun_out/final/n$N.log 2>&1; tail -1 gpurun_out/final/n$N.log > gpurun_out/final/n$N.json
python -c "import json; d=json.load(open('gpurun_out/final/n$N.json')); print($N, d['ms_per_step'], '%.3e' % d['value'], d['exposed_comm'], d['e2e']['value'])"
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/ref.json 2>&1; tail -1 gpurun_out/final/ref.json | cut -c1-300
