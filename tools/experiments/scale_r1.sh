mkdir -p gpurun_out/scale
python bench.py --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/scale/n1.json 2>gpurun_out/scale/n1.err; tail -1 gpurun_out/scale/n1.json | cut -c1-200
for N in 2 4; do
for V in "--optimizer replicated" "--optimizer sharded"; do
tag=n${N}${V:+_sharded}
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --steps 20 --warmup 5 $V > gpurun_out/scale/$tag.log 2>&1
tail -1 gpurun_out/scale/$tag.log > gpurun_out/scale/$tag.json
python -c "import json; d=json.load(open('gpurun_out/scale/$tag.json')); e=d.get('exposed_comm',{}); print('$tag', round(d['ms_per_step'],3), '%.3e'%d['value'], 'exposed', round(e.get('ms',0),3), round(e.get('frac_of_update',0),3), d.get('allreduce',{}).get('bus_gbs'))" || tail -3 gpurun_out/scale/$tag.log
done; done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29619 bench.py --gpus 4 --mode m2 --steps 6 --warmup 2 > gpurun_out/scale/n4_m2.log 2>&1; tail -1 gpurun_out/scale/n4_m2.log > gpurun_out/scale/n4_m2.json; cut -c1-150 gpurun_out/scale/n4_m2.json; python -c "import json; d=json.load(open('gpurun_out/scale/n4_m2.json')); print(d.get('exposed_comm'))"
