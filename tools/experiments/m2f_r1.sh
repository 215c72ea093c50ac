for F in "" "--m2-fused"; do
timeout 300 python bench.py --mode m2 --steps 6 --warmup 2 $F > /tmp/m.log 2>&1; tail -1 /tmp/m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W1 $F', round(d['ms_per_step'],2), d['producer'], '%.0f tok/s' % d['target_tokens_per_s'], 'update kernels %.2f ms' % d['update_path_kernels_ms_per_step'])" || tail -5 /tmp/m.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --mode m2 --steps 6 --warmup 2 $F > /tmp/m2.log 2>&1; tail -1 /tmp/m2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W2 $F', round(d['ms_per_step'],2), '%.0f tok/s' % d['target_tokens_per_s'], d.get('exposed_comm',{}).get('ms'))" || tail -5 /tmp/m2.log
done
