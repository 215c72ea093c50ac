timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "sharded" 2>&1 | tail -2
for N in 2 4; do for O in auto replicated; do for M in m1 m2; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2981$N bench.py --gpus $N --optimizer $O --mode $M > gpurun_out/sd_${N}_${O}_${M}.json 2> gpurun_out/sd_${N}_${O}_${M}.err; echo "N=$N opt=$O mode=$M rc=$?"; tail -1 gpurun_out/sd_${N}_${O}_${M}.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  value=%.4g ms=%.3f e2e=%s opt=%s launches=%s' % (d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'), d['config'].get('optimizer'), d.get('gpu_launches')))"
done; done; done
