timeout 1500 python -m pytest tests/test_gpu_multi.py -q 2>&1 | tail -3
for N in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N bench.py --gpus $N > gpurun_out/final_n$N.json 2> gpurun_out/final_n$N.err; echo "N=$N rc=$?"; tail -1 gpurun_out/final_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  value=%.4g ms=%.3f e2e=%.4g launches=%s exposed=%.3f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], d['exposed_comm']['ms']))"
done
timeout 400 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err; echo "N=1 rc=$?"; tail -1 gpurun_out/final_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  value=%.4g ms=%.3f e2e=%.4g launches=%s frac=%.3f cpu=%.3g' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], d['roofline']['frac'], d['cpu_baseline']['value']))"
