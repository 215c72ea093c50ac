timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not 5200 and not 2_31" 2>&1 | tail -2
for P in 0 1; do
SMPU_PDL=$P python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=$P big graph=%.4f calls=%.4f resident=%.4f k1add=%.0f k2=%.0f' % (d['ms_per_step'], d['graph']['ms_per_step_calls'], d['graph']['resident_microbatches']['ms_per_step'], d['kernels']['k1_add']['achieved_gbs'], d['kernels']['k2_adam']['achieved_gbs']))"
SMPU_PDL=$P python bench.py --config base --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=$P base graph=%.4f calls=%.4f' % (d['ms_per_step'], d['graph']['ms_per_step_calls']))"
done
