cp paper_1806_00187_b200/libsmpu.so /tmp/orig.so
for V in k4 k5 k6 k8; do
cp tmp_variants/libsmpu_$V.so paper_1806_00187_b200/libsmpu.so
python bench.py --config base --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V base graph=%.4f calls=%.4f k2=%.0f' % (d['ms_per_step'], d['graph']['ms_per_step_calls'], d['kernels']['k2_adam']['achieved_gbs']))"
python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V big graph=%.4f k2=%.0f' % (d['ms_per_step'], d['kernels']['k2_adam']['achieved_gbs']))"
done
cp /tmp/orig.so paper_1806_00187_b200/libsmpu.so
