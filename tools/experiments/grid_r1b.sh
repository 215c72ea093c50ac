timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not 5200" 2>&1 | tail -2
for K2 in 0 2 4; do
SMPU_K2_CTAS_PER_SM=$K2 timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1
tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('K2=$K2 ms=%.3f path=%.0f k1add=%.0f k1first=%.0f k2=%.0f clocks=%s' % (d['ms_per_step'], d['path_hbm_gbs'], k['k1_add']['achieved_gbs'], k['k1_first']['achieved_gbs'], k['k2_adam']['achieved_gbs'], d['clocks']))"
SMPU_K2_CTAS_PER_SM=$K2 timeout 300 python bench.py --config base --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1
tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('base K2=$K2 ms=%.4f path=%.0f k2=%.0f k1first=%.0f' % (d['ms_per_step'], d['path_hbm_gbs'], k['k2_adam']['achieved_gbs'], k['k1_first']['achieved_gbs']))"
done
