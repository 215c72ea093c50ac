for K1 in 4 0; do for K2 in 2 0; do
SMPU_K1_CTAS_PER_SM=$K1 SMPU_K2_CTAS_PER_SM=$K2 timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1
tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('K1=$K1 K2=$K2 ms=%.3f path=%.0f k1add=%.0f k1first=%.0f k2=%.0f clocks=%s' % (d['ms_per_step'], d['path_hbm_gbs'], k['k1_add']['achieved_gbs'], k['k1_first']['achieved_gbs'], k['k2_adam']['achieved_gbs'], d['clocks']))"
done; done
for K2 in 2 0; do
SMPU_K2_CTAS_PER_SM=$K2 timeout 300 python bench.py --config base --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > /tmp/b.log 2>&1
tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('base K2=$K2 ms=%.4f path=%.0f k2=%.0f k1first=%.0f' % (d['ms_per_step'], d['path_hbm_gbs'], k['k2_adam']['achieved_gbs'], k['k1_first']['achieved_gbs']))"
done
