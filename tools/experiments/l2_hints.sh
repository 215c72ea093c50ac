for H in 0 1 2; do
SMPU_L2_HINT=$H python paper_1806_00187_b200/_build.py > /dev/null 2>&1 || echo "build $H failed"
for r in 1 2; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/l2h_$H.json 2> gpurun_out/l2h_$H.err; tail -1 gpurun_out/l2h_$H.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hint=$H ms=%.4f calls=%.4f res=%.4f' % (d['ms_per_step'], d['graph']['ms_per_step_calls'], d['graph']['resident_microbatches']['ms_per_step']), {k:round(v['achieved_gbs']) for k,v in d['kernels'].items()})"
done; done
python paper_1806_00187_b200/_build.py > /dev/null 2>&1
