for G in real exact zero real; do
timeout 300 python bench.py --generator $G --no-e2e --no-cpu-baseline > gpurun_out/gen_$G.json 2> gpurun_out/gen_$G.err; tail -1 gpurun_out/gen_$G.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$G', 'ms=%.4f calls=%.4f res=%.4f' % (d['ms_per_step'], d['graph']['ms_per_step_calls'], d['graph']['resident_microbatches']['ms_per_step']), {k:round(v['achieved_gbs']) for k,v in d['kernels'].items()}, d['config']['generator'])"
done
