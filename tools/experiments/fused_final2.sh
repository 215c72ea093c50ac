timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -3
for C in big_ende base; do
timeout 300 python bench.py --config $C --no-e2e --no-cpu-baseline > gpurun_out/ff2_$C.json 2> gpurun_out/ff2_$C.err; echo "$C rc=$?"; tail -1 gpurun_out/ff2_$C.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' ms=%.4f calls=%.4f res=%.4f launches=%s roof=%s %.3f' % (d['ms_per_step'], d['graph']['ms_per_step_calls'], d['graph']['resident_microbatches']['ms_per_step'], d['gpu_launches'], d['roofline']['kernel'], d['roofline']['frac'])); print(' ', {k:(round(v['avg_us'],1), round(v['achieved_gbs'])) for k,v in d['kernels'].items()})"
done
