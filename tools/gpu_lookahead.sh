mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/la_pytest.log 2>&1; echo "rc $?" >> gpurun_out/la_pytest.log
tail -3 gpurun_out/la_pytest.log
for la in 1 0 1; do
  SSSVD_LOOKAHEAD=$la timeout 400 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_la$la.json 2> gpurun_out/bench_la$la.err
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_la$la.json')); print('LA=$la', d['value'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['phase_tflops'], d['step_ms'])"
done
