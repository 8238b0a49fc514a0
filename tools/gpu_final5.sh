mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?" >> gpurun_out/bench_ref.err
tail -n 2 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log
for f in bench bench_b; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['e2e']['value'], d['step_ms'], d['e2e']['step_ms'], d['e2e']['parts_ms'], d['roofline']['achieved'], d['roofline']['phase_tflops'], d['clocks'])"; done
cat gpurun_out/bench_ref.json
