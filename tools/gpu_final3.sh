mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
timeout 1500 python tools/scale_estimate.py --config 5 > gpurun_out/scale_cfg5.jsonl 2> gpurun_out/scale_cfg5.err; echo "scale rc $?" >> gpurun_out/scale_cfg5.err
tail -n 3 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log; cat gpurun_out/bench.json; cat gpurun_out/scale_cfg5.jsonl; tail -2 gpurun_out/scale_cfg5.err
