set -x
mkdir -p gpurun_out
for a in 1 2; do
  SSSVD_LEAF_ADAPT=$a timeout 600 python -m pytest tests/test_gpu_moments.py tests/test_gpu_solver.py -m gpu -q -x > gpurun_out/s9_tests_a$a.log 2>&1; echo "rc=$?" >> gpurun_out/s9_tests_a$a.log
done
for a in 0 1 2; do
  for c in 1 2 4 3; do
    SSSVD_LEAF_ADAPT=$a python tools/cfg_twice.py $c > gpurun_out/s9_cfg${c}_a$a.log 2>&1
  done
done
for a in 0 1 2; do
  SSSVD_LEAF_ADAPT=$a python tools/cfg_twice.py 5 > gpurun_out/s9_cfg5_a$a.log 2>&1
done
