# Outer block (SSSVD_NB) and shift-group (SSSVD_GROUPS) sweep with the 3M trailing update
set -x
mkdir -p gpurun_out
for nb in 128 256; do for g in 4 8; do
  SSSVD_NB=$nb SSSVD_GROUPS=$g python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/sw_cfg2_nb${nb}_g$g.jsonl 2>/dev/null
  SSSVD_NB=$nb SSSVD_GROUPS=$g python bench.py --config 4 --steps 3 --no-cpu-baseline > gpurun_out/sw_cfg4_nb${nb}_g$g.jsonl 2>/dev/null
done; done
for g in 2 8; do
  SSSVD_GROUPS=$g python bench.py --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/sw_cfg5_nb256_g$g.jsonl 2>/dev/null
done
SSSVD_GROUPS=16 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/sw_cfg2_nb128_g16.jsonl 2>/dev/null
