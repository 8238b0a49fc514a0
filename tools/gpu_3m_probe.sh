# 3M trailing-update kernel: correctness vs the 4-product kernel on ragged shapes, isolated speed on the
# config-2 / config-5 shapes, then live phases (config 2, config 5) per kernel choice.
set -x
mkdir -p gpurun_out
{
for shape in "77 35 9 3 1" "130 67 301 2 1" "64 48 16 1 1" "1000 513 64 2 1" "33 96 40 5 1" "200 49 17 1 1"; do
  python tools/zgemm_probe.py $shape 0,2,3
done
python tools/zgemm_probe.py 3968 4000 128 8 5 0,2,3
python tools/zgemm_probe.py 16128 16256 256 1 5 0,2,3
python tools/zgemm_probe.py 8064 8256 256 4 5 0,2,3
python tools/zgemm_probe.py 2048 2176 128 8 5 0,2,3
python tools/zgemm_probe.py 3968 4000 64 8 5 0,2,3
python tools/zgemm_probe.py 3968 4000 32 8 5 0,2,3
} > gpurun_out/3m_probe.jsonl 2> gpurun_out/3m_probe.err
for z in 4m 3m 3m4; do
  SSSVD_ZGEMM=$z python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/3m_bench2_$z.jsonl 2> gpurun_out/3m_bench2_$z.err
done
for z in 3m 3m4; do
  SSSVD_ZGEMM=$z python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/3m_bench5_$z.jsonl 2> gpurun_out/3m_bench5_$z.err
done
