set -x
mkdir -p gpurun_out
{
python tools/zgemm_probe.py 200 136 128 3 1 3,4,5,6
python tools/zgemm_probe.py 77 35 9 2 1 3,4,5,6
for rep in 1 2; do
python tools/zgemm_probe.py 16128 16256 256 2 5 2,3,4,5,6
python tools/zgemm_probe.py 3968 4000 128 8 10 2,3,4,5,6
python tools/zgemm_probe.py 3968 4000 64 8 10 2,3,4,5,6
python tools/zgemm_probe.py 3968 4000 32 8 10 2,3,4,5,6
done
} > gpurun_out/3m_regs.jsonl 2>&1
for z in 3m 3m8 3m244 3m248; do
  SSSVD_ZGEMM=$z python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/3mr_bench2_$z.jsonl 2> gpurun_out/3mr_bench2_$z.err
  SSSVD_ZGEMM=$z python bench.py --config 4 --steps 3 --no-cpu-baseline > gpurun_out/3mr_bench4_$z.jsonl 2> gpurun_out/3mr_bench4_$z.err
done
