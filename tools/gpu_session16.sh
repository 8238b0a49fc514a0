set -x
mkdir -p gpurun_out
rm -f /tmp/gemm5.txt /tmp/gemm5g1.txt
SSSVD_GEMM_DUMP=/tmp/gemm5.txt python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s16_bench5.jsonl 2> gpurun_out/s16_bench5.err
python tools/gemm_timeline.py /tmp/gemm5.txt > gpurun_out/s16_timeline_cfg5.txt 2>&1
tail -n 20000 /tmp/gemm5.txt | gzip > gpurun_out/s16_gemm5_tail.txt.gz
rm -f /tmp/gemm2.txt
SSSVD_GEMM_DUMP=/tmp/gemm2.txt python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s16_bench2.jsonl 2> gpurun_out/s16_bench2.err
python tools/gemm_timeline.py /tmp/gemm2.txt > gpurun_out/s16_timeline_cfg2.txt 2>&1
