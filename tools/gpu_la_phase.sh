mkdir -p gpurun_out
for la in 0 1 0 1; do
  SSSVD_LOOKAHEAD=$la timeout 300 python tools/time_phase.py 2 4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('LA=$la', d['cfg'], d['mode'], d['rep'], round(d['shifted_solves_s']*1e3,1), 'ms', round(d['solve_tflops'],2), 'TF/s wall', round(d['wall_s'],3))
"
done > gpurun_out/la_phase.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 1 -c 1 -o gpurun_out/ncu_zgemm_v0b python tools/zgemm_variants.py --reps 1 --shape 0 --variant 0 > gpurun_out/ncu_zgemm_b.log 2>&1
echo "ncu rc $?" >> gpurun_out/ncu_zgemm_b.log
cat gpurun_out/la_phase.txt; tail -1 gpurun_out/ncu_zgemm_b.log
