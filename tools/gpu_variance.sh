mkdir -p gpurun_out
for e in "X=0" "SSSVD_LEAF_C=16" "SSSVD_LEAF_W=8" "SSSVD_GROUPS=3" "SSSVD_GROUPS=8"; do
  env $e timeout 300 python tools/phase_ab.py 2 --reps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    ph=sorted(d['phase_ms']); print('$e', 'mode', d['mode'], 'median', round(d['phase_ms_median'],1), 'min', ph[0], 'max', ph[-1], 'mean', round(sum(ph)/len(ph),1), 'run_med', round(d['run_ms_median'],1))
"
done
