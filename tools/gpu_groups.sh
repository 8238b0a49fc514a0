mkdir -p gpurun_out
for c in 2 4 3; do for g in 4 8 6; do
  SSSVD_GROUPS=$g timeout 600 python tools/phase_ab.py $c --reps 4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    ph=sorted(d['phase_ms']); print('cfg $c G=$g', 'mode', d['mode'], 'median', round(d['phase_ms_median'],1), 'min', ph[0], 'max', ph[-1], 'run_med', round(d['run_ms_median'],1))
"
done; done
for g in 4 8; do
  SSSVD_GROUPS=$g timeout 900 python tools/phase_ab.py 5 --reps 1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('cfg 5 G=$g', 'mode', d['mode'], 'phase', round(d['phase_ms_median'],1), 'run', round(d['run_ms_median'],1))
"
done
