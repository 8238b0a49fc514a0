#!/bin/bash
# bench.py repeated per shift-group count (SSSVD_GROUPS): value, GEMM-busy TF/s, phase TF/s
for g in "$@"; do
  for rep in 1 2 3; do
    SSSVD_GROUPS=$g timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gs_${g}_${rep}.log 2>&1
    python - "$g" "$rep" <<'PY'
import json, sys
g, rep = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open("gpurun_out/gs_%s_%s.log" % (g, rep)).read().strip().splitlines()[-1]); r = d["roofline"]
    print("G=%s rep=%s value=%.4f e2e=%.4f gemm=%.2f phase=%.2f" % (g, rep, d["value"], d["e2e"]["value"], r["achieved"], r["phase_tflops"]))
except Exception as e:
    print("G=%s rep=%s failed %s" % (g, rep, e))
PY
  done
done
