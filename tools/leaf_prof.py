import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SSSVD_LEAF_PROF"] = "1"
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = workloads.CONFIGS[c]
a, _ = workloads.make_operator(c)
dev = sssvd.Device(0)
cfg = sssvd.RunConfig(w.a, w.b, mode=w.modes[-1], params=sssvd.SsParams(block_size=w.L, moment_degree=w.M, quadrature_count=w.N), gram_cap=1 << 30)
L = sssvd.lib()
out = (ctypes.c_uint64 * 7)()
sssvd.run_solve(a, cfg, dev)
L.sssvd_debug_leaf_profile(out)
cols = max(out[4], 1)
print("cycles/column: search+argmax %.0f | fold+publish+cluster barrier %.0f | DSMEM winner+rows %.0f | swap+update %.0f | columns %d"
      % (out[0] / cols, out[1] / cols, out[2] / cols, out[3] / cols, out[4]))
print("cycles/leaf (CTA lifetime): %.0f over %d leaves; column loop share %.0f%%"
      % (out[5] / max(out[6], 1), out[6], 100 * (out[0] + out[1] + out[2] + out[3]) / max(out[5], 1)))
