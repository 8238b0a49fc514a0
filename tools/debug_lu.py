import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd, workloads
dev = sssvd.Device(0)
rng = np.random.default_rng(0)
for n in [int(x) for x in sys.argv[1:]] or [2048, 3100, 4096, 6000, 8192]:
    g = rng.standard_normal((n, n)); g = (g + g.T) / 2 / np.sqrt(n)
    z = complex(0.3, 0.05)
    rhs = rng.standard_normal((n, 4)).astype(complex)
    t0 = time.time()
    x = sssvd.solve_block(sssvd.factor_shift(g, z), rhs)
    t = time.time() - t0
    Mz = -g + z * np.eye(n)
    r = np.linalg.norm(Mz @ x - rhs) / (np.linalg.norm(Mz, 'fro') * np.linalg.norm(x))
    print(json.dumps({"n": n, "berr": r, "xnorm": float(np.linalg.norm(x)), "t": t}), flush=True)
