import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd
from oracle import sssvd_oracle as orc
dev = sssvd.Device(0)
rng = np.random.default_rng(1)
for n, L in [(8, 2), (33, 3), (40, 10), (64, 4), (100, 5), (130, 7), (300, 8), (1000, 16)]:
    g = rng.standard_normal((n, n)); g = (g + g.T) / 2
    z = complex(0.3, 0.5)
    rhs = rng.standard_normal((n, L))
    x = sssvd.solve_block(sssvd.factor_shift(g, z), rhs.astype(complex))
    xo = orc.ShiftedFactorization(g, z).solve(rhs)
    print(json.dumps({"n": n, "L": L, "relerr": float(np.linalg.norm(x - xo) / np.linalg.norm(xo))}), flush=True)
