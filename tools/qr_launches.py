"""One thin_qr call (debug ABI) for a per-kernel launch list under ncu:
    ncu --metrics gpu__time_duration.sum --csv python tools/qr_launches.py 16384 2048"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd
m, k = int(sys.argv[1]), int(sys.argv[2])
dev = sssvd.Device(0)
a = np.random.default_rng(1).standard_normal((m, k))
dev.thin_qr(a)
