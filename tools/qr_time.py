"""Device time of the tail QR (SSSVD_DEBUG prints it) at the tail's shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd
dev = sssvd.Device(0)
rng = np.random.default_rng(0)
for m, k in [(4096, 512), (512, 512), (1000, 128), (2000, 128), (8192, 512), (16384, 2048)]:
    a = rng.standard_normal((m, k))
    for _ in range(3):
        dev.thin_qr(a)
