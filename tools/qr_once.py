"""One tail QR of the given shape (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_13655_b200 import sssvd
m, k = int(sys.argv[1]), int(sys.argv[2])
dev = sssvd.Device(0)
dev.thin_qr(np.random.default_rng(0).standard_normal((m, k)))
