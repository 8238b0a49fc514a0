"""Times the trailing-update GEMM on one shape through sssvd_debug_zgemm (variant 0 = 4-product
cp.async kernel, 1 = its TMA form, 2 = the 3-product (3M) kernel, the library default) and reports
TF/s in 8 M N K units and the check against variant 0; under ncu it is the capture target.
    python tools/zgemm_probe.py [M N K batch reps variants]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13655_b200 import sssvd  # noqa: E402

args = [int(x) for x in sys.argv[1:6]] if len(sys.argv) > 5 else [3968, 4000, 128, 8, 5]
variants = [int(v) for v in sys.argv[6].split(",")] if len(sys.argv) > 6 else [0, 1, 2]
m, n, k, b, reps = args
dev = sssvd.Device(0)
for v in variants:
    ms, mism = ctypes.c_double(), ctypes.c_int64()
    dev.check(sssvd.lib().sssvd_debug_zgemm(dev.h, v, m, n, k, b, reps, ctypes.byref(ms), ctypes.byref(mism)))
    print(json.dumps({"variant": v, "M": m, "N": n, "K": k, "batch": b, "ms": ms.value,
                      "tflops": 8.0 * m * n * k * b / (ms.value * 1e-3) / 1e12, "mismatches": mism.value}), flush=True)
