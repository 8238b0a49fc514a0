"""Time the trailing-update GEMM variants (warp tiles 32x32 / 32x16 / 16x32 / 16x16) on the
shapes the LU issues, and check each is bitwise the 32x32 kernel. Usage:
    python tools/zgemm_variants.py [--reps 20] [--shape i] [--variant v]
Variant 10 is cuBLAS zgemmStridedBatched on the same data (a comparator, not the product path)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_13655_b200 import sssvd

SHAPES = [  # (label, M, N, K, batch)
    ("cfg2 block0 trailing (NB=128, 8 shifts)", 3968, 4000, 128, 8),
    ("cfg2 mid trailing", 2048, 2080, 128, 8),
    ("cfg2 late trailing", 512, 544, 128, 8),
    ("cfg2 panel node K=64", 4032, 64, 64, 8),
    ("cfg5 block0 trailing (NB=256, 2 shifts)", 16128, 16256, 256, 2),
    ("back-subst block K=128, N=L=32", 3968, 32, 128, 8),
]


def main():
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 20
    dev = sssvd.Device(0)
    L = sssvd.lib()
    only_shape = int(sys.argv[sys.argv.index("--shape") + 1]) if "--shape" in sys.argv else None
    only_var = int(sys.argv[sys.argv.index("--variant") + 1]) if "--variant" in sys.argv else None
    for si, (label, m, n, k, b) in enumerate(SHAPES):
        if only_shape is not None and si != only_shape:
            continue
        for v in range(11):
            if only_var is not None and v != only_var:
                continue
            ms = ctypes.c_double()
            mism = ctypes.c_int64()
            dev.check(L.sssvd_debug_zgemm(dev.h, v, m, n, k, b, reps, ctypes.byref(ms), ctypes.byref(mism)))
            tf = 8.0 * m * n * k * b / (ms.value * 1e-3) / 1e12
            print(json.dumps({"shape": label, "M": m, "N": n, "K": k, "batch": b, "variant": v,
                              "ms": round(ms.value, 4), "tflops": round(tf, 2), "frac_37.1": round(tf / 37.1, 3),
                              "mismatches_vs_v0": mism.value}), flush=True)


if __name__ == "__main__":
    main()
