"""Time svd_square (QR preconditioning + one-sided Jacobi): default kernel choice vs the grid
block kernel (SSSVD_JACOBI=grid) vs the scalar grid kernel (SSSVD_JACOBI=scalar), with SSSVD_DEBUG's kernel time and sweep count on stderr."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np
    from paper_2109_13655_b200 import sssvd
    dev = sssvd.Device(0)
    for k in [int(x) for x in sys.argv[2:]]:
        rng = np.random.default_rng(k)
        u, _ = np.linalg.qr(rng.standard_normal((k, k)))
        v, _ = np.linalg.qr(rng.standard_normal((k, k)))
        s = 10.0 ** (-17.0 * np.arange(k) / (k - 1))
        b = np.triu((u * s) @ v.T)
        for it in range(2):
            t0 = time.time()
            uu, ss, vv = dev.svd_square(b)
            dt = time.time() - t0
        ref = np.linalg.svd(b, compute_uv=False)
        err = float(np.max(np.abs(ss - ref) / (1e-9 * ref + 1e-14 * ref[0])))
        print(f"k={k} {os.environ.get('SSSVD_JACOBI', 'default')}: svd_square {dt * 1e3:.1f} ms, "
              f"sigma err/bound {err:.3f}, recon {np.linalg.norm(uu * ss @ vv.T - b) / np.linalg.norm(b):.2e}", flush=True)
else:
    ks = sys.argv[1:] or ["1024", "2048"]
    for meth in ["default", "grid", "scalar"]:
        env = dict(os.environ, SSSVD_DEBUG="1")
        if meth != "default":
            env["SSSVD_JACOBI"] = meth
        subprocess.run([sys.executable, __file__, "child"] + ks, env=env)
