"""Measure the FP64 roofline denominators on one B200 (run under gpurun).

MEASURED_PEAKS.json carries HBM and bf16 only. This script records, with CUDA events:
  * cuBLAS DGEMM 8192^3 (torch.matmul float64): burst (best of 10) and sustained (4 s loop);
  * cuBLAS ZGEMM 4096^3 (complex128) burst, counted as 8 n^3 real flops;
  * cuSOLVER ZGETRF (torch.linalg.lu_factor, complex128) at n=4096 / 8192, counted 8n^3/3,
    the library figure the hand-written LU is compared against (not used by the product);
  * the DMMA / DFMA issue-rate probes from tools/fp64_peak (hand-written, see that file).
Writes gpurun_out/fp64_peaks.json.
"""
import json, os, subprocess, time
import torch

def ev_time(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize(); s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best

def main():
    os.makedirs("gpurun_out", exist_ok=True)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                            "clocks_event_reasons.active,clocks_event_reasons.sw_power_cap",
                            "--format=csv", "-lms", "200"], stdout=open("gpurun_out/fp64_clocks.csv", "w"))
    out = {"gpu": torch.cuda.get_device_name(0)}
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
    torch.matmul(a, b); torch.cuda.synchronize()
    t = ev_time(lambda: torch.matmul(a, b), 10)
    out["dgemm_8192_burst_tflops"] = 2 * n**3 / t / 1e12
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record(); cnt = 0; t0 = time.time()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b); cnt += 1
        if cnt % 4 == 0: torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    out["dgemm_8192_sustained_tflops"] = 2 * n**3 * cnt / (s.elapsed_time(e) / 1e3) / 1e12
    del a, b
    n = 4096
    za = torch.randn(n, n, dtype=torch.complex128, device="cuda"); zb = torch.randn_like(za)
    torch.matmul(za, zb)
    t = ev_time(lambda: torch.matmul(za, zb), 10)
    out["zgemm_4096_burst_tflops"] = 8 * n**3 / t / 1e12
    for n in (4096, 8192):
        z = torch.randn(n, n, dtype=torch.complex128, device="cuda")
        torch.linalg.lu_factor(z)
        t = ev_time(lambda: torch.linalg.lu_factor(z), 3)
        out[f"cusolver_zgetrf_{n}_s"] = t
        out[f"cusolver_zgetrf_{n}_tflops"] = 8 * n**3 / 3 / t / 1e12
        del z
    torch.cuda.synchronize()
    probe = subprocess.run(["./tools/fp64_peak"], capture_output=True, text=True)
    try:
        out["probe"] = json.loads(probe.stdout)
    except Exception:
        out["probe_raw"] = probe.stdout + probe.stderr
    smi.terminate()
    json.dump(out, open("gpurun_out/fp64_peaks.json", "w"), indent=1)
    print(json.dumps(out))

if __name__ == "__main__":
    main()
