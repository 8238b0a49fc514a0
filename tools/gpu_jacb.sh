mkdir -p gpurun_out
for b in 8 4 6 3; do
  echo "== b=$b"
  SSSVD_JACOBI_B=$b SSSVD_DEBUG=1 timeout 300 python tools/phase_ab.py 2 --reps 3 2>&1 | grep -E "jacobi kernel|jacobi_svd k|run_ms" | tail -12 | cut -c1-200
done
