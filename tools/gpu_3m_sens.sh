set -x
mkdir -p gpurun_out
for c in 1 2 4; do
for z in 4m 3m; do
  SSSVD_ZGEMM=$z python tools/m3_sensitivity.py $c /tmp/blocks_${c}_$z > gpurun_out/sens_${c}_$z.log 2>&1
done
python - <<PY > gpurun_out/sens_${c}_diff.log 2>&1
import numpy as np, glob
for f in sorted(glob.glob("/tmp/blocks_${c}_4m_m*.npz")):
    a=np.load(f); b=np.load(f.replace("_4m_","_3m_"))
    print(f, [float(np.linalg.norm(a[k]-b[k])/np.linalg.norm(a[k])) for k in a.files][:6])
PY
done
ncu --set full --clock-control none --import-source on -k regex:zgemm3m_kernel -s 1 -c 1 -o gpurun_out/3m_zgemm_cfg5 -f python tools/zgemm_probe.py 16128 16256 256 2 2 2 > gpurun_out/3m_ncu.log 2>&1
