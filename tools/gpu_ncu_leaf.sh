# one ncu --set full capture (source-level) of the panel leaf LU kernel and of the fused
# panel-prep kernel on config 2 (NT on), after the plain run exits 0
mkdir -p gpurun_out
timeout 300 python tools/profile_once.py 2 1 > gpurun_out/leaf_plain.log 2>&1; echo "plain rc $?" >> gpurun_out/leaf_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_lu_v3 -s 40 -c 1 -o gpurun_out/ncu_leaf python tools/profile_once.py 2 1 > gpurun_out/ncu_leaf.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu_leaf.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_prep2 -s 40 -c 1 -o gpurun_out/ncu_prep python tools/profile_once.py 2 1 > gpurun_out/ncu_prep.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu_prep.log
tail -2 gpurun_out/leaf_plain.log gpurun_out/ncu_leaf.log gpurun_out/ncu_prep.log
