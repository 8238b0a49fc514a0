mkdir -p gpurun_out
for shape in "4096 512" "512 512"; do
set -- $shape
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_launches_$1x$2.csv python tools/qr_launches.py $1 $2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/qr_launches_$1x$2.csv > gpurun_out/qr_launch_summary_$1x$2.txt 2>&1
cat gpurun_out/qr_launch_summary_$1x$2.txt
done
