# ncu --set full of K4w on config-5 UAV Rx (10 snapshots) with the cone lists
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 \
  -o gpurun_out/p5_k4w5 -f python tools/quick_regions.py 5:10:rx > gpurun_out/p5_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p5_k4w5.ncu-rep > gpurun_out/p5_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/p5_k4w5.ncu-rep 60 > gpurun_out/p5_lines.txt 2>&1
echo done
