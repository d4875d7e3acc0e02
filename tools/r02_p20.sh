# ncu --set full of the K4w refine kernel (config-5 Rx, 10 snapshots)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_region_refine -c 1 \
  -o gpurun_out/p20_refine -f python tools/quick_regions.py 5:10:rx > gpurun_out/p20_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p20_refine.ncu-rep > gpurun_out/p20_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/p20_refine.ncu-rep 45 > gpurun_out/p20_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 \
  -o gpurun_out/p20_scan -f python tools/quick_regions.py 5:10:rx > gpurun_out/p20_ncu2.log 2>&1
python tools/ncu_summary.py gpurun_out/p20_scan.ncu-rep >> gpurun_out/p20_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/p20_scan.ncu-rep 45 > gpurun_out/p20_scan_lines.txt 2>&1
echo done
