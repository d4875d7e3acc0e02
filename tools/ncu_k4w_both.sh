mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 -o gpurun_out/k4w5_full -f python tools/quick_regions.py 5:20 > gpurun_out/ncu_k4w5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 -o gpurun_out/k4w3_full -f python tools/quick_regions.py 3:200 > gpurun_out/ncu_k4w3.log 2>&1
