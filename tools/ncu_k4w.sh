mkdir -p gpurun_out
VISRT_K4_WARP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 -o gpurun_out/k4w_full -f python tools/quick_regions.py 3:200 > gpurun_out/ncu_k4w.log 2>&1
