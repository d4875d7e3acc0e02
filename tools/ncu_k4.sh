mkdir -p gpurun_out
python tools/quick_regions.py 1:101 3:200 3:2000 > gpurun_out/k4_quick.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_regions -c 1 -o gpurun_out/k4_full -f python tools/quick_regions.py 3:200 > gpurun_out/ncu_k4.log 2>&1
