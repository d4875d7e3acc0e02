# config-4 (B) matrix and config-5 region profiles (timings + one ncu capture each)
mkdir -p gpurun_out
python tools/quick_matrix.py 4 > gpurun_out/qm4.log 2>&1
python tools/quick_regions.py 5:20:tx 5:20:rx 5:20:mix > gpurun_out/qr5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 -o gpurun_out/k2w4_full -f python tools/prof_matrix.py 4 all 1 > gpurun_out/ncu_k2w4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 -o gpurun_out/k4w5rx_full -f python tools/quick_regions.py 5:10:rx > gpurun_out/ncu_k4w5rx.log 2>&1
