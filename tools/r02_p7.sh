# K4w scan split + ncu of the shrunk kernel (config-5 Rx, 10 snapshots)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 \
  -o gpurun_out/p7_k4w5 -f python tools/quick_regions.py 5:10:rx > gpurun_out/p7_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p7_k4w5.ncu-rep > gpurun_out/p7_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/p7_k4w5.ncu-rep 50 > gpurun_out/p7_lines.txt 2>&1
VISRT_NVCC_FLAGS=-DVISRT_K4W_PROF python -m paper_2501_02747_b200.build --force > gpurun_out/p7_build.log 2>&1
timeout 300 python tools/k4w_prof.py 5:20:rx 5:20:tx > gpurun_out/p7_k4wprof.log 2>&1
echo done
