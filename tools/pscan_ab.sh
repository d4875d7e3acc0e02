# A/B of the K4w column scan: serial col_vis (PSCAN=0) vs lane-parallel scan (PSCAN=1), with output hashes.
mkdir -p gpurun_out
: > gpurun_out/pscan.log
for cfg in "-DVISRT_K4W_NI=0" "-DVISRT_K4W_NI=1"; do
  VISRT_NVCC_FLAGS="$cfg" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
  echo "== $cfg" >> gpurun_out/pscan.log
  timeout 300 python tools/quick_regions.py 1:101 3:200 5:20 >> gpurun_out/pscan.log 2>&1
  timeout 300 python tools/quick_traj.py 3:1:1000 3:2:200 >> gpurun_out/pscan.log 2>&1
done
timeout 900 python -m pytest tests/test_regions_gpu.py tests/test_tables_gpu.py tests/test_trajectory_gpu.py tests/test_fullsize_gpu.py -x -q -m gpu >> gpurun_out/pscan.log 2>&1
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
