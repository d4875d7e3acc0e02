mkdir -p gpurun_out
: > gpurun_out/k4c.log
for w in 0 1; do
  echo "== VISRT_K4_WARP=$w" >> gpurun_out/k4c.log
  VISRT_K4_WARP=$w python tools/quick_regions.py 1:101 3:200 >> gpurun_out/k4c.log 2>&1
done
timeout 900 python -m pytest tests/test_regions_gpu.py tests/test_tables_gpu.py tests/test_trajectory_gpu.py -x -q -m gpu >> gpurun_out/k4c.log 2>&1
