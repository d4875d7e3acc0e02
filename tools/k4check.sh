mkdir -p gpurun_out
: > gpurun_out/k4c.log
python tools/quick_regions.py 1:101 3:20 3:200 >> gpurun_out/k4c.log 2>&1
VISRT_K4_WARP=1 python tools/quick_regions.py 3:20 >> gpurun_out/k4c.log 2>&1
VISRT_K4_WARP=0 python tools/quick_regions.py 3:20 >> gpurun_out/k4c.log 2>&1
timeout 900 python -m pytest tests/test_regions_gpu.py tests/test_tables_gpu.py tests/test_trajectory_gpu.py tests/test_golden_gpu.py tests/test_fullsize_gpu.py -x -q -m gpu >> gpurun_out/k4c.log 2>&1
