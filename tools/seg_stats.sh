mkdir -p gpurun_out
VISRT_NVCC_FLAGS="-DVISRT_SEG_STATS" python paper_2501_02747_b200/build.py --force > gpurun_out/ss_build.log 2>&1
python tools/seg_stats.py 2 > gpurun_out/seg_stats.log 2>&1
python tools/seg_stats.py 3 >> gpurun_out/seg_stats.log 2>&1
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_trajectory_gpu.py tests/test_regions_gpu.py -x -q -m gpu >> gpurun_out/seg_stats.log 2>&1
