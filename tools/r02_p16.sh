# refine fan re-filtering A/B (REFILL 6 default vs 0 vs 4)
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 1:101 > gpurun_out/p16_refill6.log 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K4W_REFILL=0" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 1:101 > gpurun_out/p16_refill0.log 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K4W_REFILL=4" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 1:101 > gpurun_out/p16_refill4.log 2>&1
echo done
