# occupancy A/B for K4w: MINB 2 (128 regs) vs 3 (85 regs)
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p13_minb2.log 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K4W_MINB=3" python -m paper_2501_02747_b200.build --force > gpurun_out/p13_build3.log 2>&1
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p13_minb3.log 2>&1
echo done
