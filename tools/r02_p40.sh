# K7 stage counts (config 2, 3)
mkdir -p gpurun_out
VISRT_NVCC_FLAGS="-DVISRT_K7_STATS" python -m paper_2501_02747_b200.build --force > gpurun_out/p40_build.log 2>&1
timeout 300 python tools/k7_stats.py 2 3 > gpurun_out/p40_k7.log 2>&1
echo done
