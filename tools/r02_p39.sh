# refine kernel MINB 2 (default) vs 3; config-3 workload wall with the reused region buffer
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:500:mix 3:200 > gpurun_out/p39_minb2.log 2>&1
timeout 600 python tools/workloads.py 3 > gpurun_out/p39_w3.jsonl 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K4R_MINB=3" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_regions.py 5:20:rx 5:500:mix 3:200 > gpurun_out/p39_minb3.log 2>&1
echo done
