# heavy-first refine ordering; cone cap 1024 vs 2048; 500-source batches (the whole-workload batch size)
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 5:500:mix 3:200 > gpurun_out/p25_regions.log 2>&1
VISRT_K4W_CONE=2048 timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 5:500:mix > gpurun_out/p25_cap2048.log 2>&1
echo done
