# i-cache test: out-of-line seg_hits; scan-only timing (refine skipped)
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p17_segni.log 2>&1
VISRT_K4W_FAN=2 timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx > gpurun_out/p17_norefine.log 2>&1
echo done
