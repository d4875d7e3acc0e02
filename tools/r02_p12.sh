mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 1:101 > gpurun_out/p12_regions.log 2>&1
echo done
