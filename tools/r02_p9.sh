# A/B: cone-list head in shared memory vs global only
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p9_smem.log 2>&1
VISRT_K4W_CONE_SMEM=0 timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p9_nosmem.log 2>&1
VISRT_K4W_CONE_SMEM=32 timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p9_smem32.log 2>&1
echo done
