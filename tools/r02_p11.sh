mkdir -p gpurun_out
VISRT_NVCC_FLAGS=-DVISRT_K4W_PROF python -m paper_2501_02747_b200.build --force > gpurun_out/p11_build.log 2>&1
timeout 300 python tools/k4w_prof.py 5:20:rx 5:20:tx > gpurun_out/p11_k4wprof.log 2>&1
echo done
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p11_regions.log 2>&1
