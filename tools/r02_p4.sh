# phase profiles: K4w (config 5 Rx/Tx) refine split, K2w (configs 2, 4)
mkdir -p gpurun_out
VISRT_NVCC_FLAGS="-DVISRT_K4W_PROF -DVISRT_K2W_PROF" python -m paper_2501_02747_b200.build --force > gpurun_out/p4_build.log 2>&1
timeout 300 python tools/k4w_prof.py 5:20:rx 5:20:tx > gpurun_out/p4_k4wprof.log 2>&1
timeout 300 python tools/k2w_prof.py 2 4 > gpurun_out/p4_k2wprof.log 2>&1
echo done
