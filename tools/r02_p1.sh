# round-2 session-3: K4w baseline timings + phase profile on config 5 (UAV Rx / train Tx)
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p1_regions.log 2>&1
VISRT_NVCC_FLAGS=-DVISRT_K4W_PROF python -m paper_2501_02747_b200.build --force > gpurun_out/p1_build.log 2>&1
timeout 300 python tools/k4w_prof.py 5:20:rx 5:20:tx > gpurun_out/p1_k4wprof.log 2>&1
echo done
