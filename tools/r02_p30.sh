# K2w slot-0 segments in shared memory: A/B
mkdir -p gpurun_out
timeout 600 python tools/quick_matrix.py 2 3 4 > gpurun_out/p30_segs.log 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K2W_SEGS=0" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 600 python tools/quick_matrix.py 2 3 4 > gpurun_out/p30_nosegs.log 2>&1
echo done
