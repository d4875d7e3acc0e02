# K2w tiled launches: 6-entry warp cache (default) vs 4
mkdir -p gpurun_out
timeout 600 python tools/quick_matrix.py 3 4 > gpurun_out/p29_wc6.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "matrix or variants" > gpurun_out/p29_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p29_pytest.log
VISRT_NVCC_FLAGS="-DVISRT_K2W_WC_TILED=4" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 600 python tools/quick_matrix.py 3 4 > gpurun_out/p29_wc4.log 2>&1
echo done
