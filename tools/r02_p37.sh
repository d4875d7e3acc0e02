# fused tree level: parents per grab 4 (default) vs 1 vs 8
mkdir -p gpurun_out
timeout 300 python tools/quick_tree.py 3:3:50 5:3:200 1:2:100 > gpurun_out/p37_grab4.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "tree or trace" > gpurun_out/p37_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p37_pytest.log
VISRT_NVCC_FLAGS="-DVISRT_K6L_GRAB=1" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_tree.py 3:3:50 5:3:200 > gpurun_out/p37_grab1.log 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K6L_GRAB=8" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_tree.py 3:3:50 5:3:200 > gpurun_out/p37_grab8.log 2>&1
echo done
