# K6 fused last level: unfold_tail (default) vs unfold_one; MINB 2; tree tests
mkdir -p gpurun_out
timeout 300 python tools/quick_tree.py 3:3:50 5:3:200 1:2:100 > gpurun_out/p26_tail.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "tree or trace or aux or dropin" > gpurun_out/p26_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p26_pytest.log
VISRT_NVCC_FLAGS="-DVISRT_K6L_MINB=2" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_tree.py 3:3:50 5:3:200 > gpurun_out/p26_minb2.log 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K6L_TAIL=0" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_tree.py 3:3:50 5:3:200 1:2:100 > gpurun_out/p26_old.log 2>&1
echo done
