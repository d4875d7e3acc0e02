# dense (P0, normal) table for the tree's plane tests
mkdir -p gpurun_out
timeout 300 python tools/quick_tree.py 3:3:50 5:3:200 1:2:100 > gpurun_out/p32_tree.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "tree or trace or aux or dropin or resolve" > gpurun_out/p32_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p32_pytest.log
echo done
