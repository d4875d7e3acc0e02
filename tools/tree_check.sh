mkdir -p gpurun_out
python tools/quick_tree.py 3:3:50 5:3:20 1:2:100 > gpurun_out/tree_q2.log 2>&1
timeout 900 python -m pytest tests/test_tree_gpu.py tests/test_golden_gpu.py tests/test_aux_gpu.py tests/test_fullsize_gpu.py -x -q -m gpu >> gpurun_out/tree_q2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tree_launches2.csv python tools/quick_tree.py 3:3:50 > gpurun_out/tree_ncu2.log 2>&1
