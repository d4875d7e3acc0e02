mkdir -p gpurun_out
python tools/quick_tree.py 3:3:50 5:3:20 1:2:100 > gpurun_out/tree_q.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tree_launches.csv python tools/quick_tree.py 3:3:50 > gpurun_out/tree_ncu.log 2>&1
