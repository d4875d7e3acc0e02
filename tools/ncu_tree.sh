mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tree_last -c 1 -o gpurun_out/k6last_full -f python tools/quick_tree.py 3:3:50 > gpurun_out/ncu_k6.log 2>&1
