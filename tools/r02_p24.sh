# K6 ncu (config 3 order-3 trees) + whole workloads of configs 1, 3, 5 (device + wall)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tree_last -c 1 -o gpurun_out/p24_k6 -f python tools/quick_tree.py 3:3:50 > gpurun_out/p24_ncu_k6.log 2>&1
timeout 1500 python tools/workloads.py 1 3 5 > gpurun_out/p24_workloads.jsonl 2> gpurun_out/p24_workloads.err
echo done
