# ncu of the fused last tree level (config 3 order 3, 50 snapshots) after pn + lazy chains
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tree_last -c 1 -o gpurun_out/p31_k6 -f python tools/quick_tree.py 3:3:50 > gpurun_out/p31_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p31_k6.ncu-rep > gpurun_out/p31_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/p31_k6.ncu-rep 40 > gpurun_out/p31_lines.txt 2>&1
echo done
