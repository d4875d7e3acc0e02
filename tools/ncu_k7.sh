mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_triples -c 1 -o gpurun_out/k7_full -f python tools/quick_chains.py 3 > gpurun_out/ncu_k7.log 2>&1
