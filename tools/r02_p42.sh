mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_triples -c 1 -o gpurun_out/p42_k7 -f python tools/quick_chains.py 3 > gpurun_out/p42_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/p42_k7.ncu-rep > gpurun_out/p42_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/p42_k7.ncu-rep 30 > gpurun_out/p42_lines.txt 2>&1
python tools/ncu_calib.py gpurun_out/p42_k7.ncu-rep k7_config3 "config3 order-2 chains, 93.4M candidate triples" > gpurun_out/p42_calib.json 2>&1
echo done
