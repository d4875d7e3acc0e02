# K7 compact buffers: A/B vs wide buffers (sha of all triples), ncu DRAM traffic
mkdir -p gpurun_out
timeout 300 python tools/quick_chains.py 1 2 3 > gpurun_out/p22_compact.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,local_load_inst,smsp__inst_executed.sum --clock-control none -k regex:k_chain_triples --csv --log-file gpurun_out/p22_ncu_compact.csv python tools/quick_chains.py 3 > /dev/null 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K7_COMPACT=0" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 300 python tools/quick_chains.py 1 2 3 > gpurun_out/p22_wide.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_chain_triples --csv --log-file gpurun_out/p22_ncu_wide.csv python tools/quick_chains.py 3 > /dev/null 2>&1
echo done
python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
VISRT_K2_STRIDE=61 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 \
  -o gpurun_out/p22_k2w4 -f python tools/prof_matrix.py 4 all 1 > gpurun_out/p22_ncu_k2w4.log 2>&1
python tools/ncu_summary.py gpurun_out/p22_k2w4.ncu-rep > gpurun_out/p22_k2w4_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/p22_k2w4.ncu-rep 60 > gpurun_out/p22_k2w4_lines.txt 2>&1
echo done2
