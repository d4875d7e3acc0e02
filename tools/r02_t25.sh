mkdir -p gpurun_out
timeout 300 python tools/quick_chains.py 1 3 > gpurun_out/t25.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_ -c 3 -o gpurun_out/f_k7 -f python tools/quick_chains.py 3 > gpurun_out/f_ncu_k7.log 2>&1
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
echo "bench_rc=$?" >> gpurun_out/f_bench.err
timeout 300 python tools/workloads.py 3 > gpurun_out/t25_workloads3.jsonl 2>> gpurun_out/t25.log
