# round-2 final measurements: every -m gpu test, the default bench line (both arms), the bench
# launch list, ncu --set full of the headline kernel (K2w, the FULL config-4 launch), of the two K7
# kernels (config 3) and of the fused tree level (config 3), and every config's whole workload
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/f_pytest.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/f_pytest.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
echo "bench_rc=$?" >> gpurun_out/f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 900 python tools/workloads.py 1 2 3 4 5 > gpurun_out/f_workloads.jsonl 2> gpurun_out/f_workloads.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-secondary --cpu-seconds 1 > gpurun_out/f_ncu_launch.log 2>&1
python tools/prof_matrix.py 4 all 2 > gpurun_out/f_k2w4_stats.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 \
  -o gpurun_out/f_k2w4 -f python tools/prof_matrix.py 4 all 1 > gpurun_out/f_ncu_k2w4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_ -c 2 \
  -o gpurun_out/f_k7 -f python tools/quick_chains.py 3 > gpurun_out/f_ncu_k7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tree_last -s 1 -c 1 \
  -o gpurun_out/f_k6 -f python tools/quick_tree.py 3:3:50 > gpurun_out/f_ncu_k6.log 2>&1
echo done > gpurun_out/f_done.txt
