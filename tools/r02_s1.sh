# round-2 session-2 baseline: every -m gpu test, the default bench line, the bench launch list,
# ncu --set full of the headline kernel (K2w config 4, every 61st pair) and of K4w (config-5 UAV Rx)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/s1_pytest.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/s1_pytest.log
timeout 900 python bench.py > gpurun_out/s1_bench.json 2> gpurun_out/s1_bench.err
echo "bench_rc=$?" >> gpurun_out/s1_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s1_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-secondary --cpu-seconds 1 > gpurun_out/s1_ncu_launch.log 2>&1
VISRT_K2_STRIDE=61 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 \
  -o gpurun_out/s1_k2w4 -f python tools/prof_matrix.py 4 all 1 > gpurun_out/s1_ncu_k2w4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 \
  -o gpurun_out/s1_k4w5 -f python tools/quick_regions.py 5:10:rx > gpurun_out/s1_ncu_k4w5.log 2>&1
echo done
