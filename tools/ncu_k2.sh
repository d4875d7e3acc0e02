mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 -o gpurun_out/k2w_full -f python bench.py --steps 1 --warmup 0 --no-secondary > gpurun_out/ncu_k2w.log 2>&1
