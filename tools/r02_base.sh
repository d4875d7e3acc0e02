# round-2 baseline: fixture parity that exists so far, config-4 headline bench,
# ncu captures of the headline (K2w config 4) and the table kernel (K4w config 5)
mkdir -p gpurun_out
python -m pytest tests/test_fullsize_ref_gpu.py -x -q > gpurun_out/r02_pt_full.log 2>&1
python bench.py --steps 5 --warmup 3 --no-secondary --cpu-seconds 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python tools/quick_regions.py 5:20:tx 5:20:rx > gpurun_out/r02_qr5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 -o gpurun_out/r02_k2w4_base -f python tools/prof_matrix.py 4 all 1 > gpurun_out/r02_ncu_k2w4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_point_regions_warp -c 1 -o gpurun_out/r02_k4w5_base -f python tools/quick_regions.py 5:10:rx > gpurun_out/r02_ncu_k4w5.log 2>&1
