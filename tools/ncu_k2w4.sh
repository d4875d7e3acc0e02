# config-4 (B) K2w: ncu full capture on every 61st pair (VISRT_K2_STRIDE; the full launch is ~1.7 s)
mkdir -p gpurun_out
VISRT_K2_STRIDE=61 python tools/prof_matrix.py 4 all 2 > gpurun_out/k2w4_stride.log 2>&1
VISRT_K2_STRIDE=61 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 -o gpurun_out/k2w4_full -f python tools/prof_matrix.py 4 all 1 > gpurun_out/ncu_k2w4.log 2>&1
