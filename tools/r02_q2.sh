# adversarial culling stress test + K2w config-4 ncu (stride 61: every 61st pair), streamed and quantised
mkdir -p gpurun_out
python -m pytest tests/test_adversarial_gpu.py -x -q > gpurun_out/r02_q2_adv.log 2>&1
VISRT_K2_STRIDE=61 python tools/prof_matrix.py 4 all 1 > gpurun_out/r02_q2_k2w4s.log 2>&1 && \
VISRT_K2_STRIDE=61 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 -o gpurun_out/r02_k2w4_stream -f python tools/prof_matrix.py 4 all 1 > gpurun_out/r02_q2_ncu1.log 2>&1
VISRT_QUANT=1 VISRT_K2_STRIDE=61 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 -o gpurun_out/r02_k2w4_quant -f python tools/prof_matrix.py 4 all 1 > gpurun_out/r02_q2_ncu2.log 2>&1
