mkdir -p gpurun_out
for g in 1 0; do VISRT_K2W_GROUPED=$g python tools/quick_matrix.py 4 > gpurun_out/k2g_$g.log 2>&1; done
python tools/quick_matrix.py 2 3 >> gpurun_out/k2g_1.log 2>&1
