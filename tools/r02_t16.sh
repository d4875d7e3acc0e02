mkdir -p gpurun_out
out=gpurun_out/t16.log
: > $out
timeout 300 python tools/quick_matrix.py 1 2 3 4 2>&1 | cut -c1-100,190-260 >> $out
timeout 1800 python -m pytest tests/test_variants_gpu.py tests/test_matrix_gpu.py tests/test_fullsize_ref_gpu.py tests/test_fullsize_gpu.py tests/test_adversarial_gpu.py tests/test_golden_gpu.py tests/test_edge_gpu.py -x -q -m gpu -k "matrix or adversarial or row_blocks or golden or edge" >> $out 2>&1
echo done >> $out
