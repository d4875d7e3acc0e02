# session-5: two-kernel K7 (screen + decide), row-block matrix entry point
mkdir -p gpurun_out
out=gpurun_out/t2.log
: > $out
timeout 300 python tools/quick_chains.py 1 2 3 >> $out 2>&1
timeout 900 python -m pytest tests/test_chains_gpu.py tests/test_variants_gpu.py tests/test_matrix_gpu.py -x -q -m gpu -k "chain or row_blocks or matrix" >> $out 2>&1
timeout 600 python -m pytest tests/test_fullsize_gpu.py tests/test_cpp_dropin.py -x -q -m gpu -k "chain or dropin" >> $out 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K7_SCREEN=0" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo "== SCREEN=0" >> $out
timeout 300 python tools/quick_chains.py 1 2 3 >> $out 2>&1
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
