# K1 row tiles vs cub selection: (A) matrices + candidate-list tests
mkdir -p gpurun_out
timeout 600 python tools/quick_matrix.py 1 2 3 4 > gpurun_out/p36_rows.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "matrix or cand or prefilter or fullsize or dropin or cache" > gpurun_out/p36_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p36_pytest.log
VISRT_NVCC_FLAGS="-DVISRT_K1_ROWS=0" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 600 python tools/quick_matrix.py 1 2 3 4 > gpurun_out/p36_cub.log 2>&1
echo done
