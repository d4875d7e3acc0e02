# K2w slot-major settling: matrix timings + sha (configs 2, 3, 4), matrix tests; K4w back to global cone lists
mkdir -p gpurun_out
timeout 600 python tools/quick_matrix.py 2 3 4 > gpurun_out/p10_matrix.log 2>&1
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 > gpurun_out/p10_regions.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "matrix or variants or adversarial" > gpurun_out/p10_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/p10_pytest.log
echo done
