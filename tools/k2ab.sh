# A/B of the K2 variants (lane-per-pair vs warp-per-pair): timings + parity tests with each.
mkdir -p gpurun_out
out=gpurun_out/k2ab.log
: > $out
for w in 0 1; do
  echo "== VISRT_K2_WARP=$w" >> $out
  VISRT_K2_WARP=$w python tools/quick_matrix.py 1 2 3 >> $out 2>&1
  VISRT_K2_WARP=$w timeout 600 python -m pytest tests/test_matrix_gpu.py tests/test_golden_gpu.py -x -q -m gpu >> $out 2>&1
done
VISRT_K2_WARP=1 VISRT_FORCE_STREAM=1 python tools/quick_matrix.py 2 >> $out 2>&1
