# session-5: run-time K2w tile shapes on config 4 (no rebuilds), then the matrix tests
mkdir -p gpurun_out
out=gpurun_out/t12.log
: > $out
for v in "16 8 8" "16 4 8" "32 8 8" "32 4 8" "24 8 8" "16 8 6" "12 8 8" "16 6 8" "20 8 8" "16 12 8" "64 2 8" "32 2 8"; do
  set -- $v
  echo "== TR=$1 TC=$2 WCT=$3" >> $out
  VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 VISRT_K2W_WCT=$3 timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-120 >> $out
done
echo "== defaults" >> $out
timeout 300 python tools/quick_matrix.py 2 3 4 2>&1 | cut -c1-220 >> $out
timeout 1500 python -m pytest tests/test_variants_gpu.py tests/test_matrix_gpu.py tests/test_fullsize_ref_gpu.py tests/test_fullsize_gpu.py tests/test_adversarial_gpu.py -x -q -m gpu -k "matrix or adversarial or row_blocks" >> $out 2>&1
echo done >> $out
