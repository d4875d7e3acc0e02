mkdir -p gpurun_out
out=gpurun_out/t15.log
: > $out
for v in "1 32" "2 32" "1 16" "2 16" "1 64" "4 16"; do
  set -- $v
  echo "== cfg2 tiled TMORTON=1 TR=$1 TC=$2" >> $out
  VISRT_K2W_TILED=1 VISRT_K2W_TMORTON=1 VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 timeout 300 python tools/quick_matrix.py 2 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
for v in "1 32" "1 48" "1 64" "2 48"; do
  set -- $v
  echo "== cfg3 TMORTON=1 TR=$1 TC=$2" >> $out
  VISRT_K2W_TMORTON=1 VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 timeout 300 python tools/quick_matrix.py 3 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
echo done >> $out
