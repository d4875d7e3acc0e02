mkdir -p gpurun_out
out=gpurun_out/t14.log
: > $out
for v in "64 2 8" "96 2 8" "32 2 8" "32 4 8" "64 4 8" "128 2 8"; do
  set -- $v
  echo "== TMORTON=1 TR=$1 TC=$2 WCT=$3" >> $out
  VISRT_K2W_TMORTON=1 VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 VISRT_K2W_WCT=$3 timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
for v in "2 16" "2 32" "1 32" "3 16" "2 24" "2 8" "1 16"; do
  set -- $v
  echo "== cfg3 TMORTON=1 TR=$1 TC=$2" >> $out
  VISRT_K2W_TMORTON=1 VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 timeout 300 python tools/quick_matrix.py 3 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
echo "== cfg2 tiled forced, morton 2x16 vs default rows" >> $out
VISRT_K2W_TILED=1 VISRT_K2W_TMORTON=1 timeout 300 python tools/quick_matrix.py 2 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
VISRT_K2W_TILED=1 timeout 300 python tools/quick_matrix.py 2 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
timeout 300 python tools/quick_matrix.py 2 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
echo done >> $out
