mkdir -p gpurun_out
out=gpurun_out/t21.log
: > $out
for v in "1 128 4 8" "1 96 4 8" "1 48 4 8" "1 64 5 8" "1 64 6 8" "1 64 4 6" "1 64 4 10" "1 24 4 8"; do
  set -- $v
  echo "== SERP=$1 TR=$2 TC=$3 WCT=$4" >> $out
  VISRT_K2W_SERP=$1 VISRT_K2W_TR=$2 VISRT_K2W_TC=$3 VISRT_K2W_WCT=$4 timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
done
echo done >> $out
