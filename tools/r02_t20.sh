mkdir -p gpurun_out
out=gpurun_out/t20.log
: > $out
for v in "0 64 2" "1 64 2" "1 64 4" "1 32 4" "1 64 3" "1 32 8" "1 16 8"; do
  set -- $v
  echo "== SERP=$1 TR=$2 TC=$3" >> $out
  VISRT_K2W_SERP=$1 VISRT_K2W_TR=$2 VISRT_K2W_TC=$3 timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
done
for v in "0" "1"; do
  echo "== cfg3/cfg2 SERP=$v (defaults)" >> $out
  VISRT_K2W_SERP=$v timeout 300 python tools/quick_matrix.py 2 3 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
done
echo "== cfg3 SERP=1 TMORTON TR=2 TC=32 / 4x16" >> $out
VISRT_K2W_SERP=1 VISRT_K2W_TR=2 VISRT_K2W_TC=32 timeout 300 python tools/quick_matrix.py 3 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
VISRT_K2W_SERP=1 VISRT_K2W_TR=4 VISRT_K2W_TC=16 timeout 300 python tools/quick_matrix.py 3 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
echo done >> $out
