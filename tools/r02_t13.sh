# session-5: K2w tiles over Morton positions
mkdir -p gpurun_out
out=gpurun_out/t13.log
: > $out
for v in "16 8 8" "8 8 8" "32 8 8" "16 16 8" "32 16 8" "8 16 8" "32 32 8" "64 8 8"; do
  set -- $v
  echo "== TMORTON=1 TR=$1 TC=$2 WCT=$3" >> $out
  VISRT_K2W_TMORTON=1 VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 VISRT_K2W_WCT=$3 timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
for v in "2 16" "4 8" "8 8" "16 8" "4 16"; do
  set -- $v
  echo "== cfg3/2 TMORTON=1 TR=$1 TC=$2" >> $out
  VISRT_K2W_TMORTON=1 VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 timeout 300 python tools/quick_matrix.py 3 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
for v in "128 1 8" "128 2 8" "64 1 8" "64 4 8" "256 1 8" "96 2 8" "64 2 6" "64 3 8" "48 2 8"; do
  set -- $v
  echo "== TR=$1 TC=$2 WCT=$3" >> $out
  VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 VISRT_K2W_WCT=$3 timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
for v in "64 2" "32 2" "16 2" "32 1" "8 4"; do
  set -- $v
  echo "== cfg3 TR=$1 TC=$2" >> $out
  VISRT_K2W_TR=$1 VISRT_K2W_TC=$2 timeout 300 python tools/quick_matrix.py 3 2>&1 | grep " all" | cut -c1-100,190-230 >> $out
done
echo done >> $out
