mkdir -p gpurun_out
out=gpurun_out/t17.log
: > $out
for h in 0 1; do
  echo "== HOMEAIM=$h (64x2)" >> $out
  VISRT_K2W_HOMEAIM=$h timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
  echo "== HOMEAIM=$h 2x64" >> $out
  VISRT_K2W_HOMEAIM=$h VISRT_K2W_TR=2 VISRT_K2W_TC=64 timeout 300 python tools/quick_matrix.py 4 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
done
for v in "-DVISRT_K2W_PRI=1" "-DVISRT_K2W_MULTI=1" "-DVISRT_K2W_HISLOT=1" "-DVISRT_K2W_ROT=0"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  timeout 300 python tools/quick_matrix.py 3 4 2>&1 | grep " all" | cut -c1-100,190-260 >> $out
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
