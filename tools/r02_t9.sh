# session-5: K2w tile shape / tiled cache size sweep on configs 3 and 4
mkdir -p gpurun_out
out=gpurun_out/t9.log
: > $out
for v in "-DVISRT_K2W_TR=2 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=6" "-DVISRT_K2W_TR=2 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=8" \
         "-DVISRT_K2W_TR=4 -DVISRT_K2W_TC=8 -DVISRT_K2W_WC_TILED=6" "-DVISRT_K2W_TR=4 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=6" \
         "-DVISRT_K2W_TR=4 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=8" "-DVISRT_K2W_TR=2 -DVISRT_K2W_TC=32 -DVISRT_K2W_WC_TILED=6" \
         "-DVISRT_K2W_TR=8 -DVISRT_K2W_TC=8 -DVISRT_K2W_WC_TILED=8" "-DVISRT_K2W_TR=3 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=6"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  timeout 300 python tools/quick_matrix.py 3 4 2>&1 | grep " all" | cut -c1-120 >> $out
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
