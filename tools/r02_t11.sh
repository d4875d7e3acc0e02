# session-5: K7 screen with the prefix pair's points read from shared memory; larger K2w tiles on config 4
mkdir -p gpurun_out
out=gpurun_out/t11.log
: > $out
timeout 300 python tools/quick_chains.py 1 2 3 >> $out 2>&1
timeout 300 python tools/quick_chains.py 3 2 >> $out 2>&1
for v in "-DVISRT_K2W_TR=8 -DVISRT_K2W_TC=8 -DVISRT_K2W_WC_TILED=6" "-DVISRT_K2W_TR=8 -DVISRT_K2W_TC=8 -DVISRT_K2W_WC_TILED=10" \
         "-DVISRT_K2W_TR=8 -DVISRT_K2W_TC=8 -DVISRT_K2W_WC_TILED=12" "-DVISRT_K2W_TR=8 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=8" \
         "-DVISRT_K2W_TR=16 -DVISRT_K2W_TC=8 -DVISRT_K2W_WC_TILED=8" "-DVISRT_K2W_TR=16 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=8" \
         "-DVISRT_K2W_TR=16 -DVISRT_K2W_TC=16 -DVISRT_K2W_WC_TILED=12" "-DVISRT_K2W_TR=4 -DVISRT_K2W_TC=32 -DVISRT_K2W_WC_TILED=8" \
         "-DVISRT_K2W_TR=32 -DVISRT_K2W_TC=32 -DVISRT_K2W_WC_TILED=12"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  timeout 300 python tools/quick_matrix.py 3 4 2>&1 | grep " all" | cut -c1-120 >> $out
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
