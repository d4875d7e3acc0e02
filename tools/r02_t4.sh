# session-5: K4w cone list after N blocked sweeps
mkdir -p gpurun_out
out=gpurun_out/t4.log
: > $out
for v in 0 2 4 8; do
  VISRT_NVCC_FLAGS="-DVISRT_K4W_CONE_AFTER=$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== CONE_AFTER=$v" >> $out
  timeout 600 python tools/quick_regions.py 5:20:rx 5:20:tx 5:200:mix 3:200 1:101 >> $out 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
