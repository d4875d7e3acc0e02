# session-5: K4w tasks per warp grab on whole-workload batch sizes
mkdir -p gpurun_out
out=gpurun_out/t22.log
: > $out
for v in 1 2 4 8 16; do
  VISRT_NVCC_FLAGS="-DVISRT_K4W_CHUNK=$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== K4W_CHUNK=$v" >> $out
  timeout 600 python tools/quick_regions.py 5:500:mix 5:20:rx 3:2000 2>&1 | cut -c1-230 >> $out
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
