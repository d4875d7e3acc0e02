mkdir -p gpurun_out
out=gpurun_out/t19.log
: > $out
timeout 300 python tools/quick_tree.py 3:3:50 3:2:200 5:3:500 1:2:100 >> $out 2>&1
for v in "-DVISRT_K2W_MINB=2" "-DVISRT_K2W_MINB=4"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  timeout 300 python tools/quick_matrix.py 2 3 4 2>&1 | grep " all" | cut -c1-100 >> $out
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
