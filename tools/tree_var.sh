# K6 build variants (development aid): order-3 trees configs 3 and 5, order-2 config 1
mkdir -p gpurun_out
out=gpurun_out/tree_var.log
for v in "${@}"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  python tools/quick_tree.py 1:2:100 3:3:50 5:3:500 >> $out 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
