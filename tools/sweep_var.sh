# Sweep build variants (development aid): matrix configs 2-4, regions configs 3 and 5, order-3 trees config 3
mkdir -p gpurun_out
out=gpurun_out/sweep_var.log
for v in "${@}"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  python tools/quick_matrix.py 2 3 4 2>&1 | grep " all:" >> $out
  python tools/quick_regions.py 3:200:mix 5:20:rx 5:20:tx >> $out 2>&1
  python tools/quick_tree.py 3:3:50 5:3:500 >> $out 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
