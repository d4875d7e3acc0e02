# K2w build variants (development aid): configs 2, 3 full and config 4 on every 7th pair
mkdir -p gpurun_out
out=gpurun_out/k2w_var.log
for v in "${@}"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  python tools/quick_matrix.py 2 3 2>&1 >> $out
  python tools/quick_matrix.py 4 2>&1 >> $out
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
