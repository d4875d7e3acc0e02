# K4w build variants (development aid): regions configs 1, 3, 5 (sha-checked) + config-1 trajectory
mkdir -p gpurun_out
out=gpurun_out/k4w_var.log
for v in "${@}"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  python tools/quick_regions.py 1:101 3:200:mix 5:20:rx 5:20:tx >> $out 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
