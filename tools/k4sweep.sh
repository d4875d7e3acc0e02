mkdir -p gpurun_out
: > gpurun_out/k4s.log
for cfg in "-DVISRT_K4W_FIRST=0" "-DVISRT_K4W_FIRST=1" "-DVISRT_K4W_FIRST=4" "-DVISRT_K4W_FIRST=8"; do
  VISRT_NVCC_FLAGS="$cfg" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
  echo "== $cfg" >> gpurun_out/k4s.log
  VISRT_K4_WARP=1 python tools/quick_regions.py 1:101 3:200 >> gpurun_out/k4s.log 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
