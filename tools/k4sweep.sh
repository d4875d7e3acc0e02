mkdir -p gpurun_out
: > gpurun_out/k4s.log
for cfg in "-DVISRT_K4W_MINB=2" "-DVISRT_K4W_MINB=3" "-DVISRT_K4W_MINB=4"; do
  VISRT_NVCC_FLAGS="$cfg" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
  echo "== $cfg" >> gpurun_out/k4s.log
  python tools/quick_regions.py 1:101 3:200 5:20 >> gpurun_out/k4s.log 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
