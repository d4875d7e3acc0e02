# K2 tuning sweep (development aid): build variants, time configs 2 and 3
mkdir -p gpurun_out
for cfg in ${K2_VARIANTS:-"-DVISRT_K2W_NOSAT=1"}; do
  VISRT_NVCC_FLAGS="$cfg" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
  echo "== $cfg" >> gpurun_out/k2sweep14.log
  python tools/quick_matrix.py 2 3 >> gpurun_out/k2sweep14.log 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
python -m pytest tests/test_matrix_gpu.py tests/test_golden_gpu.py -x -q -m gpu >> gpurun_out/k2sweep14.log 2>&1
