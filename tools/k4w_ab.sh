# A/B of K4w build flags: bash tools/k4w_ab.sh "<flags A>" "<flags B>" ... (regions + trajectory timings, output hashes)
mkdir -p gpurun_out
: > gpurun_out/k4w_ab.log
for cfg in "$@"; do
  VISRT_NVCC_FLAGS="$cfg" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
  echo "== $cfg" >> gpurun_out/k4w_ab.log
  timeout 300 python tools/quick_regions.py 1:101 3:200 5:20 >> gpurun_out/k4w_ab.log 2>&1
  timeout 300 python tools/quick_traj.py 3:1:1000 >> gpurun_out/k4w_ab.log 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
