# session-5 A/B: record loads as double2 (VISRT_SEG_V2) and the K7 mid-axis pre-reject (VISRT_K7_PRE)
mkdir -p gpurun_out
out=gpurun_out/t1.log
: > $out
for v in "-DVISRT_SEG_V2=0 -DVISRT_K7_PRE=0" "-DVISRT_SEG_V2=1 -DVISRT_K7_PRE=2" "-DVISRT_SEG_V2=1 -DVISRT_K7_PRE=1"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  timeout 300 python tools/quick_chains.py 1 2 3 >> $out 2>&1
  case "$v" in *PRE=1*) continue;; esac
  timeout 300 python tools/quick_matrix.py 2 3 4 >> $out 2>&1
  timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 >> $out 2>&1
  timeout 300 python tools/quick_tree.py 3:3:50 >> $out 2>&1
done
VISRT_NVCC_FLAGS="-DVISRT_K7_STATS" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo "== stats" >> $out
timeout 300 python tools/k7_stats.py 3 >> $out 2>&1
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
