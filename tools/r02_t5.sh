# session-5: K2w settling passes preload the blocker's plane words; one post-sweep resolve site
mkdir -p gpurun_out
out=gpurun_out/t5.log
: > $out
for v in "-DVISRT_K2W_PRELOAD=0 -DVISRT_K2W_RLOOP=0" "-DVISRT_K2W_PRELOAD=1 -DVISRT_K2W_RLOOP=0" "-DVISRT_K2W_PRELOAD=0 -DVISRT_K2W_RLOOP=1" "-DVISRT_K2W_PRELOAD=1 -DVISRT_K2W_RLOOP=1"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  timeout 300 python tools/quick_matrix.py 2 3 4 2>&1 | grep " all" >> $out
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
