# session-5: K6 fused last level, receiver-side cull before the unfold
mkdir -p gpurun_out
out=gpurun_out/t7.log
: > $out
for v in "-DVISRT_K6L_RXCULL=0" "-DVISRT_K6L_RXCULL=1"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  timeout 300 python tools/quick_tree.py 3:3:50 3:2:200 5:3:500 1:2:100 >> $out 2>&1
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "tree or trace or aux or dropin or golden" --durations=5 >> $out 2>&1
echo done >> $out
