# session-5: K6 last-level grab size / register budget, K7 decide register budget
mkdir -p gpurun_out
out=gpurun_out/t18.log
: > $out
for v in "-DVISRT_K6L_GRAB=4" "-DVISRT_K6L_GRAB=1" "-DVISRT_K6L_GRAB=2" "-DVISRT_K6L_GRAB=8" "-DVISRT_K6L_GRAB=16" "-DVISRT_K6L_MINB=2" "-DVISRT_K6L_MINB=4" \
         "-DVISRT_K7_MINB=3" "-DVISRT_K7_MINB=4" "-DVISRT_K7_MINB=6" "-DVISRT_K7_MINB=8"; do
  VISRT_NVCC_FLAGS="$v" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1 || echo "build failed $v" >> $out
  echo "== $v" >> $out
  case "$v" in
    *K6L*) timeout 300 python tools/quick_tree.py 3:3:50 5:3:500 >> $out 2>&1 ;;
    *K7*) timeout 300 python tools/quick_chains.py 3 2 2>&1 | cut -c1-150 >> $out ;;
  esac
done
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
