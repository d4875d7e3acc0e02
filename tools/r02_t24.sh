mkdir -p gpurun_out
out=gpurun_out/t24.log
: > $out
timeout 300 python tools/quick_chains.py 1 2 3 >> $out 2>&1
timeout 300 python tools/quick_chains.py 3 2 >> $out 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "chain or dropin or cache" >> $out 2>&1
VISRT_NVCC_FLAGS="-DVISRT_K7_SPLIT2=0" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo "== SPLIT2=0" >> $out
timeout 300 python tools/quick_chains.py 3 2 >> $out 2>&1
timeout 300 python tools/quick_chains.py 3 2 >> $out 2>&1
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo done >> $out
