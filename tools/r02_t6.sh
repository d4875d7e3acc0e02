# session-5: K7 decide kernel with mask-driven section pairs; per-kernel times of the two K7 kernels
mkdir -p gpurun_out
out=gpurun_out/t6.log
: > $out
timeout 300 python tools/quick_chains.py 1 2 3 >> $out 2>&1
timeout 300 python tools/quick_chains.py 3 2 >> $out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_chain --csv --log-file gpurun_out/t6_k7_launches.csv python tools/quick_chains.py 3 > /dev/null 2>&1
grep -E "k_chain" gpurun_out/t6_k7_launches.csv | awk -F'","' '{print $5, $NF}' >> $out
VISRT_NVCC_FLAGS="-DVISRT_K7_MASKS=0" python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
echo "== MASKS=0" >> $out
timeout 300 python tools/quick_chains.py 3 2 >> $out 2>&1
python paper_2501_02747_b200/build.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_chains_gpu.py tests/test_fullsize_ref_gpu.py tests/test_matrix_gpu.py -x -q -m gpu -k "chain or matrix" >> $out 2>&1
echo done >> $out
