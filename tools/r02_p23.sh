# K7 variants: compact caps + V2 hull (default) / byte-index hull / wide; time + DRAM
mkdir -p gpurun_out
for v in "" "-DVISRT_K7_HULLIDX=1" "-DVISRT_K7_COMPACT=0"; do
  VISRT_NVCC_FLAGS="$v" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
  echo "variant [$v]" >> gpurun_out/p23_chains.log
  timeout 300 python tools/quick_chains.py 2 3 >> gpurun_out/p23_chains.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_chain_triples --csv python tools/quick_chains.py 3 2>/dev/null | grep -E "dram|duration" >> gpurun_out/p23_chains.log
done
echo done
