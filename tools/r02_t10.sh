mkdir -p gpurun_out
bash tools/r02_t9.sh
timeout 2700 python tools/ref_workloads.py --full 2 4 5 3 > gpurun_out/ref_full.jsonl 2> gpurun_out/ref_full.err
echo done > gpurun_out/t10_done.txt
