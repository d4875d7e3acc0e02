# whole workloads of every config (device + wall)
mkdir -p gpurun_out
timeout 1500 python tools/workloads.py 1 2 3 4 5 > gpurun_out/p38_workloads.jsonl 2> gpurun_out/p38_workloads.err
echo done
