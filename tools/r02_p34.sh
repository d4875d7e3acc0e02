# config-1 tables regression hunt: workloads config 1 default / no cone / lane kernel
mkdir -p gpurun_out
timeout 300 python tools/workloads.py 1 > gpurun_out/p34_default.jsonl 2>&1
VISRT_K4W_CONE=0 timeout 300 python tools/workloads.py 1 > gpurun_out/p34_nocone.jsonl 2>&1
timeout 300 python tools/quick_regions.py 1:101 1:101 > gpurun_out/p34_regions.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p34_launches.csv python tools/workloads.py 1 > /dev/null 2>&1
echo done
