mkdir -p gpurun_out
out=gpurun_out/t26.log
: > $out
echo "== lazy" >> $out
timeout 300 python tools/quick_chains.py 3 3 3 2>&1 | cut -c60-200 >> $out
echo "== eager" >> $out
CUDA_MODULE_LOADING=EAGER timeout 300 python tools/quick_chains.py 3 3 3 2>&1 | cut -c60-200 >> $out
echo "== workloads 3 twice" >> $out
timeout 300 python tools/workloads.py 3 3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['total_device_ms'], {k:(v['device_ms'], v['wall_ms']) for k,v in d.items() if isinstance(v,dict)})" >> $out 2>&1
