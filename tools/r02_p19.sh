# refine_fan without the collecting-sweep fallback; per-kernel launch times
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 1:101 > gpurun_out/p19_regions.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p19_launches.csv python tools/quick_regions.py 5:20:rx 5:20:tx > /dev/null 2>&1
echo done
