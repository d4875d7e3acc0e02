mkdir -p gpurun_out
out=gpurun_out/t8.log
: > $out
python tools/quick_rows.py 4 11000 11016 >> $out 2>&1
VISRT_NOCULL=1 timeout 600 python tools/quick_rows.py 4 11000 11016 >> $out 2>&1
python tools/quick_rows.py 4 300 316 >> $out 2>&1
VISRT_NOCULL=1 timeout 600 python tools/quick_rows.py 4 300 316 >> $out 2>&1
echo done >> $out
