mkdir -p gpurun_out
out=gpurun_out/t27.log
: > $out
for c in 1024 256 512 2048 4096; do
  echo "== K4W_CONE=$c" >> $out
  VISRT_K4W_CONE=$c timeout 600 python tools/quick_regions.py 5:500:mix 3:2000 2>&1 | cut -c1-120,200-240 >> $out
done
echo "== FACEMAJOR=0" >> $out
VISRT_K4W_FACEMAJOR=0 timeout 600 python tools/quick_regions.py 5:500:mix 3:2000 2>&1 | cut -c1-120,200-240 >> $out
echo done >> $out
