# session-5: K4w whole-face shadow certificate on/off
mkdir -p gpurun_out
out=gpurun_out/t3.log
: > $out
for sh in 0 1; do
  echo "== VISRT_K4W_SHADOW=$sh" >> $out
  VISRT_K4W_SHADOW=$sh timeout 600 python tools/quick_regions.py 5:20:rx 5:20:tx 5:200:mix 3:200 1:101 >> $out 2>&1
  VISRT_K4W_SHADOW=$sh timeout 300 python tools/quick_traj.py 3:1:1000 >> $out 2>&1
done
timeout 1500 python -m pytest tests -x -q -m gpu -k "region or table or traj or adversarial or golden or edge" --durations=5 >> $out 2>&1
echo done >> $out
