mkdir -p gpurun_out
: > gpurun_out/seg.log
for w in 0 1; do
  echo "== VISRT_SEG_WARP=$w" >> gpurun_out/seg.log
  VISRT_SEG_WARP=$w VISRT_TRAJ_PROFILE=1 python tools/quick_traj.py 3:1:1000 >> gpurun_out/seg.log 2>&1
  VISRT_SEG_WARP=$w python tools/quick_tree.py 3:3:50 1:2:100 >> gpurun_out/seg.log 2>&1
done
timeout 900 python -m pytest tests/test_tables_gpu.py tests/test_trajectory_gpu.py tests/test_aux_gpu.py -x -q -m gpu >> gpurun_out/seg.log 2>&1
