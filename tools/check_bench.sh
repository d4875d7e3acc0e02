mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
VISRT_TRAJ_PROFILE=1 timeout 300 python tools/quick_traj.py 3:1:1000 3:2:200 1:1:100 1:2:100 > gpurun_out/tp.log 2>&1
