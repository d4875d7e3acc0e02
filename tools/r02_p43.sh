mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 1:101 > gpurun_out/p43_regions.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "region or adversarial or traj or table" > gpurun_out/p43_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p43_pytest.log
echo done
