# K4w i-cache shrink: timings + sha, region tests, phase profile
mkdir -p gpurun_out
timeout 300 python tools/quick_regions.py 5:20:rx 5:20:tx 3:200 1:101 > gpurun_out/p8_regions.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "region or adversarial or traj or table" > gpurun_out/p8_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/p8_pytest.log
VISRT_NVCC_FLAGS=-DVISRT_K4W_PROF python -m paper_2501_02747_b200.build --force > gpurun_out/p8_build.log 2>&1
timeout 300 python tools/k4w_prof.py 5:20:rx 5:20:tx > gpurun_out/p8_k4wprof.log 2>&1
echo done
