# Full GPU check used between milestones: tests, bench, K2 launch list + full ncu capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/pytest_all.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-secondary > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pair_bits -c 1 -o gpurun_out/k2_full -f python bench.py --steps 1 --warmup 0 --no-secondary > gpurun_out/ncu_full.log 2>&1
