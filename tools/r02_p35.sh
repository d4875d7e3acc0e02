# stream-ordered scratch: workloads config 1 + 3, region tests
mkdir -p gpurun_out
timeout 600 python tools/workloads.py 1 3 > gpurun_out/p35_workloads.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "region or table or traj or adversarial or variants" > gpurun_out/p35_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p35_pytest.log
echo done
