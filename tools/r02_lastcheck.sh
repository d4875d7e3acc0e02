mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/f_pytest.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/f_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1
timeout 900 python tools/workloads.py 1 2 3 4 5 > gpurun_out/f_workloads.jsonl 2> gpurun_out/f_workloads.err
