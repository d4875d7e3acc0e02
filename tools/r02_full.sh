# every -m gpu test + smoke
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/full_pytest.log 2>&1
echo "pytest_rc=$?" >> gpurun_out/full_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1
echo "smoke_rc=$?" >> gpurun_out/full_smoke.log
echo done
