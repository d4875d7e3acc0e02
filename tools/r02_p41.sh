# K7 prefix-pair precomputation: A/B vs HEAD, sha of the triples, chain tests
mkdir -p gpurun_out
timeout 300 python tools/quick_chains.py 1 2 3 > gpurun_out/p41_pre.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "chain or dropin or cache or tree" > gpurun_out/p41_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p41_pytest.log
echo done
