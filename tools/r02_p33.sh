# K2w pair capsule for cached blockers: A/B + matrix tests
mkdir -p gpurun_out
timeout 600 python tools/quick_matrix.py 2 3 4 > gpurun_out/p33_cap.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "matrix or variants or adversarial" > gpurun_out/p33_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p33_pytest.log
VISRT_NVCC_FLAGS="-DVISRT_K2W_PAIRCAP=0" python -m paper_2501_02747_b200.build --force > /dev/null 2>&1
timeout 600 python tools/quick_matrix.py 2 3 4 > gpurun_out/p33_nocap.log 2>&1
echo done
