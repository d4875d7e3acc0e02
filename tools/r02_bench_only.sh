mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
echo "bench_rc=$?" >> gpurun_out/f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1
