mkdir -p gpurun_out
out=gpurun_out/t23.log
: > $out
timeout 600 python tools/quick_regions.py 3:2000 3:200 1:101 5:20:rx 2>&1 | cut -c1-230 >> $out
timeout 300 python tools/quick_traj.py 3:1:1000 >> $out 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -k "region or table or traj or golden or dropin or adversarial" >> $out 2>&1
timeout 900 python tools/workloads.py 3 > gpurun_out/t23_workloads3.jsonl 2>> $out
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
echo "bench_rc=$?" >> gpurun_out/f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
echo done >> $out
