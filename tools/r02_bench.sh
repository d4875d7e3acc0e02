# default bench line + launch list of the same command
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench.err
echo "bench_rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-secondary --cpu-seconds 1 > gpurun_out/bench_ncu.log 2>&1
echo done
