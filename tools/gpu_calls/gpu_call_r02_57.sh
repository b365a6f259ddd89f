mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5"
timeout 600 $CMD > gpurun_out/plain_bench.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_s4.csv $CMD > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mode_stream -s 3 -c 1 -o gpurun_out/mode_stream_cfg3 $CMD > gpurun_out/ncu_ms.log 2>&1
ls -la gpurun_out/*.ncu-rep
