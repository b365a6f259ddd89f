mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 600 python bench.py --slabs --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_slabs1.json 2> gpurun_out/bench_slabs1.err; echo "rc=$?" >> gpurun_out/bench_slabs1.err
timeout 900 python tools/model_scaling.py --config 3 > gpurun_out/model_cfg3.jsonl 2> gpurun_out/model_cfg3.err; echo "rc=$?" >> gpurun_out/model_cfg3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:near_mode_mma -s 3 -c 1 -o gpurun_out/mma_cfg3_head python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_mma.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_bench.log 2>&1
echo done
