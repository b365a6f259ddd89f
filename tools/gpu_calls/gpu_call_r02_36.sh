mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python tools/time_lockstep.py 5 64 > gpurun_out/lockstep64.jsonl 2> gpurun_out/lockstep64.err
timeout 600 python bench.py --config 1 --no-cpu-baseline --no-nosym > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
echo done
