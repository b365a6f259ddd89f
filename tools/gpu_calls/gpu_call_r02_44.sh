mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_near_lattice.py -m gpu -q -x -k "full_size or pipelined or matches_oracle_and_direct" -p no:cacheprovider > gpurun_out/pytest_lb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lb.log
timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/bench_lb8.json 2> gpurun_out/bench_lb8.err
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/bench_c5_lb8.json 2> gpurun_out/bench_c5_lb8.err
echo done
