mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py tests/test_gpu_slabs.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_ring.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ring.log
timeout 600 python bench.py --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_ring.json 2> gpurun_out/bench_ring.err
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_c5_ring.json 2> gpurun_out/bench_c5_ring.err
timeout 600 python bench.py --config 2 --no-cpu-baseline --no-nosym --gmres-max-iter 30 > gpurun_out/bench_c2_ring.json 2> gpurun_out/bench_c2_ring.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_ring.csv python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_ring.log 2>&1
echo done
