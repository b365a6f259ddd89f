mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_dist_gmres.py tests/test_gpu_parity.py tests/test_gpu_cpp_driver.py -m gpu -q -rf --durations=15 -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b.log
timeout 300 python tools/profile_gmres.py --config 3 --iters 100 > gpurun_out/prof_gmres.txt 2>&1
timeout 300 python tools/profile_gmres.py --config 5 --nrhs 64 --iters 20 >> gpurun_out/prof_gmres.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gmres64.csv python tools/profile_gmres.py --config 5 --nrhs 64 --iters 4 > gpurun_out/ncu_gmres64.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:near_mode_mma -s 3 -c 1 -o gpurun_out/mma_cfg3 python bench.py --steps 3 --warmup 3 --trials 1 --no-cpu-baseline --no-nosym --gmres-max-iter 5 > gpurun_out/ncu_mma.log 2>&1
echo done
