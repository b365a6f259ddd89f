mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py tests/test_gpu_config_scale.py tests/test_gpu_cpp_driver.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_flag.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_flag.log
timeout 300 python tools/profile_gmres.py --config 3 --iters 100 > gpurun_out/prof_gmres_flag.txt 2>&1
FPBEM_MGS_FLAGBAR=0 timeout 300 python tools/profile_gmres.py --config 3 --iters 100 >> gpurun_out/prof_gmres_flag.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-nosym > gpurun_out/bench_flag.json 2> gpurun_out/bench_flag.err
timeout 600 python tools/time_lockstep.py 5 64 > gpurun_out/lockstep64_flag.jsonl 2>&1
echo done
