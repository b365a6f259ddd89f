mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
timeout 600 python bench.py --config 1 --no-cpu-baseline --no-nosym > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --no-cpu-baseline --no-nosym > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo done
