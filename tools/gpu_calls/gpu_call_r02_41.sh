mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python bench.py --config 1 --no-cpu-baseline --no-nosym > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
echo done
