mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_dist_gmres.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
timeout 600 python bench.py --slabs --no-cpu-baseline --no-nosym > gpurun_out/bench_slabs1.json 2> gpurun_out/bench_slabs1.err
timeout 2400 python tools/bench_configs.py --sweep --out gpurun_out/configs_r02.jsonl > gpurun_out/configs_r02.log 2>&1; echo "rc=$?" >> gpurun_out/configs_r02.log
for c in 1 2 4 5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
echo done
