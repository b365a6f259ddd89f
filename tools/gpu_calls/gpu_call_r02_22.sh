mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_dist_gmres.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_slab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slab.log
timeout 900 python tools/model_scaling.py --config 3 > gpurun_out/model_cfg3.jsonl 2> gpurun_out/model_cfg3.err
timeout 600 python bench.py --slabs --no-cpu-baseline --no-nosym --gmres-max-iter 300 > gpurun_out/bench_slabs1.json 2> gpurun_out/bench_slabs1.err
echo done
