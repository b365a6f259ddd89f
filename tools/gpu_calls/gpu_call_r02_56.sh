mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_dist_gmres.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_sl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sl.log
timeout 900 python tools/model_scaling.py --config 3 > gpurun_out/model_cfg3.jsonl 2> gpurun_out/model_cfg3.err
echo done
