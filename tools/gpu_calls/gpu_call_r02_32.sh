mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_config_scale.py -m gpu -q -x -rf -p no:cacheprovider -k "multi_rhs or batched or partition or cfg5" > gpurun_out/pytest_orbit2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_orbit2.log
timeout 900 python tools/model_rhs_shard.py > gpurun_out/model_cfg5_rhs.jsonl 2> gpurun_out/model_cfg5_rhs.err
echo done
