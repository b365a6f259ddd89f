mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_parity.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_orbit.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_orbit.log
timeout 900 python tools/model_rhs_shard.py > gpurun_out/model_cfg5_rhs.jsonl 2> gpurun_out/model_cfg5_rhs.err
FPBEM_ORBIT_JOBS=0 timeout 900 python tools/model_rhs_shard.py --ranks 4,8 > gpurun_out/model_cfg5_rhs_noorbit.jsonl 2> gpurun_out/model_cfg5_rhs_noorbit.err
echo done
