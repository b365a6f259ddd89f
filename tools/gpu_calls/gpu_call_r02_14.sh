mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_slabs.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_slab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slab.log
echo done
