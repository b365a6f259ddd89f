mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_dist_gmres.py tests/test_gpu_near_lattice.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_slab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slab.log
timeout 900 python tools/model_scaling.py --config 3 > gpurun_out/model_cfg3.jsonl 2> gpurun_out/model_cfg3.err; echo "rc=$?" >> gpurun_out/model_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p8r0.csv python tools/model_scaling.py --config 3 --only 8,0 --no-gmres --steps 3 > gpurun_out/ncu_p8.log 2>&1
echo done
