mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 600 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_dist_gmres.py -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/pytest_slab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slab.log
timeout 900 python tools/model_scaling.py --config 3 > gpurun_out/model_cfg3.jsonl 2> gpurun_out/model_cfg3.err; echo "rc=$?" >> gpurun_out/model_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p8r0.csv python tools/model_scaling.py --config 3 --only 8,0 --no-gmres --steps 3 > gpurun_out/ncu_p8.log 2>&1
FPBEM_SLAB_GRAPH=0 timeout 600 python tools/model_scaling.py --config 3 --only 8,0 --no-gmres > gpurun_out/model_p8_nograph.jsonl 2>&1
timeout 300 python tools/profile_gmres.py --config 3 --iters 100 > gpurun_out/prof_gmres.txt 2>&1
timeout 600 python tools/profile_gmres.py --config 5 --nrhs 64 --iters 10 >> gpurun_out/prof_gmres.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:mgs --csv --log-file gpurun_out/launches_mgs.csv python tools/profile_gmres.py --config 3 --iters 50 > gpurun_out/ncu_mgs.log 2>&1
echo done
