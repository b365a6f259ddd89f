mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_near_lattice.py -m gpu -x -q -k "programmatic" 2>&1 | tail -8
timeout 1500 python tools/model_scaling.py --config 3 > gpurun_out/model_scaling_cfg3_2.jsonl 2> gpurun_out/model_scaling.err; tail -5 gpurun_out/model_scaling_cfg3_2.jsonl | cut -c1-600
