mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "m2l_z_forms or flat_stream" 2>&1 | tail -30
