mkdir -p gpurun_out
export FPBEM_M2L_Z=stream FPBEM_SERIAL=1
for pr in 0 3; do for ring in 0 8; do
echo "probe $pr ring $ring"; CUDA_LAUNCH_BLOCKING=$CLB FPBEM_MS_PROBE=$pr FPBEM_MS_RING=$ring timeout 300 python tools/profile_matvec.py --config 3 --synthetic --applies 30 2>&1 | tail -2
done; done
