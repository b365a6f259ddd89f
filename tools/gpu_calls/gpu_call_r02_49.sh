mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "m2l_z_forms or flat_stream" 2>&1 | tail -5
export FPBEM_M2L_Z=stream FPBEM_SERIAL=1
for cfgw in "9 2" "6 2" "12 1" "7 2" "4 2"; do set -- $cfgw; for pr in 0 3; do
echo "warps $1 spw $2 probe $pr"; FPBEM_MS_WARPS=$1 FPBEM_MS_SPW=$2 FPBEM_MS_PROBE=$pr timeout 90 python tools/profile_matvec.py --config 3 --synthetic --applies 30 2>&1 | tail -2 | cut -c1-260
done; done
