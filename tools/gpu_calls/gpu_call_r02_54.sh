mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "m2l_z_forms or flat_stream" 2>&1 | tail -3
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_matvec.py --config 3 --applies 50 2>&1 | tail -2 | head -1| cut -c1-330; }
run FPBEM_M2L_Z=stream FPBEM_SERIAL=1
run FPBEM_M2L_Z=stream FPBEM_SERIAL=1 FPBEM_MS_WARPS=6
run FPBEM_M2L_Z=stream FPBEM_SERIAL=1 FPBEM_MS_WARPS=9 FPBEM_MS_SPW=1 FPBEM_MS_RING=9
run FPBEM_M2L_Z=stream
run FPBEM_M2L_Z=fused
