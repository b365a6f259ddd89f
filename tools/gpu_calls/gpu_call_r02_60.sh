mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "m2l_z_forms or flat_stream or fmm_matvec" 2>&1 | tail -3
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_matvec.py --config $CFG --applies 50 2>&1 | tail -2 | head -1| cut -c1-330; }
for c in 3 5; do export CFG=$c
run FPBEM_SERIAL=1
run FPBEM_SERIAL=0
done
