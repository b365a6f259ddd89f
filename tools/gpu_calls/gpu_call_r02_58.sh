mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py -m gpu -x -q 2>&1 | tail -4
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_matvec.py --config $CFG --applies 50 2>&1 | tail -2 | head -1| cut -c1-330; }
for c in 3 5 2; do export CFG=$c
run FPBEM_DFT_PF=1
run FPBEM_DFT_PF=0
run FPBEM_DFT_PF=1 FPBEM_SERIAL=1
run FPBEM_DFT_PF=0 FPBEM_SERIAL=1
done
