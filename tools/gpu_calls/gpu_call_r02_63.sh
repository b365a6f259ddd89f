mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 300 python tools/profile_matvec.py --config 5 --nrhs $NR --applies 6 2>&1 | tail -2 | head -1| cut -c1-330; }
for nr in 64 16 8; do export NR=$nr
run FPBEM_DFT_PF=0
run FPBEM_DFT_PF=1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "multi_rhs or batched" 2>&1 | tail -3
