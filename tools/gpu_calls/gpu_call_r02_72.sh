mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_near_lattice.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_matvec.py --config $CFG --applies 50 2>&1 | tail -2 | head -1| cut -c1-330; }
for c in 3 5; do export CFG=$c
run FPBEM_SERIAL=1
run FPBEM_SERIAL=0
done
for rep in 1 2; do
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']])"
done
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']])"
