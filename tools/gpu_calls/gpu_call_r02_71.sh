mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_matvec.py --config $CFG --applies 50 2>&1 | tail -2 | head -1| cut -c1-330; }
for c in 3 5; do export CFG=$c
run FPBEM_FUSE_L2P=1
run FPBEM_L2P_CTAS=4
run FPBEM_L2P_CTAS=2
done
for rep in 1 2; do
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']])"
FPBEM_L2P_CTAS=4 timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3 ctas4', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']])"
done
