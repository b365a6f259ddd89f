mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gmres" 2>&1 | tail -3
for sp in 1 0 1 0; do
FPBEM_MGS_SPARE=$sp timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('spare $sp cfg3 gmres', round(d['gmres']['solve_s'],5), d['gmres']['iterations'], round(d['gmres']['ms_per_iteration'],4), d['gmres']['final_estimate'])"
done
for sp in 1 0; do
FPBEM_MGS_SPARE=$sp timeout 600 python tools/time_lockstep.py 5 64 2>/dev/null | tail -1
done
