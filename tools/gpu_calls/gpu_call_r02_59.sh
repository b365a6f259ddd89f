mkdir -p gpurun_out
FPBEM_PDL=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py tests/test_gpu_config_scale.py -m gpu -x -q 2>&1 | tail -4
for pdl in 0 1 0 1; do
  FPBEM_PDL=$pdl timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym > gpurun_out/bench_pdl$pdl.json 2> gpurun_out/bench_pdl$pdl.err
  python - <<P
import json
d=json.load(open("gpurun_out/bench_pdl$pdl.json"))
print("pdl $pdl", round(d["ms_per_step"],4), d["trials_ms"], "gmres", d["gmres"]["solve_s"], d["gmres"]["iterations"])
P
done
FPBEM_PDL=1 timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 pdl1', d['ms_per_step'], d['gmres']['solve_s'])"
FPBEM_PDL=0 timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 pdl0', d['ms_per_step'], d['gmres']['solve_s'])"
