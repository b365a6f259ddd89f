mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2 3; do for fo in 0 2; do for cfg in 3; do
  FPBEM_FAR_ORDER=$fo timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-nosym > gpurun_out/bench_fo.json 2> gpurun_out/bench_fo.err
  python - <<P
import json
d=json.load(open("gpurun_out/bench_fo.json"))
print("far_order $fo cfg$cfg", round(d["ms_per_step"],4), [round(t,2) for t in d["trials_ms"]], "gmres", round(d["gmres"]["solve_s"],4), d["gmres"]["iterations"], "e2e", d["e2e"]["value"])
P
done; done; done
for fo in 0 2; do FPBEM_FAR_ORDER=$fo timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 fo$fo', d['ms_per_step'], d['gmres']['solve_s'])"; done
