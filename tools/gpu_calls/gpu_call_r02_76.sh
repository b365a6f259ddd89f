mkdir -p gpurun_out
for pdl in 0 2 0 2; do
  FPBEM_PDL=$pdl timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl cfg3', round(d['ms_per_step'],4), 'gmres', round(d['gmres']['solve_s'],5), d['gmres']['iterations'], 'e2e', round(d['e2e']['value']/1e9,4))"
done
for pdl in 0 2; do
  FPBEM_PDL=$pdl timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl cfg5', round(d['ms_per_step'],4), 'gmres', round(d['gmres']['solve_s'],5), d['gmres']['iterations'], 'e2e', round(d['e2e']['value']/1e9,4))"
  FPBEM_PDL=$pdl timeout 600 python bench.py --config 2 --no-cpu-baseline --no-nosym 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl cfg2', round(d['ms_per_step'],4), 'gmres', round(d['gmres']['solve_s'],5), d['gmres']['iterations'], 'e2e', round(d['e2e']['value']/1e9,4))"
done
