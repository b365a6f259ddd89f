mkdir -p gpurun_out
for pdl in 0 2 1 0 2; do
  FPBEM_PDL=$pdl timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl cfg3', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']])"
done
for pdl in 0 2; do
  FPBEM_PDL=$pdl timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl $pdl cfg5', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']])"
done
