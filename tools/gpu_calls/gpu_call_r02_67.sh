mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near_lattice.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2 3; do
  timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']], round(d['stages_serial_ms']['m2l'],4), round(d['stages_serial_ms']['near_gemm'],4))"
done
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']], round(d['stages_serial_ms']['m2l'],4), round(d['stages_serial_ms']['near_gemm'],4))"
timeout 600 python bench.py --config 2 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']], round(d['stages_serial_ms']['m2l'],4), round(d['stages_serial_ms']['near_gemm'],4))"
