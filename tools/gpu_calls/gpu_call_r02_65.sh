mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "other_orders" 2>&1 | tail -2
for w in 11 7 5 4 3; do for rep in 1 2; do
  FPBEM_MS_WARPS=$w timeout 600 python bench.py --config 3 --no-cpu-baseline --no-nosym --gmres-max-iter 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warps $w', round(d['ms_per_step'],4), [round(t,2) for t in d['trials_ms']], round(d['stages_serial_ms']['m2l'],4))"
done; done
